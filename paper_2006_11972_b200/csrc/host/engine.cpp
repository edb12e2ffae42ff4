#include <pybind11/pybind11.h>
void bind_engine(pybind11::module_&) {}
