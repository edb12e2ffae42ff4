// pybind11 module `_stagemerge`: the Python face of the C++ host library (used by tests, the
// bench driver and __graft_entry__).  The product logic lives in the C++ sources next to this
// file; this only marshals.
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <string>

namespace stagemerge::api {
std::string call(const std::string& text);
}

void bind_engine(pybind11::module_& m);

// The test build (tests/native, linked against the host-only smx stub instead of libsmx.so)
// compiles this file again with -DSMH_MODULE=_stagemerge_stub.
#ifndef SMH_MODULE
#define SMH_MODULE _stagemerge
#endif

PYBIND11_MODULE(SMH_MODULE, m) {
    m.doc() = "stagemerge host library (C++20) over the smx B200 executor";
    m.def("call", &stagemerge::api::call, "JSON command interface (same commands as the reference shim)");
    bind_engine(m);
}
