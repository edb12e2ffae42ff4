"""The C-ABI boundary: libsmx.so loads without a GPU and exports every entry point
include/smx.h declares, with the documented constants."""
import ctypes
import re

from oracle_lib import ROOT, layout
from paper_2006_11972_b200 import executor as ex

HEADER = (ROOT / "include" / "smx.h").read_text()


def declared():
    return sorted(set(re.findall(r"^(?:int|const char\*)\s+(smx_\w+)\(", HEADER, re.M)))


def test_header_declares_expected_entry_points():
    assert declared() == sorted(ex.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(str(ex.LIB_PATH))
    for name in declared():
        assert hasattr(lib, name), name


def test_constants_match_header():
    for name, val in [("SMX_OK", ex.SMX_OK), ("SMX_ECONFIG", ex.SMX_ECONFIG), ("SMX_EINTEGRITY", ex.SMX_EINTEGRITY),
                      ("SMX_EDEVICE", ex.SMX_EDEVICE), ("SMX_GEMM_EXACT", ex.GEMM_EXACT), ("SMX_GEMM_TC", ex.GEMM_TC),
                      ("SMX_HP_COLS", ex.HP_COLS), ("SMX_MET_COLS", ex.MET_COLS), ("SMX_MODEL_MLP", ex.MODEL_MLP),
                      ("SMX_MODEL_CNN", ex.MODEL_CNN)]:
        m = re.search(rf"#define {name} (\d+)", HEADER)
        assert m and int(m.group(1)) == val, name


def test_version_and_param_count_without_gpu():
    lib = ex.load_library()
    assert b"sm_100a" in lib.smx_version()
    p, pa = ctypes.c_int64(), ctypes.c_int64()
    assert lib.smx_param_count(None, ctypes.byref(p), ctypes.byref(pa)) == 0
    p_algo, p_alloc, _ = layout()
    assert (p.value, pa.value) == (p_algo, p_alloc) == (269322, 270912)


def test_open_without_gpu_fails_loudly():
    """No silent CPU fallback: opening a context needs a device."""
    import pytest

    try:
        e = ex.Executor(n_slots=1, n_ckpts=1)
    except ex.SmxError as err:
        assert "device" in str(err).lower() or "cuda" in str(err).lower()
        return
    e.close()
    pytest.skip("GPU present")


def test_struct_sizes():
    assert ctypes.sizeof(ex.ModelDesc) == 32
    assert ctypes.sizeof(ex.Stats) == 8 * 11


def test_host_stub_covers_the_whole_abi():
    """The CPU test stand-in (tests/native/smx_stub.cpp) implements every declared entry point,
    so the engine tests run against the same ABI the product links."""
    import glob

    libs = glob.glob(str(ROOT / "tests" / "native" / "_stagemerge_stub*.so"))
    assert libs, "run python -m paper_2006_11972_b200.build"
    lib = ctypes.CDLL(libs[0])
    for name in declared():
        assert hasattr(lib, name), name
