"""In-tree build of every native artefact (sm_100a CUDA + C++ host + the test oracles).

    python -m paper_2006_11972_b200.build          # everything that is out of date

Outputs (git-ignored, but shipped to the GPU box by gpurun's snapshot):
    paper_2006_11972_b200/libsmx.so               executor: CUDA kernels + C ABI (include/smx.h)
    paper_2006_11972_b200/_stagemerge*.so         host library (C++ stagemerge API) + Python binding
    oracle/liboracle.so                           CPU oracle (test infrastructure)
    tests/native/_stagemerge_stub*.so             host library over a host-only smx stub (CPU tests of the
                                                  engine / scheduler; test infrastructure, not shipped)
    oracle/_ref/libstagemerge_ref.so              reference hpseq/plan, only when /root/reference exists
"""
from __future__ import annotations

import os
import subprocess
import sys
import sysconfig
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
INCLUDE = ROOT / "include"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NLOHMANN = Path(sysconfig.get_paths()["purelib"]) / "include/cudnn_frontend/thirdparty/nlohmann"

CUDA_SOURCES = [CSRC / "smx.cu"]
CUDA_DEPS = CUDA_SOURCES + sorted((CSRC / "kernels").glob("*.cuh")) + [INCLUDE / "smx.h"]
HOST_SOURCES = sorted((CSRC / "host").glob("*.cpp"))
HOST_DEPS = HOST_SOURCES + sorted((CSRC / "host").glob("*.hpp")) + sorted((INCLUDE / "stagemerge").glob("*.hpp"))


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


def _run(cmd, cwd=None):
    print("+", " ".join(str(c) for c in cmd), flush=True)
    subprocess.run([str(c) for c in cmd], check=True, cwd=cwd)


def build_smx(force: bool = False) -> Path:
    out = PKG / "libsmx.so"
    if force or _stale(out, CUDA_DEPS):
        _run([NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-fmad=false", "-Xptxas", "-v,-warn-spills",
              "-Xcompiler", "-fPIC,-Wall", "-shared", f"-I{INCLUDE}", "-o", out, *CUDA_SOURCES])
    return out


def host_ext_path() -> Path:
    return PKG / ("_stagemerge" + sysconfig.get_config_var("EXT_SUFFIX"))


def build_host(force: bool = False) -> Path | None:
    if not HOST_SOURCES:
        return None
    out = host_ext_path()
    smx = PKG / "libsmx.so"
    if not (force or _stale(out, HOST_DEPS + [smx])):
        return out
    import pybind11
    from concurrent.futures import ThreadPoolExecutor

    objdir = PKG / "build" / "host"
    objdir.mkdir(parents=True, exist_ok=True)
    flags = ["-std=c++20", "-O2", "-ffp-contract=off", "-fPIC", "-Wall", "-Wextra", "-fvisibility=hidden",
             f"-I{INCLUDE}", f"-I{CSRC / 'host'}", f"-I{NLOHMANN}", f"-I{pybind11.get_include()}",
             f"-I{sysconfig.get_paths()['include']}"]
    headers = [d for d in HOST_DEPS if d.suffix == ".hpp"] + [INCLUDE / "smx.h"]

    def compile_one(src: Path) -> Path:
        obj = objdir / (src.stem + ".o")
        if force or _stale(obj, [src, *headers]):
            _run(["g++", *flags, "-c", "-o", obj, src])
        return obj

    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        objs = list(ex.map(compile_one, HOST_SOURCES))
    _run(["g++", "-shared", "-o", out, *objs, f"-L{PKG}", "-lsmx", "-Wl,-rpath,$ORIGIN"])
    return out


def _host_flags():
    import pybind11

    return ["-std=c++20", "-O2", "-ffp-contract=off", "-fPIC", "-Wall", "-Wextra", "-fvisibility=hidden",
            f"-I{INCLUDE}", f"-I{CSRC / 'host'}", f"-I{NLOHMANN}", f"-I{pybind11.get_include()}",
            f"-I{sysconfig.get_paths()['include']}"]


STUB_DIR = ROOT / "tests" / "native"


def build_stub(force: bool = False) -> Path | None:
    """Test-only build: the host library objects + tests/native/smx_stub.cpp (a CPU stand-in for
    every smx_* entry point) as the Python module `_stagemerge_stub`, so the engine's scheduling
    properties are testable without a GPU.  Never imported by the product package."""
    stub = STUB_DIR / "smx_stub.cpp"
    if not stub.exists():
        return None
    out = STUB_DIR / ("_stagemerge_stub" + sysconfig.get_config_var("EXT_SUFFIX"))
    objdir = PKG / "build" / "host"
    objs = [objdir / (s.stem + ".o") for s in HOST_SOURCES if s.stem != "bind"]
    deps = HOST_DEPS + [stub, INCLUDE / "smx.h", *objs]
    if not (force or _stale(out, deps)):
        return out
    flags = _host_flags()
    bind_obj = objdir / "bind_stub.o"
    stub_obj = objdir / "smx_stub.o"
    _run(["g++", *flags, "-DSMH_MODULE=_stagemerge_stub", "-c", "-o", bind_obj, CSRC / "host" / "bind.cpp"])
    _run(["g++", *[f for f in flags if f != "-fvisibility=hidden"], "-c", "-o", stub_obj, stub])
    _run(["g++", "-shared", "-o", out, *objs, bind_obj, stub_obj])
    return out


def build_oracle(force: bool = False) -> None:
    args = ["make", "-C", ROOT / "oracle"]
    if force:
        args.append("-B")
    _run(args)
    if Path("/root/reference/proj/core/src/plan.cpp").exists():
        _run(["make", "-C", ROOT / "oracle", "ref"] + (["-B"] if force else []))


def build_all(force: bool = False) -> None:
    build_smx(force)
    build_host(force)
    build_stub(force)
    build_oracle(force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
