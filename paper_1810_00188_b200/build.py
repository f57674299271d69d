"""In-tree build of the B200 extension (no JIT cache, no pip install).

Produces, next to this file:
  libermc_b200.so   C-ABI (include/ermc_b200.h) + C++ API + sm_100a kernels
  _ermc<EXT>        pybind11 drop-in for the reference's _ermc module
and, under oracle/, the test-only checkers (see oracle/Makefile).

Kernels are compiled for sm_100a only (-gencode arch=compute_100a,code=sm_100a).
trace_fp64.cu is compiled with --fmad=false and IEEE div/sqrt so its
arithmetic rounds like the reference's x86-64 build.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
import sysconfig
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
INCLUDE = ROOT / "include"
OBJ = PKG / "build"
LIB = PKG / "libermc_b200.so"
EXT = sysconfig.get_config_var("EXT_SUFFIX") or ".so"
PYMOD = PKG / f"_ermc{EXT}"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
CXX = shutil.which("g++") or "g++"

# (source, extra flags)
CUDA_SOURCES = [
    ("trace_fp64.cu", ["--fmad=false", "-prec-div=true", "-prec-sqrt=true", "-ftz=false"]),
    ("trace_fp32.cu", []),
    ("dispatch.cu", []),
    ("capi.cu", []),
    ("probe.cu", []),
]
HOST_SOURCES = ["host_tables.cpp", "host_api.cpp", "host_io.cpp"]


def _deps() -> list[Path]:
    return [p for p in list(CSRC.iterdir()) + list(INCLUDE.iterdir())
            if p.suffix in {".cu", ".cuh", ".cpp", ".hpp", ".h"}]


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def _run(cmd: list[str], verbose: bool) -> None:
    if verbose:
        print("+", " ".join(cmd), flush=True)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"build step failed: {cmd[0]} ... {cmd[-1]}")
    if verbose and res.stderr.strip():
        sys.stderr.write(res.stderr)


def build_lib(force: bool = False, verbose: bool = True) -> Path:
    deps = _deps()
    if not force and not _stale(LIB, deps):
        return LIB
    OBJ.mkdir(exist_ok=True)
    jobs = []
    exp_flags = os.environ.get("ERMC_NVCC_FLAGS", "").split()  # A/B experiments only
    for src, extra in CUDA_SOURCES:
        obj = OBJ / (src + ".o")
        jobs.append([NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", *exp_flags,
                     "-Xcompiler", "-fPIC", "-Xptxas", "-v", *extra,
                     f"-I{INCLUDE}", f"-I{CSRC}", "-c", str(CSRC / src),
                     "-o", str(obj)])
    for src in HOST_SOURCES:
        obj = OBJ / (src + ".o")
        # No -march: baseline x86-64 has no FMA, so no contraction can change
        # the reference's rounding; -ffp-contract=off makes that explicit.
        jobs.append([CXX, "-std=c++20", "-O3", "-fPIC", "-ffp-contract=off",
                     f"-I{INCLUDE}", f"-I{CSRC}", "-c", str(CSRC / src),
                     "-o", str(obj)])
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 2)) as ex:
        list(ex.map(lambda c: _run(c, verbose), jobs))
    objs = [str(OBJ / (s + ".o")) for s, _ in CUDA_SOURCES] + \
           [str(OBJ / (s + ".o")) for s in HOST_SOURCES]
    _run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", str(LIB), *objs,
          "-Xlinker", "--no-undefined", "-lpthread", "-ldl", "-lrt"], verbose)
    return LIB


def build_pymod(force: bool = False, verbose: bool = True) -> Path:
    deps = _deps() + [LIB]
    if not force and not _stale(PYMOD, deps):
        return PYMOD
    import pybind11  # noqa: PLC0415

    pyinc = sysconfig.get_paths()["include"]
    _run([CXX, "-std=c++20", "-O2", "-fPIC", "-shared", "-fvisibility=hidden",
          f"-I{INCLUDE}", f"-I{pyinc}", f"-I{pybind11.get_include()}",
          str(CSRC / "pybind_ermc.cpp"), "-o", str(PYMOD),
          f"-L{PKG}", "-lermc_b200", "-Wl,-rpath,$ORIGIN"], verbose)
    return PYMOD


def build_oracle(verbose: bool = True) -> None:
    """Test-only checkers: the C restatement always; the reference library
    (oracle/_ref) and the reference's unit tests built against this library
    (tests/_refcompat) only where /root/reference exists (this container)."""
    oracle = ROOT / "oracle"
    _run(["make", "-C", str(oracle), "oracle"], verbose)
    if Path("/root/reference/proj/src").is_dir():
        _run(["make", "-C", str(oracle), "-j8", "ref"], verbose)
        # the reference's own unit tests compiled against the drop-in API
        _run(["bash", str(ROOT / "tests" / "refcompat" / "build.sh")], verbose)


def build(force: bool = False, verbose: bool = True) -> None:
    build_lib(force, verbose)
    build_pymod(force, verbose)


if __name__ == "__main__":
    force = "--force" in sys.argv
    build(force=force)
    if "--no-oracle" not in sys.argv:
        build_oracle()
