"""In-tree build of the native libraries (sm_100a only).

librbg.so            -- CUDA kernels + the C ABI (include/rbg.h), nvcc
librbfit_b200.so     -- C++ host layer mirroring the reference API, g++, links librbg.so
librbg_datagen.so    -- host fixture generators (seeded configs), g++ -fopenmp

Built objects stay inside the package directory so they travel with the repo
snapshot to the GPU box; nothing is pip-installed.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = PKG / "_obj"

CUDA_HOME = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))
NVCC = str(CUDA_HOME / "bin" / "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                     "-Xcompiler", "-ffp-contract=off", "--expt-relaxed-constexpr",
                     f"-I{ROOT / 'include'}"] + os.environ.get("RBG_NVCC_EXTRA", "").split()
# the assembly kernels are split one translation unit per (dimension, family) so they compile in parallel
CU_SOURCES = (["rbg_util.cu", "rbg_setup.cu", "rbg_layout.cu", "rbg_assemble.cu", "rbg_solve.cu",
               "rbg_eval.cu", "rbg_api.cu", "rbg_diag.cu", "rbg_repass.cu", "rbg_band.cu"]
              + [f"rbg_asm_part_{d}_{f}.cu" for d in (2, 3) for f in range(4)])

LIB_RBG = PKG / "librbg.so"
LIB_HOST = PKG / "librbfit_b200.so"
LIB_DATAGEN = PKG / "librbg_datagen.so"
CLI = PKG / "rbfit-b200"


def _run(cmd: list[str]) -> None:
    proc = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
    if proc.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{proc.stdout}")
    if os.environ.get("RBG_BUILD_VERBOSE"):
        sys.stdout.write(proc.stdout)


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build_rbg(force: bool = False, ptxas_verbose: bool = False) -> Path:
    OBJ.mkdir(exist_ok=True)
    headers = list(CSRC.glob("*.cuh")) + [ROOT / "include" / "rbg.h"]
    jobs = []
    for src in CU_SOURCES:
        s = CSRC / src
        o = OBJ / (s.stem + ".o")
        if force or _stale(o, [s] + headers):
            extra = ["-Xptxas", "-v"] if ptxas_verbose else []
            jobs.append([NVCC, *NVCC_FLAGS, *extra, "-c", str(s), "-o", str(o)])
    with cf.ThreadPoolExecutor(max_workers=max(4, os.cpu_count() or 4)) as ex:
        list(ex.map(_run, jobs))
    objs = [OBJ / (Path(s).stem + ".o") for s in CU_SOURCES]
    if force or jobs or _stale(LIB_RBG, objs):
        _run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", str(LIB_RBG), *map(str, objs)])
    return LIB_RBG


def build_host(force: bool = False) -> Path:
    srcs = [CSRC / "rbfit_gpu.cpp", CSRC / "rbfit_io.cpp"]
    deps = srcs + [CSRC / "rbfit_gpu.hpp", ROOT / "include" / "rbg.h", LIB_RBG]
    if force or _stale(LIB_HOST, deps):
        _run(["g++", "-std=c++20", "-O2", "-fPIC", "-shared", f"-I{ROOT / 'include'}",
              "-o", str(LIB_HOST), *map(str, srcs), f"-L{PKG}", "-lrbg",
              "-Wl,-rpath,$ORIGIN"])
    return LIB_HOST


def build_datagen(force: bool = False) -> Path:
    src = CSRC / "datagen.cpp"
    if force or _stale(LIB_DATAGEN, [src]):
        _run(["g++", "-std=c++20", "-O2", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off",
              "-o", str(LIB_DATAGEN), str(src)])
    return LIB_DATAGEN


def build_cli(force: bool = False) -> Path:
    """rbfit-b200: the reference's gen-synthetic / fit / eval / bench-blocks front end."""
    src = CSRC / "rbfit_b200_main.cpp"
    deps = [src, CSRC / "rbfit_gpu.hpp", LIB_HOST, LIB_DATAGEN]
    if force or _stale(CLI, deps):
        _run(["g++", "-std=c++20", "-O2", f"-I{ROOT / 'include'}", "-o", str(CLI), str(src), f"-L{PKG}",
              "-lrbfit_b200", "-lrbg", "-lrbg_datagen", "-Wl,-rpath,$ORIGIN"])
    return CLI


def build_oracle(force: bool = False) -> None:
    """CPU checkers (test infrastructure): our C restatement always; the
    reference's own sources only where /root/reference exists."""
    args = ["make", "-s", "-C", str(ROOT / "oracle"), "oracle"]
    if Path("/root/reference/proj/core/src/coo.cpp").exists():
        args.append("ref")
    if force:
        args.insert(1, "-B")
    _run(args)


def build_all(force: bool = False) -> None:
    if shutil.which(NVCC) is None and not Path(NVCC).exists():
        raise RuntimeError(f"nvcc not found at {NVCC}")
    build_rbg(force)
    build_host(force)
    build_datagen(force)
    build_cli(force)
    build_oracle(force)


if __name__ == "__main__":
    if "--check" in sys.argv:  # device bounds checks (debugging only)
        NVCC_FLAGS.append("-DRBG_DEVCHECK")
    build_all(force="--force" in sys.argv or "--check" in sys.argv)
    print("built:", LIB_RBG, LIB_HOST, LIB_DATAGEN)
