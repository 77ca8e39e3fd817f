"""In-tree build of the engine's shared library (libplnmf_gpu.so).

Every CUDA source is compiled for sm_100a only
(``-gencode arch=compute_100a,code=sm_100a``) with ``-lineinfo`` so ncu's
source page maps to the kernels; host C++ is compiled without FMA contraction
(``-ffp-contract=off``) so the host-side arithmetic that must be bit-identical
to the reference (init_factors, ||A||^2) stays so.  Objects go to
``build/``; the .so lands next to this file (git-ignored, shipped to the GPU
box by gpurun).
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
BUILD = ROOT / "build" / "plnmf_gpu"
LIB = PKG / "libplnmf_gpu.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + [
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off",
    "-Xptxas", "-v", "--expt-relaxed-constexpr", f"-I{ROOT / 'include'}", f"-I{CSRC}",
]
# developer experiments only (e.g. -DPLNMF_CHAIN_ONLY); never set for a real build
NVCC_FLAGS += os.environ.get("PLNMF_NVCC_EXTRA", "").split()
HOST_FLAGS = ["-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", "-Wall", "-Wextra",
              f"-I{ROOT / 'include'}", f"-I{CSRC}", "-I/usr/local/cuda/include"]


def _nvcc() -> str:
    for cand in ("/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _cxx() -> str:
    # The image's $CXX wrapper lacks some spec files; plain g++ is fine here.
    for cand in ("/usr/bin/g++", shutil.which("g++")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("g++ not found")


def _compile(src: Path) -> tuple[Path, str]:
    obj = BUILD / (src.name + ".o")
    if src.suffix == ".cu":
        cmd = [_nvcc(), *NVCC_FLAGS, "-c", str(src), "-o", str(obj)]
    else:
        cmd = [_cxx(), *HOST_FLAGS, "-c", str(src), "-o", str(obj)]
    deps = [src, *CSRC.glob("*.cuh"), *CSRC.glob("*.hpp"), ROOT / "include" / "plnmf_gpu.h"]
    # the compile command is part of the object's identity (e.g. PLNMF_NVCC_EXTRA experiments)
    stamp = obj.with_suffix(obj.suffix + ".cmd")
    same_cmd = stamp.exists() and stamp.read_text() == " ".join(cmd)
    if same_cmd and obj.exists() and all(obj.stat().st_mtime >= d.stat().st_mtime for d in deps):
        return obj, ""
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
    stamp.write_text(" ".join(cmd))
    return obj, res.stderr


def build(verbose: bool = False) -> Path:
    BUILD.mkdir(parents=True, exist_ok=True)
    srcs = sorted([*CSRC.glob("*.cu"), *CSRC.glob("*.cpp")])
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        results = list(ex.map(_compile, srcs))
    log = "\n".join(r[1] for r in results if r[1])
    (BUILD / "ptxas.log").write_text(log)
    if verbose and log:
        print(log)
    objs = [str(r[0]) for r in results]
    newest = max(Path(o).stat().st_mtime for o in objs)
    if not LIB.exists() or LIB.stat().st_mtime < newest:
        cmd = [_nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", str(LIB), *objs,
               "-Xlinker", "--no-undefined", "-lpthread", "-ldl", "-lrt"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
    build_cli()
    return LIB


CLI = PKG / "plnmf-gpu"


def build_cli() -> Path:
    """The C++ command-line front end (csrc/cli/plnmf_gpu.cpp), linked against the
    engine library through the C-ABI only (rpath: the package directory)."""
    src = CSRC / "cli" / "plnmf_gpu.cpp"
    deps = [src, ROOT / "include" / "plnmf_gpu.h", LIB]
    if CLI.exists() and all(CLI.stat().st_mtime >= d.stat().st_mtime for d in deps):
        return CLI
    cmd = [_cxx(), "-O2", "-std=c++17", "-Wall", "-Wextra", f"-I{ROOT / 'include'}", str(src), "-o", str(CLI),
           f"-L{PKG}", "-l:libplnmf_gpu.so", "-Wl,-rpath,$ORIGIN"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"CLI build failed: {' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
    return CLI


def build_oracle() -> None:
    """Builds oracle/ (the C restatement; and the reference itself when
    /root/reference is present).  Test infrastructure, not the product."""
    env = dict(os.environ)
    env["CC"] = "/usr/bin/gcc" if os.path.exists("/usr/bin/gcc") else "gcc"
    env["CXX"] = _cxx()
    res = subprocess.run(["make", "-C", str(ROOT / "oracle"), "-j8"], capture_output=True, text=True, env=env)
    if res.returncode != 0:
        raise RuntimeError(f"oracle build failed\n{res.stdout}\n{res.stderr}")


if __name__ == "__main__":
    build(verbose="-v" in sys.argv)
    build_oracle()
    print(LIB)
