"""Build the B200 library in-tree: libhetplan_b200.so (C++ host library +
sm_100a kernels + C-ABI). nvcc for .cu (compute_100a/sm_100a, -lineinfo),
g++ for host .cpp, parallel, mtime-incremental. No torch extension, no JIT
cache: the .so lives next to this file and travels with the repo snapshot.
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
BUILD = PKG / "_build"
LIB = PKG / "libhetplan_b200.so"
SITE = Path(sys.prefix) / "lib" / f"python{sys.version_info.major}.{sys.version_info.minor}" / "site-packages"
JSON_DIR = SITE / "include" / "cudnn_frontend" / "thirdparty" / "nlohmann"
NCCL_INC = SITE / "nvidia" / "nccl" / "include"
CUDA = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))
GENCODE = ["-gencode", "arch=compute_100a,code=sm_100a"]
INCLUDES = [f"-I{ROOT / 'include'}", f"-I{CSRC}", f"-I{JSON_DIR}", f"-I{CUDA / 'include'}"]


def _sources():
    cu = sorted(CSRC.glob("*.cu"))
    cpp = sorted((CSRC / "host").glob("*.cpp"))
    return cu, cpp


def _deps_mtime():
    files = list(CSRC.rglob("*.cu*")) + list(CSRC.rglob("*.h*")) + list((ROOT / "include").rglob("*.h*"))
    return max(f.stat().st_mtime for f in files)


def _compile(src: Path, verbose: bool) -> Path:
    obj = BUILD / (src.stem + (".cu.o" if src.suffix == ".cu" else ".o"))
    if obj.exists() and obj.stat().st_mtime >= max(src.stat().st_mtime, _deps_mtime()):
        return obj
    if src.suffix == ".cu":
        cmd = [str(CUDA / "bin" / "nvcc"), *GENCODE, "-O3", "-lineinfo", "-std=c++17",
               "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr", "-Xptxas", "-v", *os.environ.get("HP_NVCC_EXTRA", "").split(),
               *INCLUDES, "-c", str(src), "-o", str(obj)]
    else:
        cmd = ["g++", "-std=c++20", "-O2", "-fPIC", "-Wall", "-Wno-unused-function",
               *INCLUDES, f"-I{NCCL_INC}", "-c", str(src), "-o", str(obj)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {src.name}\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    if verbose and src.suffix == ".cu":
        (BUILD / (src.stem + ".ptxas.txt")).write_text(r.stderr)
    return obj


def build(verbose: bool = False, force: bool = False) -> Path:
    if shutil.which(str(CUDA / "bin" / "nvcc")) is None:
        raise RuntimeError("nvcc not found")
    BUILD.mkdir(exist_ok=True)
    if force:
        for f in BUILD.glob("*.o"):
            f.unlink()
    cu, cpp = _sources()
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        objs = list(ex.map(lambda s: _compile(s, True), cu + cpp))
    if LIB.exists() and LIB.stat().st_mtime >= max(o.stat().st_mtime for o in objs):
        return LIB
    nccl_lib = SITE / "nvidia" / "nccl" / "lib"
    cmd = [str(CUDA / "bin" / "nvcc"), *GENCODE, "-shared", "-o", str(LIB), *map(str, objs),
           f"-L{CUDA / 'lib64'}", "-lcudart", f"-L{nccl_lib}", "-l:libnccl.so.2",
           "-Xlinker", f"-rpath,{CUDA / 'lib64'}", "-Xlinker", f"-rpath,{nccl_lib}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(verbose=True, force="--force" in sys.argv))
