"""Build an experiment variant of the library with extra nvcc defines, into
exp/libhetplan_b200_<tag>.so (exp/ is git-ignored; it travels to the GPU box).
Only the .cu objects are recompiled (into exp/<tag>/); host objects are
shared with the normal build. Load a variant with HP_LIB_PATH=<path>.

  python tools/build_variant.py <tag> -DHP_FOO=1 [-DHP_BAR ...]
"""
from __future__ import annotations

import concurrent.futures as cf
import importlib.util
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def main():
    tag, defs = sys.argv[1], sys.argv[2:]
    spec = importlib.util.spec_from_file_location("b", ROOT / "paper_2403_01136_b200" / "build.py")
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    b.build()  # host objects up to date
    out = ROOT / "exp" / tag
    out.mkdir(parents=True, exist_ok=True)
    cu, cpp = b._sources()

    def comp(src):
        obj = out / (src.stem + ".cu.o")
        cmd = [str(b.CUDA / "bin" / "nvcc"), *b.GENCODE, "-O3", "-lineinfo", "-std=c++17",
               "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr", *defs, *b.INCLUDES, "-c",
               str(src), "-o", str(obj)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            raise RuntimeError(r.stderr)
        return obj

    with cf.ThreadPoolExecutor(8) as ex:
        objs = list(ex.map(comp, cu))
    objs += [b.BUILD / (s.stem + ".o") for s in cpp]
    lib = ROOT / "exp" / f"libhetplan_b200_{tag}.so"
    nccl = b.SITE / "nvidia" / "nccl" / "lib"
    cmd = [str(b.CUDA / "bin" / "nvcc"), *b.GENCODE, "-shared", "-o", str(lib), *map(str, objs),
           f"-L{b.CUDA / 'lib64'}", "-lcudart", f"-L{nccl}", "-l:libnccl.so.2",
           "-Xlinker", f"-rpath,{b.CUDA / 'lib64'}", "-Xlinker", f"-rpath,{nccl}"]
    subprocess.run(cmd, check=True)
    print(lib)


if __name__ == "__main__":
    main()
