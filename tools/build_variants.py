"""Build A/B variants of libliftcut_b200.so that differ in one translation unit's -D flags.

    python tools/build_variants.py lcb_stream.cu name1:DEF=1,DEF2=3 name2:DEF=2 ...

Objects of the other sources are compiled once; each variant recompiles the named
source with its defines and links build_variants/<name>.so.  Run a variant on the GPU
with LCB_LIB_PATH=build_variants/<name>.so.
"""
import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2509_18612_b200", "csrc")
OUT = os.path.join(ROOT, "build_variants")
FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
         "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC,-O2,-ffp-contract=off", "-I", os.path.join(ROOT, "include")]


def obj(src, defs, tag):
    o = os.path.join(OUT, "obj", f"{os.path.basename(src)}.{tag}.o")
    cmd = ["nvcc", *FLAGS, *[f"-D{d}" for d in defs], "-c", src, "-o", o]
    subprocess.run(cmd, check=True)
    return o


def main():
    target = sys.argv[1]
    variants = [(a.split(":")[0], [d for d in a.split(":")[1].split(",") if d] if ":" in a else [])
                for a in sys.argv[2:]]
    os.makedirs(os.path.join(OUT, "obj"), exist_ok=True)
    others = [s for s in sorted(glob.glob(os.path.join(CSRC, "*.cu"))) if os.path.basename(s) != target]
    with ThreadPoolExecutor(8) as ex:
        base = list(ex.map(lambda s: obj(s, [], "base"), others))
        vobjs = list(ex.map(lambda v: obj(os.path.join(CSRC, target), v[1], v[0]), variants))
    for (name, _), vo in zip(variants, vobjs):
        so = os.path.join(OUT, f"{name}.so")
        subprocess.run(["nvcc", "-shared", *FLAGS[2:4], "-o", so, *base, vo, "-ldl"], check=True)
        print(so)


if __name__ == "__main__":
    main()
