"""Build an A/B variant of liba3g_b200.so with extra nvcc defines into
ab_variants/<name>/liba3g_b200.so (select it with A3G_LIB=<path>).
    python tools/build_variant.py lane_minb3 -DA3G_LANE_MINB=3
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_07421_b200 import build as B  # noqa: E402


def main():
    name, defs = sys.argv[1], sys.argv[2:]
    out = os.path.join(ROOT, "ab_variants", name)  # git-ignored, travels with gpurun
    os.makedirs(out, exist_ok=True)
    objs = []
    for src in B._sources():
        obj = os.path.join(out, os.path.basename(src) + ".o")
        cmd = [B.nvcc()] + B.GENCODE + B.COMMON + defs
        cmd += (["-c", src] if src.endswith(".cu") else ["-x", "c++", "-c", src]) + ["-o", obj]
        objs.append((cmd, obj))
    procs = [subprocess.Popen(c) for c, _ in objs]
    if any(p.wait() for p in procs):
        sys.exit("variant build failed")
    lib = os.path.join(out, "liba3g_b200.so")
    subprocess.run([B.nvcc()] + B.GENCODE + ["-shared", "-o", lib] + [o for _, o in objs] + ["-ldl", "-lpthread"],
                   check=True)
    print(lib)


if __name__ == "__main__":
    main()
