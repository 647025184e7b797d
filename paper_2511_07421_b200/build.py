"""In-tree build of the sm_100a C-ABI library ``liba3g_b200.so``.

nvcc -gencode arch=compute_100a,code=sm_100a (explicit gencode: plain
-arch=sm_100a would also embed compute_100 PTX). Objects go to build/,
the shared library next to this file so it travels with the repo snapshot.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys
import sysconfig

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build", "a3g_b200")
LIB = os.path.join(PKG, "liba3g_b200.so")


def nvcc() -> str:
    for c in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


GENCODE = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off",
          "-I", os.path.join(ROOT, "include"), "-I", CSRC, "--expt-relaxed-constexpr"]


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def _headers():
    return glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(ROOT, "include", "*.h"))


def _compile(src: str, verbose: bool) -> str:
    obj = os.path.join(BUILD, os.path.basename(src) + ".o")
    newest_dep = max([os.path.getmtime(src)] + [os.path.getmtime(h) for h in _headers()])
    if os.path.exists(obj) and os.path.getmtime(obj) >= newest_dep:
        return obj
    cmd = [nvcc()] + GENCODE + COMMON + ["-c", src, "-o", obj]
    if src.endswith(".cu"):
        cmd += ["-Xptxas", "-v"] if verbose else []
    else:
        cmd = [nvcc()] + GENCODE + COMMON + ["-x", "c++", "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"nvcc failed on {os.path.basename(src)}")
    if verbose and r.stderr:
        sys.stderr.write(r.stderr)
    return obj


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    if force:
        for o in glob.glob(os.path.join(BUILD, "*.o")):
            os.remove(o)
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), _sources()))
    if os.path.exists(LIB) and os.path.getmtime(LIB) >= max(os.path.getmtime(o) for o in objs):
        return LIB
    cmd = [nvcc()] + GENCODE + ["-shared", "-o", LIB] + objs + ["-ldl", "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link of liba3g_b200.so failed")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))


# ---------------------------------------------------------------- drop-in ----
# The C++ drop-in (dropin/*.cpp) implements the reference's own declarations
# (proj/include/a3gnn) over the C-ABI, so it compiles against the reference's
# headers; built where /root/reference exists (this container), the outputs
# travel to the GPU box with the repo snapshot.
REF_INCLUDE = "/root/reference/proj/include"
DROPIN = os.path.join(PKG, "dropin")
DROPIN_OUT = os.path.join(DROPIN, "_build")
DROPIN_LIBS = {
    # sampler + cache hot functions only: the reference's train()/executor run on them
    "liba3gnn_b200_sampling.so": ["registry.cpp", "sampler_b200.cpp", "cache_b200.cpp"],
    # + the trainer (forward / backward / grad_on_batch / sgd_step /
    # sync_gradients / train / evaluate_full_graph) and the executor
    # (execute_pipeline / profile_stage_costs) on the device
    "liba3gnn_b200.so": ["registry.cpp", "sampler_b200.cpp", "cache_b200.cpp", "trainer_b200.cpp",
                         "pipeline_b200.cpp", "evaluator_b200.cpp"],
}


def build_dropin(ref_lib_dir: str | None = None, force: bool = False) -> list:
    """g++ the drop-in libraries (and, given the compiled reference's
    directory, the dropin_check test driver). Returns the outputs built."""
    if not os.path.isdir(REF_INCLUDE):
        return []
    os.makedirs(DROPIN_OUT, exist_ok=True)
    cxx = shutil.which("g++") or "g++"
    common = ["-std=c++20", "-O2", "-fPIC", "-Wall", "-Wextra", "-I", REF_INCLUDE, "-I", os.path.join(ROOT, "include"),
              "-I", DROPIN]
    srcs_all = glob.glob(os.path.join(DROPIN, "*.cpp")) + glob.glob(os.path.join(DROPIN, "*.hpp"))
    newest = max([os.path.getmtime(p) for p in srcs_all] + [os.path.getmtime(LIB)])
    built = []
    for name, srcs in DROPIN_LIBS.items():
        out = os.path.join(DROPIN_OUT, name)
        if not force and os.path.exists(out) and os.path.getmtime(out) >= newest:
            continue
        cmd = [cxx] + common + ["-shared", "-o", out] + [os.path.join(DROPIN, s) for s in srcs] + [
            "-L", PKG, "-la3g_b200", "-Wl,-rpath,$ORIGIN/../.."]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"drop-in build failed: {name}")
        built.append(out)
    if ref_lib_dir and os.path.exists(os.path.join(ref_lib_dir, "libref_a3gnn.so")):
        out = os.path.join(DROPIN_OUT, "dropin_check")
        if force or not os.path.exists(out) or os.path.getmtime(out) < newest:
            rel = os.path.relpath(ref_lib_dir, DROPIN_OUT)
            cmd = [cxx, "-std=c++20", "-O2", "-I", REF_INCLUDE, "-o", out, os.path.join(DROPIN, "dropin_check.cpp"),
                   "-L", ref_lib_dir, "-lref_a3gnn", f"-Wl,-rpath,$ORIGIN/{rel}", "-lpthread"]
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError("dropin_check build failed")
            built.append(out)
        # the device Evaluator's check: reference alone / linked with the drop-in
        nj = os.path.join(sysconfig.get_paths()["purelib"], "include", "cudnn_frontend", "thirdparty")
        for name, extra in (("tuner_check", []),
                            ("tuner_check_b200", ["-DA3G_DEVICE_EVAL", "-I", DROPIN, "-L", DROPIN_OUT, "-la3gnn_b200",
                                                  "-Wl,-rpath,$ORIGIN"])):
            out = os.path.join(DROPIN_OUT, name)
            if not force and os.path.exists(out) and os.path.getmtime(out) >= newest:
                continue
            rel = os.path.relpath(ref_lib_dir, DROPIN_OUT)
            cmd = [cxx, "-std=c++20", "-O2", "-I", REF_INCLUDE, "-I", nj, "-o", out,
                   os.path.join(DROPIN, "tuner_check.cpp")] + extra + [
                "-L", ref_lib_dir, "-lref_a3gnn", f"-Wl,-rpath,$ORIGIN/{rel}", "-lpthread"]
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError(f"{name} build failed")
            built.append(out)
    return built
