"""CPU tests of the product's host side and the C-ABI library (no GPU calls):
generator / plan / seeds / init_model / A3G1 bit-exact vs the reference's
golden vectors; every symbol declared in include/a3g.h is exported."""
import os
import re
import subprocess
import sys

import numpy as np
import pytest

from helpers import load_golden
from paper_2511_07421_b200 import _lib, graph as G, train as T

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("name", ["pl500", "pl3000"])
def test_generator_bit_exact(name):
    rec = load_golden(name)
    n, m, F, seed = (int(x) for x in rec["gen"])
    for threads in (1, 4):
        g = G.generate_power_law(n, m, 2.5, F, seed, threads=threads)
        for k in ("row_offsets", "col_indices", "features", "labels", "train_mask", "test_mask"):
            assert np.array_equal(getattr(g, k), rec[k]), k


@pytest.mark.parametrize("name", ["pl500", "pl3000"])
def test_plan_seed_init(name):
    rec = load_golden(name)
    tn = np.flatnonzero(rec["train_mask"]).astype(np.uint32)
    assert np.array_equal(T.plan_epoch_order(tn, 3, 99), rec["plan_e3"])
    got = [T.sampling_seed(1, e, s, 0) for e in range(3) for s in range(4)]
    assert np.array_equal(np.array(got, dtype=np.uint64), rec["sampling_seeds"])
    w1, w2 = T.init_model(T.ModelSpec(rec["features"].shape[1], 8, 4), 1)
    assert np.array_equal(w1, rec["init_w1"]) and np.array_equal(w2, rec["init_w2"])


def test_init_model_errors():
    with pytest.raises(_lib.ParameterError):
        T.init_model(T.ModelSpec(0, 8, 4), 1)


def test_a3g1_roundtrip(tmp_path):
    g = G.generate_power_law(700, 2, 2.5, 5, 9)
    p = str(tmp_path / "g.a3g")
    G.save_graph(g, p)
    h = G.load_graph(p)
    for k in ("row_offsets", "col_indices", "features", "labels", "train_mask", "test_mask"):
        assert np.array_equal(getattr(g, k), getattr(h, k))
    with open(p, "r+b") as f:
        f.write(b"XXXX")
    with pytest.raises(_lib.IoError):
        G.load_graph(p)
    with pytest.raises(_lib.IoError):
        G.load_graph(str(tmp_path / "missing.a3g"))


def test_from_edges_sorted():
    g = G.from_edges(5, [(1, 2), (0, 3), (1, 0), (4, 4)], 2)
    assert g.row_offsets.tolist() == [0, 1, 3, 3, 3, 4]
    assert g.col_indices.tolist() == [3, 0, 2, 4]
    with pytest.raises(_lib.ParameterError):
        G.from_edges(3, [(0, 5)], 2)
    G.validate(g)


def test_generator_errors():
    for args in [(10, 2, 1.0, 4, 1), (10, 0, 2.5, 4, 1), (10, 2, 2.5, 0, 1), (1, 2, 2.5, 4, 1)]:
        with pytest.raises(_lib.ParameterError):
            G.generate_power_law(*args)


def _declared():
    src = open(os.path.join(ROOT, "include", "a3g.h")).read()
    return sorted(set(re.findall(r"\b(a3g_[a-z0-9_]+)\s*\(", src)))


def test_abi_exports_every_declared_symbol():
    L = _lib.lib()
    declared = _declared()
    assert len(declared) >= 35
    for name in declared:
        assert hasattr(L, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (a3g_\w+)", out))
    assert set(declared) <= exported
    # the python binding covers the whole header
    assert set(declared) <= set(_lib.exported_symbols())


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_string():
    assert b"sm_100a" in _lib.lib().a3g_version()


def test_library_requests_hardware_queues():
    """Loading the library asks for 32 CUDA hardware work queues (the pipeline's nine streams)
    unless the process preset the variable: checked in a fresh process, through libc."""
    code = ("import ctypes, os\n"
            "os.environ.pop('CUDA_DEVICE_MAX_CONNECTIONS', None)\n"
            "libc = ctypes.CDLL(None); libc.unsetenv(b'CUDA_DEVICE_MAX_CONNECTIONS')\n"
            "libc.getenv.restype = ctypes.c_char_p\n"
            "ctypes.CDLL(%r)\n"
            "print(libc.getenv(b'CUDA_DEVICE_MAX_CONNECTIONS').decode())\n") % _lib.LIB_PATH
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr[-1000:]
    assert out.stdout.strip() == "32"


@pytest.mark.parametrize("name", ["c1", "c2", "c3"])
def test_generator_matches_reference_at_baseline_scale(name):
    """The multithreaded host generator reproduces the REFERENCE generator's
    graphs bit for bit at the BASELINE scales (C2: 112.8M edges x 602-d
    features; C3: 2.45M nodes): sha256 of every array vs the fingerprints the
    compiled reference wrote (tests/golden/make_generator_hashes.py)."""
    import hashlib
    import json
    rec = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                                      "generator_hashes.json")))[name]
    n, m, F, seed = rec["gen"]
    g = G.generate_power_law(n, m, 2.5, F, seed)
    assert g.num_edges == rec["num_edges"]
    for arr in ("row_offsets", "col_indices", "features", "labels", "train_mask", "test_mask"):
        assert hashlib.sha256(memoryview(np.ascontiguousarray(getattr(g, arr))).cast("B")).hexdigest() == rec[arr], arr
