"""f2: the tuner's ground-truth Evaluator on the device executor
(a3gnn_b200.hpp make_device_evaluator; surrogate.hpp:19,79-88,
tuner.cpp:29-120). The reference's own PPO tuner stays host-side and drives
it; the knobs are mapped onto cache ratio, fanout level and pipeline depth.

* on the same design points (fanout level 0 = the reference's fanouts) the
  device evaluator's memory estimate equals the reference executor's
  (same batches, same analytic model) and its accuracy is within 3 test
  nodes (fp32 device vs fp64);
* the knob mapping resolves as documented;
* tuner::tune completes within its budget on device evaluations.
"""
import os
import re
import subprocess

import pytest

from paper_2511_07421_b200 import build as B

REF = os.path.join(B.DROPIN_OUT, "tuner_check")
DEV = os.path.join(B.DROPIN_OUT, "tuner_check_b200")
N = 20000
NTEST = int(0.4 * N)

needs_build = pytest.mark.skipif(not (os.path.exists(REF) and os.path.exists(DEV)),
                                 reason="tuner check not built (needs the reference headers at build time)")


def run(exe):
    r = subprocess.run([exe, str(N)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    return r.stdout.strip().splitlines()


def _num(line, key):
    return float(re.search(rf"{key} ([0-9.e+-]+)", line).group(1))


@needs_build
def test_reference_evaluator_runs_on_cpu():
    lines = run(REF)
    assert sum(l.startswith("point") for l in lines) == 4


@needs_build
@pytest.mark.gpu
def test_device_evaluator_matches_reference_and_drives_the_tuner():
    ref, dev = run(REF), run(DEV)
    pts = [l for l in dev if l.startswith("point")]
    assert len(pts) == 4
    for a, b in zip(ref, pts):
        assert _num(a, "mem") == _num(b, "mem"), (a, b)
        assert abs(_num(a, "accuracy") - _num(b, "accuracy")) <= 3.0 / NTEST, (a, b)
        assert _num(b, "thr_positive") == 1
    m = next(l for l in dev if l.startswith("mapping"))
    assert "fanouts 15,10" in m and "streams 4" in m and "ratio 0.200" in m and "partitions 1" in m
    t = next(l for l in dev if l.startswith("tune"))
    assert 1 <= _num(t, "evaluations") <= 8 and _num(t, "feasible") == 1
