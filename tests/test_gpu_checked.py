"""Race / synchronisation checks of the pipelined sweeps without compute-sanitizer (closed on the
GPU pool): the verification build libsgm_checked.so (csrc/check.cuh) checks the producer/consumer
hand-off (stage tags, release counts), the SPIKE tail/head exchanges (exchange tags), poisons every
slab before it is refilled and sleeps at random at every hand-off.  Over a matrix of launch
configurations (scripts/checked_cases.py) it must report no violation, give bit-identical results
from run to run under the random delays, and agree bit for bit with the product library.  Two
injected faults (a premature slab release, a skipped exchange barrier) must be caught -- so the
checks are shown to fire, not just to stay quiet."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCRIPT = os.path.join(ROOT, "scripts", "checked_cases.py")

pytestmark = pytest.mark.gpu


def _run(out, variant, reps=1, cases="", inject=0):
    env = dict(os.environ)
    env.pop("SGM_LIB_VARIANT", None)
    env.pop("SGM_CHECK_INJECT", None)
    if variant == "checked":
        env["SGM_LIB_VARIANT"] = "checked"
    if inject:
        env["SGM_CHECK_INJECT"] = str(inject)
    cmd = [sys.executable, SCRIPT, str(out), "--reps", str(reps)] + (["--cases", cases] if cases else [])
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1]), np.load(out)


@pytest.fixture(scope="module")
def product(tmp_path_factory):
    from paper_2302_04979_b200 import build
    build.build(checked=True)
    return _run(tmp_path_factory.mktemp("prod") / "prod.npz", "product")


def test_checked_build_clean_and_bitwise_equal(product, tmp_path):
    summ_p, res_p = product
    summ, res = _run(tmp_path / "chk.npz", "checked", reps=3)
    assert summ["variant"] == "checked" and "checked" in summ["version"]
    assert summ_p["variant"] == "product" and "checked" not in summ_p["version"]
    for name, c in summ["cases"].items():
        assert c["violations"] == 0, (name, c)
        assert c["reps_identical"], name  # random delays do not change a bit
        assert c["finite"], name
        # same arithmetic: the poisoned, delayed run reproduces the product library exactly
        assert np.array_equal(res[name], res_p[name]), name


@pytest.mark.parametrize("inject", [1, 2])
def test_checked_build_detects_injected_faults(product, tmp_path, inject):
    # 1: consumers release a slab before reading it (WAR race with the producer's next fill);
    # 2: consumers skip the barrier in front of the SPIKE history scan (RAW race on the tails)
    summ_p, res_p = product
    cases = "p3_128,p2_long_x,p3_exact_spike"
    summ, res = _run(tmp_path / "inj.npz", "checked", cases=cases, inject=inject)
    caught = 0
    for name, c in summ["cases"].items():
        wrong = not np.array_equal(res[name], res_p[name])
        caught += (c["violations"] > 0) or wrong
    assert caught >= 1, summ
