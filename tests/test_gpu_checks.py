"""Device bounds checks.  compute-sanitizer is closed on the GPU pool
(runs under it left GPUs needing a reset), so the library has a diagnostic build,
libsim_checked.so (-DECO_CHECKS=1), whose kernels assert every cell, slot, list position
and outbox index they compute.  A fresh process runs it over 50 steps of: the tiny world
and a 64x64 world through the graph path and through the instrumented path (every phase
a separate kernel), the paper-scale network on a small grid (split policy, k_post with P
warps), a 3-world batch, a 20-world Hd = 32 batch (the compacted policy tiles, the single mutation
sequence), the paper's CNN-LSTM world (network 1) and a 4-band banded world; any failed assert aborts the process.
The same runs with the product build must give the same step records (the checks change
no result)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import json, sys
sys.path.insert(0, ROOT)
import numpy as np
import workloads
from paper_2302_09334_b200 import sim
out = {}
cases = {
    "tiny": (workloads.tiny().replace(repr_steps=5, e_repr_gt=10200), None),
    "grid64": (workloads.tiny().replace(rows=64, cols=64, slots=400, n_initial=300, repr_steps=6, e_repr_gt=10300,
                                        seeds=(9,)), None),
    "hd32": (workloads.tiny().replace(rows=40, cols=96, slots=600, n_initial=400, hidden=32, obs_radius=3,
                                      repr_steps=6, e_repr_gt=10300, seeds=(4,)), None),
    "batch": (workloads.tiny().replace(seeds=(1, 2, 3), repr_steps=5, e_repr_gt=10200), None),
    "batch_hd32": (workloads.tiny().replace(rows=40, cols=96, slots=600, n_initial=400, hidden=32, obs_radius=3,
                                            repr_steps=6, e_repr_gt=10300, seeds=tuple(range(40, 60))), None),
    "cnn": (workloads.paper_world_cnn().replace(rows=40, cols=60, slots=200, n_initial=120, repr_steps=20,
                                                 seeds=(11,)), None),
    "coloc": (workloads.paper_world_coloc().replace(rows=40, cols=60, slots=300, n_initial=150, repr_steps=20,
                                                    seeds=(12,)), None),
    "banded": (workloads.tiny().replace(rows=40, cols=96, slots=600, n_initial=400, hidden=32, obs_radius=3,
                                        repr_steps=6, e_repr_gt=10300, seeds=(4,)), dict(n_bands=4)),
}
for name, (wc, bands) in cases.items():
    w = sim.World(wc, bands=bands)
    w.step(50)
    w.synchronize()
    recs = w.step_log(0, 50)
    if bands is None:
        for _ in range(10):
            w.step_timed()
    w.synchronize()
    out[name] = recs.tolist()
    w.destroy()
print(json.dumps(out))
'''


def _run(lib):
    env = dict(os.environ, ECO_LIBSIM_OVERRIDE=lib) if lib else dict(os.environ)
    code = SCRIPT.replace("ROOT", repr(ROOT))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=600)
    return r


def test_checked_build_runs_clean_and_changes_nothing():
    from paper_2302_09334_b200 import build
    checked = build.build_checked()
    rc = _run(checked)
    assert rc.returncode == 0, f"checked build failed:\n{rc.stderr[-3000:]}"
    ref = _run(None)
    assert ref.returncode == 0, ref.stderr[-2000:]
    a = json.loads(rc.stdout.strip().splitlines()[-1])
    b = json.loads(ref.stdout.strip().splitlines()[-1])
    assert a == b


COMPACT_SCRIPT = r'''
import hashlib, json, sys
sys.path.insert(0, ROOT)
import numpy as np
import workloads
from paper_2302_09334_b200 import sim
wc = workloads.paper_scale().replace(rows=120, cols=200, slots=16384, n_initial=3000, seeds=(21,))
w = sim.World(wc)
w.step(40)
st = w.get_state()
live = st["alive"][0] == 1
h = hashlib.sha256()
for k in sim.STATE_FIELDS:
    a = st[k][0][live] if k in ("weights", "h", "c") else st[k][0]
    h.update(np.ascontiguousarray(a).tobytes())
print(json.dumps({"digest": h.hexdigest(), "records": w.step_log(0, 40).tolist()}))
w.destroy()
'''


def test_compacted_policy_forced_on_one_world_changes_nothing():
    """ECO_POL_COMPACT=1 compacts the policy's tiles for ONE world whose slots need more than a
    wave of blocks (default: several worlds only): same state and records as the default."""
    code = COMPACT_SCRIPT.replace("ROOT", repr(ROOT))
    outs = []
    for v in ("1", "0"):
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                           env=dict(os.environ, ECO_POL_COMPACT=v), timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(json.loads(r.stdout.strip().splitlines()[-1]))
    assert outs[0] == outs[1] and len(outs[0]["records"]) == 40
