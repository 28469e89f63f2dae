"""Graph path vs instrumented path from the same state: first step whose record differs."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads  # noqa: E402
from paper_2302_09334_b200 import sim  # noqa: E402

W = int(sys.argv[1]) if len(sys.argv) > 1 else 5
K = int(sys.argv[2]) if len(sys.argv) > 2 else 400
wc = workloads.paper_scale()
world = sim.World(wc, device=0, log_capacity=max(8192, K + 16))
world.step(W)
snap = world.get_state()
t0 = world.t
world.step(K)
log_g = world.step_log(t0, K)[:, 0]
st_g = world.get_state()
world.set_state(snap)
for k in range(K):
    world.step_timed()
log_t = world.step_log(t0, K)[:, 0]
st_t = world.get_state()
bad = [k for k in range(K) if log_g[k] != log_t[k]]
print("first differing step", (t0 + bad[0]) if bad else None, "n", len(bad))
if bad:
    k = bad[0]
    for f in log_g.dtype.names:
        if log_g[f][k] != log_t[f][k]:
            print("  ", f, log_g[f][k], log_t[f][k])
    print("births around", [int(x) for x in log_g["births"][max(0, k - 3):k + 2]])
for f in ("alive", "cell", "energy", "weights"):
    a, b = st_g[f], st_t[f]
    print(f, "equal" if np.array_equal(a, b) else f"differs in {int(np.sum(a != b))} entries")
