import sys; sys.path.insert(0, '.')
import numpy as np, workloads
from paper_2302_09334_b200 import sim
w = sim.World(workloads.paper_scale(), device=0, log_capacity=16384)
w.step(10005); w.synchronize()
lg = w.step_log(5, 10000)[:, 0]
nc = lg["deferred_no_cell"] + lg["deferred_claim"] + lg["deferred_capacity"] + lg["births"]
for lo, hi in ((0, 1000), (1000, 2000), (2000, 5000), (5000, 10000)):
    a = nc[lo:hi]
    print(lo, hi, "n_cand q50", np.median(a), "q90", np.quantile(a, .9), "max", a.max(), "agents", lg["agents_at_start"][lo:hi].mean())
