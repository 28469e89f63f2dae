"""Time sim_set_state of the paper-scale world's t=5 state from pinned host buffers with
subsets of the fields (where the e2e leg's H2D time goes)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2302_09334_b200 import sim  # noqa: E402

wc = workloads.paper_scale()
w = sim.World(wc)
w.step(5)
snap = w.get_state()
pinned = {}
for k, v in snap.items():
    if isinstance(v, np.ndarray):
        tt = torch.empty(v.shape, dtype=getattr(torch, str(v.dtype)), pin_memory=True)
        tt.numpy()[...] = v
        pinned[k] = tt.numpy()
    else:
        pinned[k] = v
allf = [k for k in pinned if isinstance(pinned[k], np.ndarray)]
subsets = {"all": allf, "weights+alive+cell": ["weights", "alive", "cell"], "alive+cell": ["alive", "cell"],
           "all-but-weights": [k for k in allf if k != "weights"], "all-but-logits": [k for k in allf if k != "logits"],
           "none": []}
for name, fs in subsets.items():
    st = {k: pinned[k] for k in fs}
    st["t"] = pinned["t"]
    ts = []
    for rep in range(7):
        w.synchronize()
        t0 = time.perf_counter()
        w.set_state(st)
        ts.append(time.perf_counter() - t0)
    print(f"{name:22s} set_state ms median {np.median(ts[2:]) * 1e3:.3f} min {min(ts[2:]) * 1e3:.3f}", flush=True)
