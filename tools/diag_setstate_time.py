"""Time sim_set_state of the paper-scale world's state from pinned host buffers (the e2e
leg's H2D), zero-copy gather vs DMA runs (ECO_SETSTATE_ZC), then sim_step(20)."""
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
live = np.flatnonzero(snap["alive"][0])
runs = 1 + int((np.diff(live) != 1).sum())
ts = []
for rep in range(6):
    w.synchronize()
    t0 = time.perf_counter()
    w.set_state(pinned)
    t1 = time.perf_counter()
    w.step(20)
    w.synchronize()
    t2 = time.perf_counter()
    ts.append((t1 - t0, t2 - t1))
ts = np.array(ts[1:]) * 1e3
print(os.environ.get("ECO_SETSTATE_ZC", "auto"), f"live {live.size} runs {runs}", "set_state ms", np.round(ts[:, 0], 3),
      "step(20) ms", np.round(ts[:, 1], 3))
