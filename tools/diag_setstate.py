"""Wall time of sim_set_state from pinned host buffers (the e2e leg's one-off cost) beside a
plain pinned H2D copy of the same bytes."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2302_09334_b200 import sim  # noqa: E402

world = sim.World(workloads.paper_scale(), device=0)
world.step(5)
snap = world.get_state()
pinned, nbytes = {}, 0
for k, v in snap.items():
    if isinstance(v, np.ndarray):
        tt = torch.empty(v.shape, dtype=getattr(torch, str(v.dtype)), pin_memory=True)
        tt.numpy()[...] = v
        pinned[k] = tt.numpy()
        nbytes += v.nbytes
    else:
        pinned[k] = v
out = {"state_bytes": nbytes, "set_state_ms": []}
for _ in range(5):
    world.synchronize()
    t0 = time.perf_counter()
    world.set_state(pinned)
    out["set_state_ms"].append((time.perf_counter() - t0) * 1e3)
src = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
dst = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
for _ in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    out.setdefault("h2d_copy_ms", []).append((time.perf_counter() - t0) * 1e3)
print(out)
