"""Diagnostic: agent-sharded stepping of a world as 2 ranks on one GPU, synchronising after
every launch to locate a failure."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads  # noqa: E402
from paper_2302_09334_b200 import sim  # noqa: E402

import torch  # noqa: E402

wc = workloads.paper_scale().replace(slots=2048, n_initial=600)
ref = sim.World(wc)
ranks = [sim.World(wc) for _ in range(2)]
for r, w in enumerate(ranks):
    w.shard(2, r)
for k in range(60):
    for r in ranks:
        r.step_policy()
        r.synchronize()
    bufs = [r.exchange_tensors() for r in ranks]
    m0, m1 = bufs[0][0].view(-1, 4), bufs[1][0].view(-1, 4)
    n = int(ranks[0].step_log(k - 1, 1)[0, 0]["population"]) if k > 0 else 600
    both = ((m0 != 0).any(1) & (m1 != 0).any(1))
    if both.any():
        print("step", k, "list positions written by both ranks:", int(both.sum()), torch.nonzero(both)[:5].flatten().tolist())
    m = bufs[0][0] + bufs[1][0]
    rec = bufs[0][1] + bufs[1][1]
    for b in bufs:
        b[0].copy_(m)
        b[1].copy_(rec)
    torch.cuda.synchronize()
    for i, r in enumerate(ranks):
        try:
            r.step_post()
            r.synchronize()
        except Exception as e:
            print("post failed at step", k, "rank", i, e)
            raise
    ref.step(1)
    la, lr = ranks[0].step_log(k, 1)[0, 0], ref.step_log(k, 1)[0, 0]
    if la != lr:
        print("step", k, "record differs:", {f: (int(la[f]), int(lr[f])) for f in la.dtype.names if la[f] != lr[f]})
print("done")
