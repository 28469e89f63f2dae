"""Per-step time of the agent-free 8192x16384 world along its natural trajectory (L2 flushed):
how the step approaches the streaming floor as the grid fills.  Also an all-full grid."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2302_09334_b200 import sim  # noqa: E402

wc = workloads.regrowth_micro(8192, 16384)
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    world = sim.World(wc, device=0, stream=s, log_capacity=2048)
    fb = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    fr = torch.ones((256 << 20) // 4, dtype=torch.float32, device="cuda")
    out = {}
    t = 0
    for mark in (10, 100, 200, 250, 300, 400, 500, 700, 900, 1200, 1600, 2400):
        world.step(mark - t)
        t = mark
        ts = []
        for _ in range(5):
            fb.zero_()
            fr.sum()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            world.step(1)
            b.record(s)
            world.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
            t += 1
        rec = world.step_log(t - 1, 1)[0, 0]
        out[mark] = (round(float(np.median(ts)), 1), int(rec["resources"]), int(rec["grown"]))
        print(mark, out[mark], flush=True)
