"""k_post end clocks (ECO_END_CLOCK build via ECO_LIBSIM_OVERRIDE) in the bench's regime: W
warm-up steps, then K single steps with the L2 flushed before each (as bench.py), averaged:
the latest end of the P warps and of the dynamics warps after block 0's start, block 0's
phase clocks and the event-timed step."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import workloads  # noqa: E402
from paper_2302_09334_b200 import sim  # noqa: E402

W, K = (int(sys.argv[1]) if len(sys.argv) > 1 else 5), (int(sys.argv[2]) if len(sys.argv) > 2 else 20)
flush = "--no-flush" not in sys.argv
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    world = sim.World(workloads.paper_scale(), device=0, stream=s, log_capacity=W + K + 8)
    fb = torch.empty(bench.FLUSH_BYTES, dtype=torch.uint8, device="cuda")
    fr = torch.ones(bench.FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")
    if "--preflush" in sys.argv:
        fb.zero_()
        fr.sum()
    world.step(W)
    world.synchronize()
    world.phase_ns(reset=True)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    if "--twice" in sys.argv:  # a first timed loop, a host synchronisation, then the measured loop
        for k in range(K):
            if flush:
                fb.zero_()
                fr.sum()
            evs[k][0].record(s)
            world.step(1)
            evs[k][1].record(s)
        world.synchronize()
        print("first loop per-step us:", np.round(np.array([a.elapsed_time(b) for a, b in evs]) * 1e3, 1).tolist())
    if "--lead" in sys.argv:  # the GPU busy ~1 ms before the first timed step: the host runs ahead
        torch.cuda._sleep(2_000_000)
    for k in range(K):
        if flush:
            fb.zero_()
            fr.sum()
        evs[k][0].record(s)
        world.step(1)
        evs[k][1].record(s)
    world.synchronize()
ph = {k: v / K / 1e3 for k, v in world.phase_ns().items()}
per = np.array([a.elapsed_time(b) for a, b in evs]) * 1e3
step = float(per.mean())
print("per-step us (t = W..W+K):", np.round(per, 1).tolist())
print({"flush": flush, "W": W, "K": K, "step_us": round(step, 2), "p_warps_end_us": round(ph["reserved4"], 2),
       "dyn_end_us": round(ph["reserved5"], 2), **{k: round(v, 2) for k, v in ph.items() if not k.startswith("reserved")}})
