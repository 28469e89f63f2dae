"""Event-timed cost of launching nearly empty work between L2 flushes (the bench's timing
pattern): one tiny kernel, a CUDA graph of two tiny kernels, and the library's step, to
separate launch and event overhead from the step's own kernels."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import workloads  # noqa: E402
from paper_2302_09334_b200 import sim  # noqa: E402

s = torch.cuda.Stream()
K = 2000
with torch.cuda.stream(s):
    fb = torch.empty(bench.FLUSH_BYTES, dtype=torch.uint8, device="cuda")
    fr = torch.ones(bench.FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")
    x = torch.zeros(32, device="cuda")
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        x.add_(1.0)
        x.mul_(1.0)
    world = sim.World(workloads.paper_scale(), device=0, stream=s, log_capacity=8192)
    world.step(3000)

    def run(fn):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        torch.cuda.synchronize()
        for k in range(K):
            fb.zero_()
            fr.sum()
            evs[k][0].record(s)
            fn()
            evs[k][1].record(s)
        torch.cuda.synchronize()
        return float(np.median([a.elapsed_time(b) for a, b in evs]) * 1e3)

    print({"one_tiny_kernel_us": run(lambda: x.add_(1.0)), "graph_of_two_tiny_kernels_us": run(g.replay),
           "library_step_us": run(lambda: world.step(1))})
