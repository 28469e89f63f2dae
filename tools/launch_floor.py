"""The event-timed floor of a step in bench.py's loop: flush L2 (256 MiB memset + read), event,
a CUDA graph of 1 or 2 tiny kernels, event; median over K steps (us)."""
import sys

import numpy as np
import torch

FLUSH = 256 << 20
K = 200
s = torch.cuda.Stream()
x = torch.zeros(1, device="cuda")
with torch.cuda.stream(s):
    fb = torch.empty(FLUSH, dtype=torch.uint8, device="cuda")
    fr = torch.ones(FLUSH // 4, dtype=torch.float32, device="cuda")
    for nk in (1, 2):
        g = torch.cuda.CUDAGraph()
        x.add_(1)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for _ in range(nk):
                x.add_(1)
        for flush in (True, False):
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
            for k in range(K):
                if flush:
                    fb.zero_()
                    fr.sum()
                evs[k][0].record(s)
                g.replay()
                evs[k][1].record(s)
            torch.cuda.synchronize()
            t = np.array([a.elapsed_time(b) for a, b in evs]) * 1e3
            print(f"graph of {nk} tiny kernel(s), flush={flush}: median {np.median(t):.2f} us, min {t.min():.2f}")
