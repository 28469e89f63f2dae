"""The 64-world ensemble's graph kernels (policy, k_post) at step ~t with the slot pool shrunk
(same agents, fewer empty policy blocks): what the empty contexts of the full 8,192-slot
pools cost the policy launch.  Usage: python tools/diag_ens_slots.py [slots ...]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2302_09334_b200 import sim  # noqa: E402

W, K = 20, 30
for slots in [int(a) for a in sys.argv[1:]] or [8192, 2048]:
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        wc = workloads.ensemble().replace(slots=slots)
        world = sim.World(wc, device=0, stream=s, log_capacity=256)
        fb = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
        fr = torch.ones((256 << 20) // 4, dtype=torch.float32, device="cuda")
        world.step(W)
        world.synchronize()
        g = np.zeros(2)
        for k in range(K):
            fb.zero_()
            fr.sum()
            tg = world.step_graph_timed()
            g += (tg["policy"], tg["post"])
        log = world.step_log(W, K)
        print({"slots": slots, "policy_us": round(g[0] / K * 1e3, 1), "post_us": round(g[1] / K * 1e3, 1),
               "agents_mean": float(log["agents_at_start"].sum() / K), "births_mean": float(log["births"].sum() / K)})
        world.destroy()
