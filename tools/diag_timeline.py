"""Per-step kernel timeline of the graph path (diagnostic build with -DECO_TIMELINE): the
policy's and k_post's first-block start and last-block end (globaltimer), L2 flushed between
steps as in bench.py.  Prints medians (us) of policy, gap, k_post, and the step."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2302_09334_b200 import build as B  # noqa: E402

diag = os.path.join(B.HERE, "libsim_timeline.so")
if not (os.environ.get("DIAG_NOBUILD") and os.path.exists(diag)):
    B.build(defines=("ECO_TIMELINE",), out=diag)
os.environ["ECO_LIBSIM_OVERRIDE"] = diag
import torch  # noqa: E402

import bench  # noqa: E402
import workloads  # noqa: E402
from paper_2302_09334_b200 import sim  # noqa: E402

W, K = (int(sys.argv[1]) if len(sys.argv) > 1 else 3000), (int(sys.argv[2]) if len(sys.argv) > 2 else 1000)
flush = "--no-flush" not in sys.argv
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    world = sim.World(workloads.paper_scale(), device=0, stream=s, log_capacity=W + K + 8)
    fb = torch.empty(bench.FLUSH_BYTES, dtype=torch.uint8, device="cuda")
    fr = torch.ones(bench.FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")
    world.step(W)
    world.synchronize()
    world.phase_ns(reset=True)
    for _ in range(K):
        if flush:
            fb.zero_()
            fr.sum()
        world.step(1)
    world.synchronize()
out = np.zeros(16 + 32768, np.int64)
sim._check(sim.lib().sim_get_phase_ns(world._h, sim._ptr(out), -1))
tl = out[16:16 + 4096].view(np.uint64).reshape(1024, 4).copy()
tl[:, 0] = ~tl[:, 0]
tl[:, 2] = ~tl[:, 2]
ts = [(W + k) & 1023 for k in range(K)]
r = tl[ts].astype(np.float64)
pol = (r[:, 1] - r[:, 0]) / 1e3
gap = (r[:, 2] - r[:, 1]) / 1e3
post = (r[:, 3] - r[:, 2]) / 1e3
nxt = (r[1:, 0] - r[:-1, 3]) / 1e3
med = lambda a: round(float(np.median(a)), 2)  # noqa: E731
print({"flush": flush, "policy_us": med(pol), "policy_to_post_gap_us": med(gap), "post_us": med(post),
       "post_to_next_policy_us": med(nxt), "policy_start_to_post_end_us": med(pol + gap + post)})
