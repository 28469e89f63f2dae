"""k_post end clocks (diagnostic build with -DECO_END_CLOCK, loaded via ECO_LIBSIM_OVERRIDE):
per launch, the latest end of the split's P warps and of the dynamics warps after block 0's
start, averaged over K steps of the paper-scale world, beside block 0's phase clocks and
the graph step time."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2302_09334_b200 import sim  # noqa: E402

W, K = (int(sys.argv[1]) if len(sys.argv) > 1 else 5), (int(sys.argv[2]) if len(sys.argv) > 2 else 10000)
s = torch.cuda.Stream()
world = sim.World(workloads.paper_scale(), device=0, stream=s, log_capacity=W + K + 8)
world.step(W)
world.synchronize()
world.phase_ns(reset=True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
world.step(K)
e1.record(s)
world.synchronize()
ph = {k: v / K / 1e3 for k, v in world.phase_ns().items()}
print(os.environ.get("ECO_LIBSIM_OVERRIDE"), {"step_us": e0.elapsed_time(e1) / K * 1e3, "r6": ph["reserved6"], "r7": ph["reserved7"],
      "p_warps_end_us": ph["reserved4"], "dyn_end_us": ph["reserved5"],
      **{k: round(v, 2) for k, v in ph.items() if not k.startswith("reserved")}})
