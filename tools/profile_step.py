"""Run the paper-scale world W steps through the graph path, then ONE more step whose
record (agents, active inputs, births) is written to --out as JSON together with the
algorithmic bytes of its policy launch (bench.policy_bytes).  Meant to run under
    ncu --set full -k regex:k_policy --launch-skip W --launch-count 1 ...
so the captured launch is exactly the described step (k_post: --launch-skip W - 1 too)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import workloads  # noqa: E402
from paper_2302_09334_b200 import sim  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--warmup", type=int, default=3000)
ap.add_argument("--out", required=True)
a = ap.parse_args()
wc = workloads.paper_scale()
world = sim.World(wc, device=0)
world.step(a.warmup)
world.synchronize()
t = world.t
world.step(1)
world.synchronize()
rec = world.step_log(t, 1)[0, 0]
agents, nnz, births = int(rec["agents_at_start"]), int(rec["obs_nnz"]), int(rec["births"])
out = {"workload": wc.name, "step": t, "agents": agents, "obs_nnz": nnz, "births": births,
       "policy_algorithmic_bytes": bench.policy_bytes(wc, agents, nnz),
       "step_algorithmic_bytes": bench.step_bytes(wc, agents, nnz, births)}
json.dump(out, open(a.out, "w"), indent=1)
print(json.dumps(out))
