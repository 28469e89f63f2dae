"""Run the paper-scale world W steps through the graph path, then ONE instrumented step
(sim_step_timed: the split policy, the phase kernels and k_prepare_p, the P rows of the next
step) whose record (agents, active inputs, births, population) is written to --out as JSON
with the algorithmic bytes of its policy and k_prepare_p launches (bench.policy_bytes,
bench.hh_bytes).  Meant to run under
    ncu --set full -k regex:"k_policy_half|k_prepare_p|k_post" --launch-skip 2W --launch-count 3
(launches: one k_prepare_p at start, W x (policy, k_post), then the timed policy and
k_prepare_p), which captures the graph path's last k_post and the described step's policy
and P rows."""
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
ap.add_argument("--config", default="paper_scale", choices=("paper_scale", "large_world", "ensemble", "paper_world",
                                                                 "paper_world_cnn", "paper_world_coloc"))
ap.add_argument("--out", required=True)
a = ap.parse_args()
wc = getattr(workloads, a.config)()
world = sim.World(wc, device=0)
world.step(a.warmup)
world.synchronize()
t = world.t
world.step_timed()
world.synchronize()
lg, lp = world.step_log(t, 1)[0], world.step_log(t - 1, 1)[0]  # every world's record
rec = {f: int(lg[f].sum()) for f in lg.dtype.names}  # summed over the worlds
prev = {f: int(lp[f].sum()) for f in lp.dtype.names}  # the step of the captured k_post
agents, nnz, births = int(rec["agents_at_start"]), int(rec["obs_nnz"]), int(rec["births"])
out = {"workload": wc.name, "step": t, "agents": agents, "obs_nnz": nnz, "births": births,
       "population": int(rec["population"]),
       "policy_algorithmic_bytes": bench.policy_bytes(wc, agents, nnz),
       "hh_algorithmic_bytes": bench.hh_bytes(wc, int(rec["population"])),
       "post_algorithmic_bytes": bench.post_bytes(wc, int(prev["agents_at_start"]), int(prev["births"])),
       "post_step": t - 1,
       "step_algorithmic_bytes": bench.step_bytes(wc, agents, nnz, births)}
json.dump(out, open(a.out, "w"), indent=1)
print(json.dumps(out))
