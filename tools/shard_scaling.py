"""Agent-sharded strong-scaling estimate on ONE GPU (this environment has one).

For G ranks, G handles of the same world are stepped in lock step on this GPU, the host
sequencing each rank's policy launch, the SUM-combine of the exchange buffers and each
rank's dynamics launch (no kernel waits on another rank's).  Every launch is timed alone
with CUDA events, so a rank's per-step time on a G-GPU node is estimated as
    max over ranks (policy) + allreduce + max over ranks (dynamics)
with the allreduce of the 16 B/slot move records taken as a measured device-to-device copy
of that size (NVLink/NCCL time is not measured here).  The trajectory is checked against the
unsharded world (records identical).  Prints one JSON object.
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads  # noqa: E402
from paper_2302_09334_b200 import sim  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="large_world")
    ap.add_argument("--ranks", default="1,2,4")
    ap.add_argument("--warmup", type=int, default=150)
    ap.add_argument("--steps", type=int, default=30)
    a = ap.parse_args()
    import torch
    wc = workloads.large_world() if a.config == "large_world" else workloads.paper_scale()
    out = {"config": wc.name, "warmup": a.warmup, "steps": a.steps, "results": []}
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    cur = torch.cuda.Stream()  # the handles run on this stream; events are recorded on it
    torch.cuda.set_stream(cur)
    ref = sim.World(wc, stream=cur, log_capacity=a.warmup + a.steps + 16)
    ref.step(a.warmup)
    snap = ref.get_state()
    e0, e1 = ev(), ev()
    torch.cuda.synchronize()
    e0.record()
    ref.step(a.steps)
    e1.record()
    torch.cuda.synchronize()
    ref_ms = e0.elapsed_time(e1) / a.steps
    ref_log = ref.step_log(a.warmup, a.steps)
    agents = float(ref_log["agents_at_start"].mean())
    ref.destroy()
    for G in [int(x) for x in a.ranks.split(",")]:
        if G == 1:
            out["results"].append({"ranks": 1, "step_ms": ref_ms, "agents_mean": agents})
            continue
        ranks = [sim.World(wc, stream=cur, log_capacity=a.warmup + a.steps + 16) for _ in range(G)]
        for r, w in enumerate(ranks):
            w.set_state(snap)
            w.shard(G, r)
        bufs = [w.exchange_tensors() for w in ranks]
        pol = np.zeros((a.steps, G))
        post = np.zeros((a.steps, G))
        comb = np.zeros(a.steps)
        for k in range(a.steps):
            for r, w in enumerate(ranks):
                s0, s1 = ev(), ev()
                torch.cuda.synchronize()
                s0.record()
                w.step_policy()
                w.synchronize()
                s1.record()
                torch.cuda.synchronize()
                pol[k, r] = s0.elapsed_time(s1)
            c0, c1 = ev(), ev()
            c0.record()
            m = sum(b[0] for b in bufs)
            ctr = sum(b[1] for b in bufs)
            for b in bufs:
                b[0].copy_(m)
                b[1].copy_(ctr)
            c1.record()
            torch.cuda.synchronize()
            comb[k] = c0.elapsed_time(c1) / (2 * G)  # ~ one buffer's copy: the allreduce stand-in
            for r, w in enumerate(ranks):
                s0, s1 = ev(), ev()
                s0.record()
                w.step_post()
                w.synchronize()
                s1.record()
                torch.cuda.synchronize()
                post[k, r] = s0.elapsed_time(s1)
        lg = ranks[0].step_log(a.warmup, a.steps)
        same = all(np.array_equal(w.step_log(a.warmup, a.steps), ref_log) for w in ranks)
        if not same:
            bad = [k for k in range(a.steps) if lg[k] != ref_log[k]]
            if bad:
                k = bad[0]
                print("first differing step", a.warmup + k, {f: (int(lg[f][k][0]), int(ref_log[f][k][0]))
                      for f in lg.dtype.names if lg[f][k][0] != ref_log[f][k][0]}, file=sys.stderr)
        est = pol.max(1) + comb + post.max(1)
        out["results"].append({
            "ranks": G, "step_ms_estimate": float(est.mean()), "policy_ms_max": float(pol.max(1).mean()),
            "dynamics_ms_max": float(post.max(1).mean()), "exchange_ms": float(comb.mean()),
            "speedup_estimate": ref_ms / float(est.mean()), "efficiency_estimate": ref_ms / float(est.mean()) / G,
            "records_equal_unsharded": bool(same)})
        for w in ranks:
            w.destroy()
        torch.cuda.synchronize()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
