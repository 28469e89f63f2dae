"""Diagnostic: large world, unsharded vs G-rank sharded (host-sequenced on one GPU), step by
step from the same state; reports the first step whose integer state differs and where."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads  # noqa: E402
from paper_2302_09334_b200 import sim  # noqa: E402
import torch  # noqa: E402

G = int(sys.argv[1]) if len(sys.argv) > 1 else 2
W = int(sys.argv[2]) if len(sys.argv) > 2 else 150
K = int(sys.argv[3]) if len(sys.argv) > 3 else 20
wc = workloads.large_world()
F = ("resources", "alive", "cell", "energy", "age", "repr")
ref = sim.World(wc, log_capacity=W + K + 16)
ref.step(W)
snap = ref.get_state()
ranks = [sim.World(wc, log_capacity=W + K + 16) for _ in range(G)]
for r, w in enumerate(ranks):
    w.set_state(snap)
    w.shard(G, r)
bufs = [w.exchange_tensors() for w in ranks]
for k in range(K):
    ref.step(1)
    for w in ranks:
        w.step_policy()
    for w in ranks:
        w.synchronize()
    m = sum(b[0] for b in bufs)
    c = sum(b[1] for b in bufs)
    for b in bufs:
        b[0].copy_(m)
        b[1].copy_(c)
    torch.cuda.synchronize()
    for w in ranks:
        w.step_post()
    sr = ref.get_state(F)
    ss = [w.get_state(F) for w in ranks]
    lr, ls = ref.step_log(W + k, 1)[0, 0], ranks[0].step_log(W + k, 1)[0, 0]
    live = sr["alive"][0] == 1
    def eq(f, a, b):
        if f in ("cell", "energy", "age", "repr"):
            return np.array_equal(a[f][0][live], b[f][0][live])
        return np.array_equal(a[f], b[f])
    diff = [f for f in F if not eq(f, sr, ss[0])]
    rdiff = {f: (int(ls[f]), int(lr[f])) for f in ls.dtype.names if ls[f] != lr[f]}
    cross = [f for f in F if not all(eq(f, ss[0], x) for x in ss[1:])]
    print("step", W + k, "state diff", diff, "record diff", rdiff, "ranks disagree", cross, flush=True)
    if diff or rdiff:
        for f in diff:
            d = (sr[f] != ss[0][f])
            if f in ("cell", "energy", "age", "repr"):
                d = d & (sr["alive"] == 1)
            idx = np.argwhere(d)[:5]
            print("  ", f, idx.tolist(), [(int(sr[f][tuple(i)]), int(ss[0][f][tuple(i)])) for i in idx])
        break
