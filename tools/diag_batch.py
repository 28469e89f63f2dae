"""Diagnostic: step a batched ensemble and the matching single worlds in lock-step and
report the first step/world/field where they differ (GPU only)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads  # noqa: E402
from paper_2302_09334_b200 import sim  # noqa: E402

seeds = (100, 131, 163)
wc = workloads.ensemble(seeds).replace(slots=4096)
batched = sim.World(wc)
singles = [sim.World(wc.replace(seeds=(s,))) for s in seeds]
for t in range(80):
    gb = batched.get_state()
    for wi, sw in enumerate(singles):
        g1 = sw.get_state()
        for k in sim.STATE_FIELDS:
            a, b = gb[k][wi], g1[k][0]
            if k not in ("resources", "alive"):
                live = g1["alive"][0] == 1
                a, b = a[live], b[live]
            if not np.array_equal(a, b):
                bad = np.argwhere(a != b)[:5]
                print(f"step {t} world {wi} field {k} differs at {bad.tolist()}")
                lb = batched.step_log(t - 1, 1)[0, wi] if t > 0 else None
                ls = sw.step_log(t - 1, 1)[0, 0] if t > 0 else None
                print("batched rec", lb)
                print("single  rec", ls)
                sys.exit(1)
    batched.step(1)
    for sw in singles:
        sw.step(1)
print("no difference in 80 steps")
