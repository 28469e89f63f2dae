"""Diagnostic: a small banded world stepped next to the unbanded one (for compute-sanitizer)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import workloads  # noqa: E402
from paper_2302_09334_b200 import sim  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "tiny"
G = int(sys.argv[2]) if len(sys.argv) > 2 else 2
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
wc = {"tiny": workloads.tiny().replace(slots=64, n_initial=40), "paper": workloads.paper_scale()}[cfg]
ban = sim.World(wc, bands=dict(n_bands=G))
print("created", flush=True)
for t in range(steps):
    ban.step(1)
    ban.synchronize()
    print("step", t, "ok", flush=True)
st = ban.get_state()
print("alive", int(st["alive"].sum()), "res", int(st["resources"].sum()))
