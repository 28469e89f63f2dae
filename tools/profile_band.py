"""Drive the banded large world for an ncu launch list: configs[3] as G bands (agent-weighted
rows at its population cap) stepped W steps on this GPU, then one more step.  Under
`ncu --metrics gpu__time_duration.sum -s <skip>` the per-kernel durations of one banded step
(every band's kernels) come out; tools/band_scaling.py gives the phase sums."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import workloads  # noqa: E402

ROWS = {2: [0, 1023, 1600], 4: [0, 663, 1023, 1321, 1600], 8: [0, 422, 663, 854, 1023, 1177, 1321, 1460, 1600]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--G", type=int, default=8)
    ap.add_argument("--warmup", type=int, default=160)
    ap.add_argument("--steps", type=int, default=2)
    a = ap.parse_args()
    from paper_2302_09334_b200 import sim
    wc = workloads.large_world()
    w = sim.World(wc, bands=dict(n_bands=a.G, band_rows=ROWS[a.G], band_slots=int(wc.slots / a.G * 1.6 + 4096)))
    w.step(a.warmup)
    w.synchronize()
    for _ in range(a.steps):
        w.band_step_timed()
    print("done", w.t)


if __name__ == "__main__":
    main()
