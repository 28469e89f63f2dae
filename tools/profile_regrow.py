"""Drive the configs[2] regrowth world for ncu: steps an agent-free 8192x16384 world (seed 2)
through sim_step (whose graph launches k_regrow_tiled once per step; the first launch is the
regrowth of step 0).  Under `ncu -k regex:k_regrow_tiled -s N -c 1` the captured launch is
the regrowth of step N (growth phase for N < ~100, saturated for N > ~500)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import workloads  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--grid", default="8192x16384")
    a = ap.parse_args()
    from paper_2302_09334_b200 import sim
    H, W = (int(x) for x in a.grid.split("x"))
    world = sim.World(workloads.regrowth_micro(H, W), log_capacity=max(4096, a.steps + 8))
    world.step(a.steps)
    world.synchronize()
    log = world.step_log(0, a.steps)[:, 0]
    print(f"{a.grid}: {a.steps} steps, resources {int(log['resources'][-1])}")
    world.destroy()


if __name__ == "__main__":
    main()
