"""The paper's own run on one B200: its world (App. B.4), its agents (App. B.5: the CNN-LSTM,
sampled) and its reproduction (same-cell offspring), 1e6 steps ("1e6
timesteps took 20 minutes on a single GPU"), with the Appendix C metrics on the device.

Steps in chunks of the step-log capacity, reading each chunk's records (population,
resources, births, deaths) and summarising them; wall time of the whole run (including the
record reads, the work a user's loop does) and the device time of the steps.  Writes one
JSON object (--out).  Usage: python tools/paper_run.py --steps 1000000 --out X.json"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import workloads  # noqa: E402
from paper_2302_09334_b200 import sim  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=1_000_000)
    ap.add_argument("--config", default="paper_world_coloc", choices=("paper_world_coloc", "paper_world_cnn"))
    ap.add_argument("--chunk", type=int, default=4096)
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    import torch
    wc = getattr(workloads, a.config)()
    s = torch.cuda.Stream()
    world = sim.World(wc, stream=s, log_capacity=2 * a.chunk)
    pop, res, births, deaths, walls = [], [], [], [], []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dev_ms = 0.0
    life, read_le = [], 0
    mv = np.zeros(sim.MOVE_BINS, np.int64)
    read_mv = 0
    t0 = time.perf_counter()
    done = 0
    extinct_at = None
    while done < a.steps:
        k = min(a.chunk, a.steps - done)
        e0.record(s)
        world.step(k)
        e1.record(s)
        log = world.step_log(done, k)[:, 0]  # (synchronises)
        dev_ms += e0.elapsed_time(e1)
        pop.append(log["population"].copy())
        res.append(log["resources"].copy())
        births.append(int(log["births"].sum()))
        deaths.append(int(log["deaths_energy"].sum() + log["deaths_age"].sum() + log["deaths_wall"].sum()))
        walls.append(int(log["deaths_wall"].sum()))
        done += k
        n_le = done // sim.LIFE_WINDOW  # 500-step windows completed: ages at death (App. C)
        if n_le > read_le:
            d_, a_ = world.life_windows(read_le, n_le - read_le)
            life += [float(a_[j, 0] / d_[j, 0]) if d_[j, 0] else None for j in range(n_le - read_le)]
            read_le = n_le
        n_mv = done // sim.MOVE_WINDOW  # 50-step windows completed: the 17-bin movement histogram
        if n_mv > read_mv:
            mv += world.move_hist(read_mv, n_mv - read_mv)[:, 0].sum(axis=0)
            read_mv = n_mv
        if extinct_at is None and int(log["population"][-1]) == 0:
            extinct_at = done
            break
    wall = time.perf_counter() - t0
    pop = np.concatenate(pop)
    res = np.concatenate(res)
    world.destroy()
    lv = [x for x in life if x is not None]
    idx = np.linspace(0, pop.size - 1, num=min(200, pop.size)).astype(int)
    out = {"config": a.config, "world": f"{wc.rows}x{wc.cols}", "slots": wc.slots, "steps": done,
           "extinct_at": extinct_at, "wall_s": wall, "device_ms": dev_ms,
           "steps_per_s_wall": done / wall, "steps_per_s_device": done / (dev_ms / 1e3),
           "paper": {"steps": 1_000_000, "wall_s": 1200, "source": "PAPER.md:340 (unnamed GPU, JAX)"},
           "speedup_vs_paper_wall": (1200 / 1e6) / (wall / done),
           "population": {"mean": float(pop.mean()), "min": int(pop.min()), "max": int(pop.max()),
                          "at_cap_fraction": float((pop >= wc.slots).mean()), "series_200": pop[idx].tolist()},
           "resources": {"mean": float(res.mean()), "min": int(res.min()), "max": int(res.max()),
                         "series_200": res[idx].tolist()},
           "births": int(sum(births)), "deaths": int(sum(deaths)), "wall_deaths": int(sum(walls)),
           "life_expectancy_500": {"windows": len(life), "with_deaths": len(lv),
                                   "mean": float(np.mean(lv)) if lv else None, "first": life[:5], "last": life[-5:]},
           "movement_histogram_17_bins": mv.tolist()}
    json.dump(out, open(a.out, "w"), indent=1)
    print(json.dumps({k: v for k, v in out.items() if k not in ("population", "resources")}))


if __name__ == "__main__":
    main()
