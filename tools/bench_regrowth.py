"""Regrowth microbenchmark (BASELINE.json configs[2]): agent-free worlds
of 200x400, 2048x4096 and 8192x16384 cells, seed 2, 1000 steps each.

For every grid: the whole world step through sim_step (CUDA graph; with no agents the step
is the regrowth of the next step's grid plus the bookkeeping of the cooperative kernel),
timed per step with CUDA events, L2 flushed between steps (256 MiB memset + 256 MiB read,
as bench.py); then the same steps replayed through sim_step_timed, which runs the regrowth
as the standalone k_regrow kernel, timed alone.  Reported separately for the growth phase
(steps 0-199, Philox-bound while the grid fills) and the saturated phase (steps 200-999,
full 4-cell groups skip Philox), plus the aggregate:
  * cell-updates/s of the step and of the regrowth kernel;
  * the regrowth kernel's fraction of the HBM roofline at its algorithmic bytes (bit planes:
    H*W/8 read + H*W/8 written per step, 0.25 B/cell).
Writes one JSON object (stdout, and --out).  Not a bench.py line: BASELINE's headline is
the paper-scale world step; this is the supporting measurement D.2 asks for.
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import workloads  # noqa: E402


def run_grid(H, W, steps, flush, flush_rd, stream):
    import torch
    from paper_2302_09334_b200 import sim
    wc = workloads.regrowth_micro(H, W)
    with torch.cuda.stream(stream):
        world = sim.World(wc, device=0, stream=stream, log_capacity=steps + 8)
        snap = world.get_state()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        torch.cuda.synchronize()
        for k in range(steps):
            flush.zero_()
            flush_rd.sum()
            evs[k][0].record(stream)
            world.step(1)
            evs[k][1].record(stream)
        torch.cuda.synchronize()
        step_ms = np.array([a.elapsed_time(b) for a, b in evs])
        log = world.step_log(0, steps)[:, 0]
        # replay with the standalone regrowth kernel timed alone
        world.set_state(snap)
        kern_ms = np.zeros(steps)
        for k in range(steps):
            flush.zero_()
            flush_rd.sum()
            kern_ms[k] = world.step_timed()["regrow"]
        log2 = world.step_log(0, steps)[:, 0]
        # the config's run as ONE sim_step(steps) call bracketed by CUDA events (no event pair or
        # L2 flush per step: the grid's two planes exceed the L2 from 2048x4096 up anyway)
        world.set_state(snap)
        world.synchronize()
        ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ea.record(stream)
        world.step(steps)
        eb.record(stream)
        world.synchronize()
        call_ms = ea.elapsed_time(eb)
        log3 = world.step_log(0, steps)[:, 0]
        world.destroy()
    cells = H * W
    peak, peak_src = bench.peaks()

    def part(lo, hi):
        s, kk = step_ms[lo:hi].sum() / 1e3, kern_ms[lo:hi].sum() / 1e3
        n = (hi - lo) * cells
        bytes_ = (hi - lo) * cells / 4  # 0.25 B per cell: bit plane read + written
        return {"steps": [lo, hi], "step_cell_updates_per_s": n / s, "step_us": s / (hi - lo) * 1e6,
                "regrow_kernel_cell_updates_per_s": n / kk, "regrow_kernel_us": kk / (hi - lo) * 1e6,
                "regrow_kernel_GBps": bytes_ / kk / 1e9, "regrow_kernel_hbm_frac": bytes_ / kk / 1e9 / peak,
                "grown": int(log["grown"][lo:hi].sum())}

    return {"grid": f"{H}x{W}", "cells": cells, "steps": steps,
            "growth": part(0, min(200, steps)), "saturated": part(min(200, steps), steps), "all": part(0, steps),
            "one_call": {"what": f"sim_step({steps}) as one call, CUDA events around it", "ms": call_ms,
                         "step_us": call_ms / steps * 1e3, "cell_updates_per_s": steps * cells / (call_ms / 1e3),
                         "plane_GBps": steps * cells / 4 / (call_ms / 1e3) / 1e9},
            "final_resources": int(log["resources"][-1]),
            "replay_identical": bool(np.array_equal(log, log2) and np.array_equal(log, log3)),
            "peak_GBps": peak, "peak_source": peak_src}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--grids", default="200x400,2048x4096,8192x16384")
    ap.add_argument("--out")
    a = ap.parse_args()
    import torch
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(device=dev)
    flush = torch.empty(bench.FLUSH_BYTES, dtype=torch.uint8, device=dev)
    flush_rd = torch.ones(bench.FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    out = {"benchmark": "regrowth microbenchmark (BASELINE.json configs[2], seed 2)", "data": "synthetic",
           "l2": "flushed between steps (256 MiB memset + 256 MiB read)", "results": []}
    for g in a.grids.split(","):
        H, W = (int(x) for x in g.split("x"))
        out["results"].append(run_grid(H, W, a.steps, flush, flush_rd, stream))
        print(json.dumps(out["results"][-1]), file=sys.stderr, flush=True)
    txt = json.dumps(out, indent=1)
    if a.out:
        open(a.out, "w").write(txt)
    print(txt)


if __name__ == "__main__":
    main()
