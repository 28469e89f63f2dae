"""One-GPU estimate of the banded large world's multi-GPU step time and efficiency
(BASELINE configs[3]; only one GPU is available to this build).

* T(1): the unbanded configs[3] world (1600x3200, 262,144 slots, 64,000 initial agents) at
  its population cap, device-timed per step (CUDA events; the split-policy graph path).
* For G = 2, 4, 8: the same world as G bands on this one GPU (identical trajectory), equal
  rows and agent-weighted rows (each band ~A/G agents at the timed steps, from the unbanded
  world's agent rows); after the warm-up, sim_band_step_timed times every band's phases
  alone (the bands run one after the other), i.e. what each band's own GPU would spend.
* Estimate of a G-GPU step: sum over phases of the slowest band's phase time (the P rows of
  the split policy overlap the phases after them, as on the second stream of sim_step), plus the
  phase barriers (5 neighbour token exchanges and 1 all-reduce per step) at an ASSUMED
  latency (--nbr-us, --all-us: NCCL over NVLink, not measured here); the exchanges
  themselves are pull kernels inside the phase times.  E(G) = T(1) / (G T(G)).
* Graph estimate (the per-GPU step captured as one CUDA graph, NCCL barriers inside, as
  api_band.inc does): the banded world's one-GPU graph step (all G bands one after the
  other, T_graph) / G, times the slowest band's share of the event-timed band totals, plus
  the same assumed barriers.  The event-timed phases above include every launch's own
  latency; inside a graph consecutive kernels start ~1 us apart.
Writes one JSON object (stdout, --out)."""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import workloads  # noqa: E402


def weighted_rows(rows_hist: np.ndarray, G: int, min_rows: int = 3) -> list:
    """Row boundaries giving each band about 1/G of the agents (>= min_rows rows each)."""
    H = rows_hist.size
    cum = np.cumsum(rows_hist)
    tot = cum[-1]
    b = [0]
    for k in range(1, G):
        y = int(np.searchsorted(cum, tot * k / G)) + 1
        y = max(y, b[-1] + min_rows)
        y = min(y, H - (G - k) * min_rows)
        b.append(y)
    b.append(H)
    return b


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--warmup", type=int, default=160)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--gs", default="2,4,8")
    ap.add_argument("--nbr-us", type=float, default=10.0)
    ap.add_argument("--all-us", type=float, default=15.0)
    ap.add_argument("--config", default="large_world")
    ap.add_argument("--out")
    a = ap.parse_args()
    import torch
    from paper_2302_09334_b200 import sim
    wc = {"large_world": workloads.large_world(), "paper_scale": workloads.paper_scale()}[a.config]
    stream = torch.cuda.Stream()
    res = {"workload": wc.name, "warmup": a.warmup, "timed_steps": a.steps,
           "assumed_barrier_us": {"neighbour": a.nbr_us, "allreduce": a.all_us}, "bands": []}
    with torch.cuda.stream(stream):
        w1 = sim.World(wc, stream=stream)
        w1.step(a.warmup)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record(stream)
        w1.step(a.steps)
        ev[1].record(stream)
        torch.cuda.synchronize()
        t1 = ev[0].elapsed_time(ev[1]) / a.steps
        st = w1.get_state(("alive", "cell"))
        w1.step(a.steps)  # the window the banded phase timing replays
        log1 = w1.step_log(a.warmup, 2 * a.steps)[:, 0]
        w1.destroy()
    cells = st["cell"][0][st["alive"][0] == 1]
    hist = np.bincount(cells // wc.cols, minlength=wc.rows)
    res["T1_ms"] = t1
    res["agents"] = int(log1["agents_at_start"].mean())
    for G in (int(g) for g in a.gs.split(",")):
        for kind in ("equal", "weighted"):
            rows = [int(b * wc.rows // G) for b in range(G + 1)] if kind == "equal" else weighted_rows(hist, G)
            per_band = [int(hist[rows[b]:rows[b + 1]].sum()) for b in range(G)]
            slots = int(min(wc.slots, max(per_band) * 1.5 + 4096))  # (the band's pool; the cap is global)
            with torch.cuda.stream(stream):
                wb = sim.World(wc, stream=stream, bands=dict(n_bands=G, band_rows=rows, band_slots=min(slots, wc.slots)))
                wb.step(a.warmup)
                # graph mode: the G bands' whole steps as one CUDA graph per step, bands one
                # after the other (what a graph-captured per-GPU step spends, summed over bands)
                ev[0].record(stream)
                wb.step(a.steps)
                ev[1].record(stream)
                torch.cuda.synchronize()
                tg = ev[0].elapsed_time(ev[1]) / a.steps
                ph = np.zeros((G, len(sim.BAND_PHASES)))
                for _ in range(a.steps):
                    ph += wb.band_step_timed()
                ph /= a.steps
                lb = wb.step_log(a.warmup, 2 * a.steps)[:, 0]
                wb.destroy()
            assert np.array_equal(lb, log1), "banded records differ from the unbanded world"
            slowest = ph.max(axis=0)
            # the P rows (prep_p) run on a second stream from the end of the band's policy on,
            # beside every later phase
            ip, ipol = sim.BAND_PHASES.index("prep_p"), sim.BAND_PHASES.index("policy")
            rest = float(slowest[ipol + 1:].sum() - slowest[ip])
            compute = float(slowest[:ipol + 1].sum() + max(rest, slowest[ip]))
            barriers = (5 * a.nbr_us + a.all_us) / 1e3  # 5 neighbour barriers, 1 all-reduce per step
            est = compute + barriers
            # graph estimate: the mean band step inside the one-GPU graph (T_graph / G), scaled by
            # the slowest band's share of the event-timed band totals (the imbalance)
            tot = ph.sum(axis=1)
            est_g = tg / G * float(tot.max() / tot.mean()) + barriers
            res["bands"].append({
                "G": G, "rows": kind, "band_rows": rows, "agents_per_band": per_band, "band_slots": slots,
                "phase_ms_slowest_band": dict(zip(sim.BAND_PHASES, slowest.round(5).tolist())),
                "band_total_ms": ph.sum(axis=1).round(5).tolist(),
                "est_step_ms_compute": compute, "est_step_ms": est,
                "est_efficiency": t1 / (G * est), "est_efficiency_compute_only": t1 / (G * compute),
                "graph_step_ms_all_bands": tg, "est_graph_step_ms": est_g,
                "est_graph_efficiency": t1 / (G * est_g),
                "est_graph_efficiency_compute_only": t1 / (G * (est_g - barriers)),
                "records_equal_unbanded": True})
            print(json.dumps(res["bands"][-1]), file=sys.stderr, flush=True)
    txt = json.dumps(res, indent=1)
    if a.out:
        open(a.out, "w").write(txt)
    print(txt)


if __name__ == "__main__":
    main()
