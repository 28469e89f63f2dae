#!/usr/bin/env python
"""Benchmark of the world step (BASELINE.json metric: agent-steps/s and grid cell-updates/s
per world step, % of the B200 HBM roofline) on the paper-scale world (configs[1]).

One bench "step" is one world step: regrowth, observation, per-agent LSTM + argmax,
movement/consumption/physiology, death/reproduction/mutation (all of SURVEY.md §8(a)).

Our arm (default):
  * creates the configs[1] world (200x400, 8192 slots, 1000 agents, 7x7x2 obs, Hd 32,
    seed 1; under torchrun rank r runs an independent replica with seed 1 + r, weak
    scaling, no data-path collective), runs W warm-up steps, then times EXACTLY K steps
    through sim_step (one CUDA graph per step), each bracketed by CUDA events on the
    library's stream, with L2 flushed between timed steps: a 256 MiB memset (evicts every
    line the step left) followed by a 256 MiB read, so the evicted lines are clean and the
    next step is not charged for writing back the flush buffer's dirty lines;
  * replays the same K steps from a snapshot twice, L2 flushed between steps: through
    sim_step_timed (the phases as separate kernels, events around each) for the per-kernel
    breakdown, and through sim_step_graph_timed (the graph's own two kernels launched
    directly, events between them) for `roofline` (the longer of the two, at its
    algorithmic bytes; `traffic` from the newest profiles/*_ncu_summary.json of the same
    workload) and `kernels_roofline`; both replays must reproduce the timed run's records;
  * e2e: the same K steps through the public API from pinned HOST buffers: sim_set_state
    (H2D of the whole state), then sim_step(K) (one call), each step's record written by the
    device into a mapped pinned host ring (sim_set_record_mirror: the D2H of the result
    without a copy operation), wall clock, checked equal to the timed run's records; the
    sim_step(K) call alone is also bracketed by CUDA events (`one_call`: SURVEY.md D.4's
    procedure, no per-step event pair or L2 flush);
  * whole_run_sample (when K covers only the first steps of the config's 10,000-step run,
    as the driver's --steps 20 does): 20 more single steps spread evenly over the rest of the
    run, timed the same way, the steps between them advanced untimed;
  * cpu_baseline: the oracle (oracle/, single thread) on a bounded sample of the same
    workload from the same start state.
--impl reference: the oracle as the reference arm (no GPU code on that path).
"""
import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import workloads  # noqa: E402

METRIC = "agent-steps/s (paper-scale world step)"
UNIT = "agent-steps/s"
FLUSH_BYTES = 256 << 20
RUN_SAMPLES = 20  # whole_run_sample: single steps timed over the rest of the run


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10000)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", default="paper_scale", choices=("paper_scale", "tiny", "large_world", "ensemble", "paper_world",
                                                                   "paper_world_cnn", "paper_world_coloc"))
    ap.add_argument("--cpu-budget-s", type=float, default=15.0)
    ap.add_argument("--ref-budget-s", type=float, default=120.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-replay", action="store_true")
    ap.add_argument("--no-run-sample", action="store_true",
                    help="skip whole_run_sample (steps sampled over the rest of the config's run)")
    ap.add_argument("--shard", action="store_true",
                    help="one world over all ranks (agent-sharded, NCCL allreduce of the move records "
                         "each step; strong scaling) instead of one replica per rank")
    ap.add_argument("--no-flush", action="store_true",
                    help="diagnostic: do not flush L2 between timed steps (the line says so in config.l2)")
    ap.add_argument("--no-l2-persist", action="store_true",
                    help="ablation: no L2-persisting window on the hot-state arena (ECO_L2_PERSIST=0)")
    ap.add_argument("--out", default=None, help="also write the JSON line to this file")
    ap.add_argument("--cpu-baseline-suite", default=None, metavar="OUT",
                    help="run the oracle's CPU baseline of BASELINE.md section 3 on every config, write OUT, exit")
    ap.add_argument("--quick", action="store_true", help="(with --cpu-baseline-suite) fewer steps")
    return ap.parse_args()


def workload(name: str, rank: int, world_size: int = 1) -> workloads.WorldConfig:
    """The rank's share of the workload: one independent replica per rank (seed + rank) for
    the single-world configs, a contiguous slice of the ensemble's worlds for `ensemble`
    (weak scaling for the former, the ensemble's worlds split for the latter)."""
    if name == "paper_scale":
        wc = workloads.paper_scale()
        return wc.replace(seeds=(wc.seeds[0] + rank,))
    if name == "tiny":
        return workloads.tiny().replace(seeds=(rank,))
    if name == "large_world":
        return workloads.large_world().replace(seeds=(3 + rank,))
    if name in ("paper_world", "paper_world_cnn", "paper_world_coloc"):  # the paper's world, agents, reproduction
        wc = getattr(workloads, name)()
        return wc.replace(seeds=(wc.seeds[0] + rank,))
    return workloads.ensemble().replace(seeds=tuple(workloads.ensemble_shard(world_size, rank)))


class Reducer:
    """Cross-rank reductions of the bench (max of the timed region, sums of work units);
    identity without torch.distributed.  `device` is where the gloo/nccl tensors live."""

    def __init__(self, dist=None, device="cpu"):
        self.dist, self.device = dist, device

    def barrier(self):
        if self.dist is not None:
            self.dist.barrier()

    def _all(self, v: float, op) -> float:
        if self.dist is None:
            return float(v)
        import torch
        t = torch.tensor([float(v)], dtype=torch.float64, device=self.device)
        self.dist.all_reduce(t, op=op)
        return float(t.item())

    def max(self, v: float) -> float:
        return self._all(v, None if self.dist is None else self.dist.ReduceOp.MAX)

    def sum(self, v: float) -> float:
        return self._all(v, None if self.dist is None else self.dist.ReduceOp.SUM)

    def sum_array(self, a: np.ndarray) -> np.ndarray:
        """Element-wise int64 SUM over ranks (NCCL on the device / gloo on the CPU)."""
        if self.dist is None:
            return np.asarray(a, np.int64).copy()
        import torch
        t = torch.from_numpy(np.ascontiguousarray(a, np.int64)).to(self.device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)
        return t.cpu().numpy()


def ensemble_end_stats(seeds_all, seeds_mine, last_records, red: Reducer) -> dict:
    """SURVEY.md §8(e) E.1 / north_star (ii): the only cross-GPU traffic of the ensemble, its
    end-of-run statistics -- each world's population and resource total after the run, placed
    in the row of its seed (zero rows elsewhere) and SUM-reduced over the ranks."""
    idx = {s: k for k, s in enumerate(seeds_all)}
    tab = np.zeros((len(seeds_all), 2), np.int64)
    for s, rec in zip(seeds_mine, last_records):
        tab[idx[s]] = (int(rec["population"]), int(rec["resources"]))
    tab = red.sum_array(tab)
    return {"worlds": len(seeds_all), "population_total": int(tab[:, 0].sum()),
            "resources_total": int(tab[:, 1].sum()), "population_min_max": [int(tab[:, 0].min()), int(tab[:, 0].max())],
            "extinct_worlds": int((tab[:, 0] == 0).sum()), "per_world": tab.tolist()}


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            mp = json.load(f)
        return float(mp["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    REASONS = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-i", str(self.device), "-lms", "200"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, smax, reasons = [], [], set()
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for name, val in zip(self.REASONS, parts[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------------- bytes model
def split_policy(wc) -> bool:
    """Whether the library splits the gate sum (api.cu: one world, hidden 32): the P rows
    P = W_hh h + b are made beside the dynamics and the policy reads them."""
    return wc.n_worlds == 1 and wc.hidden == 32


def policy_bytes(wc, agents: int, nnz: int, split: bool = None) -> int:
    """Algorithmic bytes of the policy kernel: the W_ih
    columns of active inputs, W_out, b_out, h and c read+written, 32 B of SoA fields and
    claims per agent, and either W_hh and b (unsplit) or the agent's P row (split)."""
    Hd = wc.hidden
    if getattr(wc, "network", 0) == 1:
        # the paper's CNN-LSTM (k_policy_cnn_blk): every agent reads its whole parameter row
        # (2445 floats), h and c read and written, 32 B of SoA fields and the claim
        return agents * (4 * wc.n_params + 16 * Hd + 32)
    split = split_policy(wc) if split is None else split
    rec = 4 * 4 * Hd if split else 4 * (4 * Hd * Hd + 4 * Hd)
    per_agent_fixed = rec + 4 * (5 * Hd + 5) + 16 * Hd + 32
    return 4 * 4 * Hd * nnz + agents * per_agent_fixed


def hh_bytes(wc, agents: int) -> int:
    """Algorithmic bytes of the P rows (split policy): W_hh and b read, h read, P written."""
    Hd = wc.hidden
    return agents * (4 * (4 * Hd * Hd + 4 * Hd) + 4 * Hd + 4 * 4 * Hd)


def post_bytes(wc, agents: int, births: int) -> int:
    """Algorithmic bytes of the cooperative k_post launch: (split) the P rows of the agents
    alive at the step's start (hh_bytes), the R and O bit planes read and written (H*W/2 B),
    the mutation (parent's P weights read, child's written: 8P per birth) and 64 B of
    per-agent dynamics state (move record, energy/age/repr read and written, list entry)."""
    hh = hh_bytes(wc, agents) if split_policy(wc) else 0
    return hh + wc.rows * wc.cols // 2 + births * 8 * wc.n_params + 64 * agents


def step_bytes(wc, agents: int, nnz: int, births: int) -> int:
    """Whole-step algorithmic bytes: B_agent per live agent (the unsplit
    policy's bytes: active W_ih columns, W_hh, b, W_out, b_out, h and c, 32 B of SoA) + the R
    and O bit planes read and written (H*W/2 B) + 8P per birth (parent read, child written).
    The split design's extra P-row traffic (written by k_post, read by the policy: ~1.2 KB
    per agent) is not counted: it is this implementation's cost, not the method's."""
    return policy_bytes(wc, agents, nnz, split=False) + wc.rows * wc.cols // 2 + births * 8 * wc.n_params


def workload_config(wc, args, world_size: int, sharded: bool, t0: int) -> dict:
    """The `config` object of both arms' JSON lines (the same workload, the same dict)."""
    return {"workload": f"{wc.name} (BASELINE.json configs[1])" if args.config == "paper_scale" else wc.name,
            "grid": f"{wc.rows}x{wc.cols}", "slots": wc.slots, "n_initial": wc.n_initial,
            "obs": f"{2 * wc.obs_radius + 1}x{2 * wc.obs_radius + 1}x{3 if getattr(wc, 'network', 0) else 2}",
            "hidden": wc.hidden,
            "network": "paper CNN-LSTM, sampled (PAPER.md:346-350)" if getattr(wc, "network", 0)
            else "LSTM + linear head, argmax",
            "seed": int(wc.seeds[0]), "n_worlds": wc.n_worlds, "timed_steps": [t0, t0 + args.steps],
            "parallelism": (f"agent-sharded: one world over {world_size} GPUs (policy by slot owner, "
                            "dynamics on every rank, NCCL SUM-allreduce of the move records per step)")
            if sharded else "replicas (one independent world per GPU, seed 1+rank)" if world_size > 1
            else "single device", "global_batch": wc.slots * (1 if sharded else world_size)}


# ------------------------------------------------------------------------ our arm
def run_ours(args, rank, world_size, local_rank):
    if args.no_l2_persist:
        os.environ["ECO_L2_PERSIST"] = "0"
    import torch
    from paper_2302_09334_b200 import sim

    dist = None
    if world_size > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    sharded = args.shard and world_size > 1
    wc = workload(args.config, 0 if args.shard else rank, world_size)  # --shard: the same world everywhere
    if sharded:  # state capture and the instrumented replay are per-rank views: skip them
        args.no_replay = args.no_e2e = args.no_cpu_baseline = True
    K, W = args.steps, args.warmup
    stream = torch.cuda.Stream(device=dev)
    red = Reducer(dist, dev)
    barrier, allmax, allsum = red.barrier, red.max, red.sum

    with torch.cuda.stream(stream):
        if sharded:
            from paper_2302_09334_b200.shard import ShardedWorld
            world = ShardedWorld(wc, dist, local_rank, stream=stream, log_capacity=max(4096, W + K + 8))
        else:
            world = sim.World(wc, device=local_rank, stream=stream, log_capacity=max(4096, W + K + 8))
        flush = torch.empty(FLUSH_BYTES, dtype=torch.uint8, device=dev)
        flush_rd = torch.ones(FLUSH_BYTES // 4, dtype=torch.float32, device=dev)

        def flush_l2():
            flush.zero_()
            flush_rd.sum()  # clean lines: no dirty write-back lands in the timed step

        # the flush's first call allocates the reduction's output (a new device mapping): made
        # here, not before the first timed step (it cost that step 10-30 us, measured)
        flush_l2()
        world.step(W)
        world.synchronize()
        world.phase_ns(reset=True)  # the phase clocks cover the timed steps only
        need_snap = not (args.no_replay and args.no_e2e and args.no_cpu_baseline)
        snap = world.get_state() if need_snap else None
        t0 = world.t
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        clocks = ClockSampler(local_rank)
        clocks.start()
        barrier()
        torch.cuda.synchronize()
        for k in range(K):
            if not args.no_flush:
                flush_l2()
            evs[k][0].record(stream)
            world.step(1)
            evs[k][1].record(stream)
        torch.cuda.synchronize()
        barrier()
        clk = clocks.stop()
        world.synchronize()
        post_phases = {k_: v / K / 1e3 for k_, v in world.phase_ns().items()}
        for k_ in [k_ for k_ in post_phases if k_.startswith("reserved")]:
            post_phases.pop(k_)
        step_ms = np.array([a.elapsed_time(b) for a, b in evs], np.float64)
        total_ms = float(step_ms.sum())
        log = world.step_log(t0, K)
        agents = int(log["agents_at_start"].sum())
        nnz = int(log["obs_nnz"].sum())
        births = int(log["births"].sum())
        max_ms = allmax(total_ms)
        ens_stats = (ensemble_end_stats(workloads.ensemble().seeds, wc.seeds, log[-1], red)
                     if args.config == "ensemble" else None)
        all_agents = agents if sharded else allsum(agents)  # sharded: one world, counted once
        value = all_agents / (max_ms / 1e3)
        cells = K * wc.rows * wc.cols * wc.n_worlds

        # -- replay of the same K steps with per-kernel events
        kern = None
        if not args.no_replay:
            world.set_state(snap)
            ksum = np.zeros(sim.NUM_KERNELS)
            ssum = 0.0
            for k in range(K):
                if not args.no_flush:
                    flush_l2()
                tm = world.step_timed()
                ksum += np.array([tm[n] for n in sim.KERNEL_NAMES])
                ssum += tm["step_ms"]
            log2 = world.step_log(t0, K)
            replay_identical = bool(np.array_equal(log2, log))
            # the graph path's own two kernels, launched directly with events between them
            world.set_state(snap)
            gsum = np.zeros(2)
            for k in range(K):
                if not args.no_flush:
                    flush_l2()
                tg = world.step_graph_timed()
                gsum += (tg["policy"], tg["post"])
            log3 = world.step_log(t0, K)
            kern = {"kernel_ms_total": dict(zip(sim.KERNEL_NAMES, ksum.tolist())), "step_ms_total": ssum,
                    "replay_identical": replay_identical and bool(np.array_equal(log3, log)),
                    "graph_kernel_ms_total": {"policy": gsum[0], "post": gsum[1]}}

        # -- e2e through the public API from pinned host buffers
        e2e = None
        if not args.no_e2e:
            pinned = {}
            h2d = 0
            n_live = int(snap["alive"].sum())
            for k_, v in snap.items():
                if isinstance(v, np.ndarray):
                    tt = torch.empty(v.shape, dtype=getattr(torch, str(v.dtype)), pin_memory=True)
                    tt.numpy()[...] = v
                    pinned[k_] = tt.numpy()
                    # the library reads the live slots' weights only (a dead slot's weights are
                    # unspecified, sim.h), every other field whole
                    h2d += n_live * wc.n_params * 4 if k_ == "weights" else v.nbytes
                else:
                    pinned[k_] = v
            rec_bytes = sim.RECORD_DTYPE.itemsize * wc.n_worlds
            # every step's record is written by the device into a mapped pinned host ring as
            # the step completes (sim_set_record_mirror): no copy operation per step
            cap = 1 << (K - 1).bit_length()
            rec_pin = torch.empty((cap, rec_bytes), dtype=torch.uint8, pin_memory=True).numpy()
            rec_host = rec_pin.view(sim.RECORD_DTYPE).reshape(cap, wc.n_worlds)
            world.set_record_mirror(rec_host, cap)  # (re-captures both step graphs at once)
            world.synchronize()
            torch.cuda.synchronize()
            barrier()
            ev_a, ev_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            te = time.perf_counter()
            world.set_state(pinned)
            ev_a.record(stream)
            world.step(K)  # the user's call: K steps in one sim_step (eight-step graphs)
            ev_b.record(stream)
            world.synchronize()
            e_s = time.perf_counter() - te
            call_ms = allmax(ev_a.elapsed_time(ev_b))  # the one sim_step(K) call alone, on the device
            world.set_record_mirror(None)
            got = rec_host[(np.arange(t0, t0 + K) & (cap - 1))]
            assert np.array_equal(got, log), "e2e records differ from the timed run"
            e_s = allmax(e_s)
            e2e = {"value": all_agents / e_s, "unit": UNIT, "h2d_bytes_per_step": h2d / K,
                   "d2h_bytes_per_step": rec_bytes, "seconds": e_s, "step_call_device_ms": call_ms}
        # -- the rest of the config's run, sampled: when K covers only the run's first steps (the
        # driver's --steps 20 times t = 5..25, ~1,000 agents in 8,192 slots), M more single
        # steps spread evenly over the remaining steps of the run are timed the same way (L2
        # flush, events around one sim_step(1)), the steps between them advanced untimed
        run_sample = None
        if (not sharded and not args.no_run_sample and args.config == "paper_scale" and world.t == t0 + K
                and wc.steps - world.t >= 40 * RUN_SAMPLES):
            stride = (wc.steps - world.t) // RUN_SAMPLES
            s_ms, s_t, s_agents, s_bytes = [], [], 0, 0
            ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            for i in range(RUN_SAMPLES):
                world.step(stride - 1)
                flush_l2()
                ea.record(stream)
                world.step(1)
                eb.record(stream)
                world.synchronize()
                r = world.step_log(world.t - 1, 1)
                s_t.append(int(world.t - 1))
                s_ms.append(ea.elapsed_time(eb))
                s_agents += int(r["agents_at_start"].sum())
                s_bytes += step_bytes(wc, int(r["agents_at_start"].sum()), int(r["obs_nnz"].sum()),
                                      int(r["births"].sum()))
            run_sample = {"t": s_t, "step_ms": s_ms, "agents": s_agents, "bytes": s_bytes,
                          "max_ms": allmax(float(sum(s_ms))), "all_agents": allsum(s_agents)}
        world.destroy()

    result = None
    if rank == 0:
        peak, peak_src = peaks()
        result = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world_size, "steps": K, "warmup": W,
            "ms_per_step": max_ms / K, "higher_is_better": True, "scaling": "strong" if sharded else "weak",
            "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": workload_config(wc, args, world_size, sharded, t0),
            "l2": ("NOT flushed (diagnostic run)" if args.no_flush
                   else "flushed between timed steps (256 MiB memset + 256 MiB read on the library stream)")
            + ("" if args.no_l2_persist else "; the step graph's kernels mark the library's hot-state arena "
               "(counters, planes, lists, SoA, P rows, h, c, claims: everything but the weights, first 32 MiB) "
               "L2-persisting, so the flush cannot evict it; the weights stream from HBM every step"),
            "cell_updates_per_s": cells * (1 if sharded else world_size) / (max_ms / 1e3),
            "agents_mean": agents / K,
            **({"ensemble_end_stats": {k_: v_ for k_, v_ in ens_stats.items() if k_ != "per_world"}}
               if ens_stats else {}),
            # the paper's own timing is of its own world with its own network (1e6
            # steps in ~20 min on an unnamed GPU with JAX, ~833 world steps/s): context for the
            # paper-world configs, not vs_baseline (BASELINE.json publishes no number)
            **({"vs_paper": {"world_steps_per_s": 1e3 / (max_ms / K), "paper_world_steps_per_s": 833.0,
                             "ratio": 1e3 / (max_ms / K) / 833.0,
                             "note": "PAPER.md:340, unnamed GPU, JAX; context only"}}
               if args.config in ("paper_world_cnn", "paper_world_coloc") else {}),
            "births_mean": births / K,
            "gpu_launches": 2 * K,  # per rank: the policy kernel and the cooperative k_post
            "post_phase_us_per_step": post_phases,
            "clocks": clk,
        }
        if not sharded and wc.slots > 0:  # (from the records alone: no replay needed)
            sb = step_bytes(wc, agents, nnz, births)
            result["step_roofline"] = {"bytes_per_step": sb / K, "achieved_GBps": sb / (max_ms / 1e3) / 1e9,
                                       "frac": sb / (max_ms / 1e3) / 1e9 / peak,
                                       "dense_equiv_GBps": step_bytes(wc, agents, agents * wc.n_inputs, births)
                                       / (max_ms / 1e3) / 1e9}
        if kern is not None:
            ks = kern["kernel_ms_total"]
            sb = step_bytes(wc, agents, nnz, births)
            # the graph path's two kernels (events around each, same launches as the graph);
            # the roofline line is the one with the larger time.  The instrumented replay's
            # standalone P-row kernel (k_prepare_p) is reported beside them.
            gk = kern["graph_kernel_ms_total"]
            gstep = gk["policy"] + gk["post"]
            cands = {
                "policy": (("k_policy_cnn_blk (15x15x3 window + the paper's CNN-LSTM + softmax sampling + move claim)"
                            if getattr(wc, "network", 0) else
                            "k_policy_half (observe + LSTM gates from P + argmax + move claim)" if wc.hidden == 32 else
                            f"k_policy_reg<{wc.hidden}> (observe + LSTM + argmax + move claim)"),
                           policy_bytes(wc, agents, nnz), gk["policy"], gstep),
                "post": ("k_post (move/consume/physiology/death, birth claims + rank + placement, regrowth, "
                         "mutation; P rows of the next step on 4 warps per block)",
                         post_bytes(wc, agents, births), gk["post"], gstep)}
            if split_policy(wc):
                cands["hh"] = ("k_prepare_p (standalone P rows in the instrumented replay; inside k_post in graph mode)",
                               hh_bytes(wc, int(log["population"].sum())), ks["hh"], kern["step_ms_total"])
            rl = {}
            for kname, (desc, byt, ms, step_ms_tot) in cands.items():
                achieved = byt / (ms / 1e3) / 1e9
                ratio, ratio_src = traffic_ratio(kname, wc.name, agents / K)
                rl[kname] = {
                    "kernel": desc, "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": achieved / peak, "traffic": ratio * byt / K if ratio else None,
                    "traffic_source": ratio_src, "bytes_per_launch": byt / K, "launch_ms": ms / K,
                    "peak_source": peak_src, "share_of_step": ms / step_ms_tot}
            dom = max(("policy", "post"), key=lambda k_: rl[k_]["launch_ms"])
            result["roofline"] = rl[dom]
            result["kernels_roofline"] = rl
            result["kernel_ms_per_step"] = {k: v / K for k, v in ks.items()}
            result["graph_kernel_ms_per_step"] = {k: v / K for k, v in kern["graph_kernel_ms_total"].items()}
            result["replay_identical"] = kern["replay_identical"]
        if e2e is not None:
            result["e2e"] = e2e
            # SURVEY.md §8(d) D.4's procedure beside the per-step one: the K steps as ONE sim_step(K)
            # call bracketed by CUDA events (no event pair, graph-launch gap or L2 flush per step;
            # the records still mirrored to the host), and D.3c's run-level fraction of it
            cms = e2e["step_call_device_ms"]
            sb_run = step_bytes(wc, agents, nnz, births)
            result["one_call"] = {
                "what": "the same K steps as one sim_step(K) call, CUDA events around the call (SURVEY.md D.4); "
                        "L2 not flushed between its steps",
                "ms_per_step": cms / K, "value": all_agents / (cms / 1e3), "unit": UNIT,
                "step_roofline": {"bytes_per_step": sb_run / K, "achieved_GBps": sb_run / (cms / 1e3) / 1e9,
                                  "frac": sb_run / (cms / 1e3) / 1e9 / peak}}
        if run_sample is not None:
            rs = run_sample
            result["whole_run_sample"] = {
                "what": f"{RUN_SAMPLES} single steps spread evenly over the rest of the config's {wc.steps}-step run "
                        "(each after an L2 flush, events around one sim_step(1); the steps between advanced "
                        "untimed): the run's regimes beside the timed region's first steps",
                "t": rs["t"], "ms_per_step": rs["max_ms"] / RUN_SAMPLES,
                "value": rs["all_agents"] / (rs["max_ms"] / 1e3), "unit": UNIT,
                "agents_mean": rs["agents"] / RUN_SAMPLES,
                "step_roofline": {"bytes_per_step": rs["bytes"] / RUN_SAMPLES,
                                  "achieved_GBps": rs["bytes"] / (sum(rs["step_ms"]) / 1e3) / 1e9,
                                  "frac": rs["bytes"] / (sum(rs["step_ms"]) / 1e3) / 1e9 / peak},
                "step_us": [round(v * 1e3, 2) for v in rs["step_ms"]]}
    return result, snap, wc


def traffic_ratio(kname="policy", workload="paper_scale", agents=None):
    """DRAM bytes (read + write) over algorithmic bytes of the kernel's launch (policy: the
    k_policy launch; hh: k_prepare_p) in a committed ncu --set full summary
    (profiles/<generation>_*_ncu_summary.json, tools/ncu_summary.py): of the newest
    generation (the name's prefix, e.g. r2a) that captured this workload, the capture whose
    live-agent count is closest to the bench's mean; the roofline's `traffic` is this ratio
    times the bench's algorithmic bytes per launch (the captured launch is one step of the
    same workload, not the bench's own launches)."""
    tag = {"policy": "k_policy", "hh": "k_prepare_p", "post": "k_post"}[kname]
    import glob
    found = []
    for f in glob.glob(os.path.join(ROOT, "profiles", "*_ncu_summary.json")):
        try:
            d = json.load(open(f))
            st = d.get("step", {})
            if st.get("workload", "paper_scale") != workload:
                continue  # a capture of another workload
            for rec in d["launches"]:
                if tag in rec["kernel"] and "traffic_over_algorithmic" in rec:
                    gen = os.path.basename(f).split("_")[0]
                    dist = abs(st.get("agents", 0) - agents) if agents is not None else 0
                    found.append((gen, -dist, float(rec["traffic_over_algorithmic"]), os.path.relpath(f, ROOT)))
                    break
        except Exception:
            continue
    if not found:
        return None, None
    best = max(found)
    return best[2], best[3]


# -------------------------------------------------------------- oracle (CPU) legs

# ----------------------------------------------------- the CPU baseline suite
# `bench.py --cpu-baseline-suite OUT`: the oracle (oracle/, single-threaded C99) on the host CPU
# of the GPU box per config, reported like the GPU numbers (agent-steps/s, cell-updates/s,
# wall time; CPU model, 1 core per process, nproc): tiny all 100 steps; paper-scale the
# first 200; regrowth 1000 steps at 200x400, 100 at 2048x4096, 10 at 8192x16384; the large
# world extrapolated (its canonical state would hold 17.8 GB of weights); the ensemble as one
# world and as one world per host core in separate processes; the paper's own world with
# the paper's network and reproduction beside the paper's ~833 world steps/s.
def _suite_host() -> dict:
    model = None
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count(), "cpus_usable": len(os.sched_getaffinity(0))}


def _suite_world(wc, steps, world=0):
    t0 = time.perf_counter()
    import oracle
    w = oracle.OracleWorld(wc, world)
    t_init = time.perf_counter() - t0
    agents = 0
    t0 = time.perf_counter()
    for _ in range(steps):
        agents += int(w.st["alive"].sum())
        r = w.step()
        assert r["status"] == 0
    el = time.perf_counter() - t0
    return {"steps": steps, "wall_s": el, "init_s": t_init, "agent_steps": agents,
            "agent_steps_per_s": agents / el, "cell_updates_per_s": wc.rows * wc.cols * steps / el,
            "world_steps_per_s": steps / el, "mean_agents": agents / steps}


def _suite_regrow(rows, cols, steps):
    import oracle
    wc = workloads.regrowth_micro(rows, cols)
    R = oracle.OracleWorld(wc).st["resources"].copy()
    t0 = time.perf_counter()
    for t in range(steps):
        R, _ = oracle.regrow(wc, t, R)
    el = time.perf_counter() - t0
    return {"grid": f"{rows}x{cols}", "steps": steps, "wall_s": el, "us_per_step": el / steps * 1e6,
            "cell_updates_per_s": rows * cols * steps / el}


def _suite_ens_worker(args):
    seed, steps = args
    wc = workloads.ensemble(seeds=(seed,))
    return _suite_world(wc, steps)


def cpu_baseline_suite(out: str, q: bool = False) -> dict:
    import multiprocessing as mp
    res = {"kind": "oracle", "cores_per_process": 1, **_suite_host(), "configs": {}}
    res["configs"]["tiny"] = _suite_world(workloads.tiny(), 20 if q else 100)
    res["configs"]["paper_scale"] = _suite_world(workloads.paper_scale(), 20 if q else 200)
    res["configs"]["regrowth_micro"] = [_suite_regrow(200, 400, 100 if q else 1000),
                                        _suite_regrow(2048, 4096, 5 if q else 100),
                                        _suite_regrow(8192, 16384, 1 if q else 10)]
    ps = res["configs"]["paper_scale"]
    per_agent = ps["wall_s"] / ps["agent_steps"]  # (the LSTM dominates: the cell cost is folded in)
    lw = workloads.large_world()
    res["configs"]["large_world"] = {
        "run": False, "why": "the oracle's canonical state would hold 17.8 GB of fp32 weights",
        "extrapolated_s_per_step_at_cap": per_agent * lw.slots,
        "extrapolated_agent_steps_per_s": 1.0 / per_agent}
    steps = 20 if q else 200
    one = _suite_world(workloads.ensemble(seeds=(100,)), steps)
    ncores = min(res["cpus_usable"], 32)  # (each process holds a 555 MB world)
    seeds = [100 + (k % 64) for k in range(ncores)]
    t0 = time.perf_counter()
    with mp.get_context("fork").Pool(ncores) as pool:
        outs = pool.map(_suite_ens_worker, [(s, steps) for s in seeds])
    el = time.perf_counter() - t0
    agg = sum(o["agent_steps"] for o in outs)
    res["configs"]["ensemble"] = {
        "one_world": one, "one_core_64_worlds_in_sequence_agent_steps_per_s": one["agent_steps_per_s"],
        "per_core_processes": {"processes": ncores, "worlds": len(seeds), "steps_each": steps, "wall_s": el,
                               "agent_steps_per_s": agg / el,
                               "note": "one world per host core, all cores busy (memory bandwidth shared)"}}
    pw = _suite_world(workloads.paper_world_coloc(), 40 if q else 200)
    pw["paper_world_steps_per_s_reported"] = 833.0
    pw["paper_note"] = "PAPER.md:340: 1e6 steps in ~20 min on 'a single GPU' with JAX (model not stated)"
    res["configs"]["paper_world_coloc"] = pw
    open(out, "w").write(json.dumps(res, indent=1))
    return res


def oracle_rate(wc, start_state, budget_s, max_steps):
    import oracle
    w = oracle.OracleWorld(wc, state=start_state)
    agents = 0
    steps = 0
    a0 = int(w.st["alive"].sum())
    t0 = time.perf_counter()
    while steps < max_steps and time.perf_counter() - t0 < budget_s:
        agents += int(w.st["alive"].sum())
        w.step()
        steps += 1
    el = time.perf_counter() - t0
    return agents / el, steps, el, a0, int(w.st["alive"].sum()), w.t


def host_cpu() -> dict:
    """The host CPU the oracle ran on: model name, logical CPUs (nproc) and the CPUs this
    process may use (the oracle itself is single-threaded: cores = 1)."""
    model = None
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    try:
        usable = len(os.sched_getaffinity(0))
    except Exception:
        usable = None
    return {"cpu_model": model, "nproc": os.cpu_count(), "cpus_usable": usable}


def run_reference(args, rank):
    if rank != 0:
        return None
    import oracle
    wc = workload(args.config, 0)
    w = oracle.OracleWorld(wc)
    for _ in range(args.warmup):
        w.step()
    rate, steps, el, a0, a1, t1 = oracle_rate(wc, w.state(), args.ref_budget_s, args.steps)
    sample = (f"oracle world steps t={args.warmup}..{t1} ({steps} of the {args.steps} requested steps, "
              f"bounded to {args.ref_budget_s:.0f} s; agents {a0}->{a1}); rate metric, so comparable")
    return {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": args.gpus,
        "steps": steps, "warmup": args.warmup, "ms_per_step": el / max(steps, 1) * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(wc, args, args.gpus, False, args.warmup),
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample, **host_cpu()},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    args = parse_args()
    if args.cpu_baseline_suite:
        res = cpu_baseline_suite(args.cpu_baseline_suite, args.quick)
        print(json.dumps(res))
        return
    rank = int(os.environ.get("RANK", "0"))
    world_size = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        res = run_reference(args, rank)
        if res is not None:
            line = json.dumps(res)
            print(line, flush=True)
            if args.out:
                open(args.out, "w").write(line + "\n")
        return
    res, snap, wc = run_ours(args, rank, world_size, local_rank)
    if rank == 0:
        if not args.no_cpu_baseline and world_size == 1 and snap is not None:
            w0 = {k: (v[0] if isinstance(v, np.ndarray) else v) for k, v in snap.items()}
            # (a rate: as many oracle steps from the start state as fit the budget, whatever K is —
            # the driver's K = 20 alone would be 0.3 s of CPU work)
            rate, steps, el, a0, a1, t1 = oracle_rate(wc.replace(seeds=(wc.seeds[0],)), w0, args.cpu_budget_s,
                                                      max(args.steps, 100000))
            res["cpu_baseline"] = {
                "value": rate, "unit": UNIT, "cores": 1, "kind": "oracle", **host_cpu(),
                "sample": f"{steps} oracle world steps from the timed region's start state (t={w0['t']}..{t1}, "
                          f"agents {a0}->{a1}), {el:.1f} s on one host core",
            }
        line = json.dumps(res)
        print(line, flush=True)
        if args.out:
            open(args.out, "w").write(line + "\n")
    if world_size > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
