"""The N > 1 path on CPU: world-size-2 gloo process groups (127.0.0.1 rendezvous).

bench.py under torchrun gives each rank an independent share of the work (SURVEY.md §8e:
replicas of the single-world configs, a contiguous slice of the ensemble's worlds) with no
data-path collective; only the timed region's max and the work sums are reduced.  These
tests run that host logic with two gloo ranks, each stepping its shard of a small ensemble
with the oracle, and check that the reduced statistics equal one process stepping every
world (worlds are independent), and that the timing reduction is a max.
"""
import os
import socket
import sys
import tempfile

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import workloads  # noqa: E402

SEEDS = (21, 22, 23, 24, 25)
STEPS = 15


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _shard_stats(seeds):
    """Per-world oracle runs of the tiny config; returns (agent-steps, births, deaths, final pop)."""
    import oracle
    out = np.zeros(4, np.float64)
    for sd in seeds:
        wc = workloads.tiny().replace(seeds=(sd,))
        ow = oracle.OracleWorld(wc, 0)
        for _ in range(STEPS):
            r = ow.step()
            out[0] += r["population"] + r["deaths_energy"] + r["deaths_age"] - r["births"]  # agents at step start
            out[1] += r["births"]
            out[2] += r["deaths_energy"] + r["deaths_age"]
        out[3] += int(ow.state()["alive"].sum())
    return out


def _worker(rank, world_size, port, path):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world_size)
    try:
        red = bench.Reducer(dist, "cpu")
        mine = workloads.ensemble_shard(world_size, rank, SEEDS)
        stats = _shard_stats(mine)
        red.barrier()
        tot = [red.sum(v) for v in stats]
        tmax = red.max(1.0 + rank)  # stands in for each rank's timed region
        n_worlds = red.sum(len(mine))
        if rank == 0:
            np.save(path, np.array(tot + [tmax, n_worlds]))
    finally:
        dist.destroy_process_group()


def _shard_worker(rank, world_size, port, path):
    """The agent-sharded exchange (paper_2302_09334_b200.shard.combine_) on gloo: each rank
    holds the move records of its own slots (zero elsewhere) and its policy counters; after
    the SUM-allreduce every rank holds every slot's record and the world's counters."""
    import torch
    import torch.distributed as dist
    from paper_2302_09334_b200.shard import combine_
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world_size)
    try:
        S = 97
        rng = np.random.default_rng(5)
        full = rng.integers(-2**31, 2**31 - 1, size=(S, 4), dtype=np.int64).astype(np.int32)
        owner = np.arange(S) % world_size
        mine = np.where((owner == rank)[:, None], full, 0).astype(np.int32)
        m = torch.from_numpy(mine.reshape(-1).copy())
        ctr = torch.tensor([10 * (rank + 1), rank], dtype=torch.int64)
        combine_([m, ctr], dist)
        if rank == 0:
            np.save(path, np.concatenate([m.numpy().astype(np.int64), ctr.numpy(), full.reshape(-1).astype(np.int64)]))
    finally:
        dist.destroy_process_group()


def test_agent_sharded_exchange_on_gloo():
    import torch.multiprocessing as mp
    path = os.path.join(tempfile.mkdtemp(), "exchange.npy")
    mp.spawn(_shard_worker, args=(2, _free_port(), path), nprocs=2, join=True)
    got = np.load(path)
    S4 = 97 * 4
    assert np.array_equal(got[:S4], got[S4 + 2:])  # every slot's record on every rank (wraps exactly)
    assert list(got[S4:S4 + 2]) == [30, 1]


def test_ensemble_shards_partition_the_worlds():
    for n in range(1, 9):
        parts = [workloads.ensemble_shard(n, r) for r in range(n)]
        flat = [s for p in parts for s in p]
        assert flat == list(range(100, 164))  # contiguous, disjoint, complete, in order
        sizes = [len(p) for p in parts]
        assert max(sizes) - min(sizes) <= 1
    # bench hands each rank its slice; the single-world configs get one replica per rank
    assert bench.workload("ensemble", 1, 2).seeds == tuple(range(132, 164))
    assert bench.workload("paper_scale", 3, 8).seeds == (4,)


def test_reducer_without_dist_is_identity():
    red = bench.Reducer()
    red.barrier()
    assert red.max(2.5) == 2.5 and red.sum(3.0) == 3.0


def test_two_gloo_ranks_reduce_to_the_single_process_result():
    import torch.multiprocessing as mp
    path = os.path.join(tempfile.mkdtemp(), "reduced.npy")
    mp.spawn(_worker, args=(2, _free_port(), path), nprocs=2, join=True)
    got = np.load(path)
    want = _shard_stats(SEEDS)
    assert np.array_equal(got[:4], want), (got, want)
    assert got[4] == 2.0  # max over ranks, not the sum
    assert got[5] == len(SEEDS)


# ------------------------------------------------------------- banded mode (E.2) host logic
def _band_worker(rank, world_size, port, path):
    """Each rank holds its band's share of one world (paper_2302_09334_b200.banded.split_state,
    the layout sim_get_state returns for a band); gathered over gloo, rank 0 merges them."""
    import torch.distributed as dist
    from paper_2302_09334_b200 import banded
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world_size)
    try:
        wc = workloads.tiny().replace(rows=24, cols=40, slots=300)
        full = workloads.random_state(wc, seed=11, n_alive=180, t=7)
        rows = banded.agent_weighted_rows(full["cell"][full["alive"] == 1] // wc.cols, wc.rows, world_size)
        mine = banded.split_state(full, rows, rank, wc.cols)
        parts = [None] * world_size
        dist.all_gather_object(parts, mine)
        if rank == 0:
            merged = banded.merge_band_states(parts, rows, wc.cols)
            np.save(path, np.array([_same_by_cell(full, merged), int(mine["alive"].sum()),
                                    int(parts[1]["alive"].sum())]))
    finally:
        dist.destroy_process_group()


def _same_by_cell(a, b) -> int:
    if a["t"] != b["t"] or not np.array_equal(a["resources"], b["resources"]):
        return 0
    la, lb = np.flatnonzero(a["alive"] == 1), np.flatnonzero(b["alive"] == 1)
    ma, mb = dict(zip(a["cell"][la].tolist(), la)), dict(zip(b["cell"][lb].tolist(), lb))
    if ma.keys() != mb.keys():
        return 0
    for c in ma:
        for f in ("energy", "age", "repr", "last_action", "ate", "h", "c", "weights", "logits"):
            if not np.array_equal(a[f][ma[c]], b[f][mb[c]]):
                return 0
    return 1


def test_banded_states_split_and_merge_on_gloo():
    import torch.multiprocessing as mp
    path = os.path.join(tempfile.mkdtemp(), "banded.npy")
    mp.spawn(_band_worker, args=(2, _free_port(), path), nprocs=2, join=True)
    same, n0, n1 = np.load(path)
    assert same == 1 and n0 + n1 == 180 and abs(int(n0) - int(n1)) <= 40  # agent-weighted rows


def test_band_rows_helpers():
    from paper_2302_09334_b200 import banded
    assert banded.equal_band_rows(200, 8) == [0, 25, 50, 75, 100, 125, 150, 175, 200]
    rng = np.random.default_rng(3)
    ys = np.minimum((rng.random(50000) ** 0.5 * 1600).astype(int), 1599)  # more agents lower down
    for G in (2, 4, 8):
        rows = banded.agent_weighted_rows(ys, 1600, G)
        assert rows[0] == 0 and rows[-1] == 1600 and all(b - a >= 3 for a, b in zip(rows, rows[1:]))
        per = np.bincount(banded.band_of_rows(rows, ys), minlength=G)
        assert per.max() / per.mean() < 1.05  # balanced by agents
    # degenerate: every agent in one row still leaves every band its halo depth
    rows = banded.agent_weighted_rows(np.full(100, 7), 40, 8)
    assert all(b - a >= 3 for a, b in zip(rows, rows[1:])) and rows[-1] == 40
    assert list(banded.band_of_rows([0, 5, 9, 20], [0, 4, 5, 8, 9, 19])) == [0, 0, 1, 1, 2, 2]


def _ens_stats_worker(rank, world_size, port, path):
    """bench.ensemble_end_stats on gloo: each rank fills the rows of its own worlds' seeds
    with their (population, resources); the SUM-reduction leaves every world's row on every
    rank."""
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world_size)
    try:
        seeds = workloads.ensemble().seeds
        mine = workloads.ensemble_shard(world_size, rank)
        recs = [{"population": 1000 + s, "resources": 7 * s} for s in mine]
        st = bench.ensemble_end_stats(seeds, mine, recs, bench.Reducer(dist, "cpu"))
        if rank == 0:
            np.save(path, np.array([st["population_total"], st["resources_total"], st["worlds"]]))
    finally:
        dist.destroy_process_group()


def test_ensemble_end_stats_reduce_over_two_gloo_ranks():
    import torch.multiprocessing as mp
    path = os.path.join(tempfile.mkdtemp(), "ens.npy")
    mp.spawn(_ens_stats_worker, args=(2, _free_port(), path), nprocs=2, join=True)
    got = np.load(path)
    seeds = workloads.ensemble().seeds
    assert list(got) == [sum(1000 + s for s in seeds), sum(7 * s for s in seeds), 64]
