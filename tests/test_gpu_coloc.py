"""GPU parity of co-location (the paper's reproduction on the
parent's cell; any number of agents per cell; R43-R47) with the
paper's network (k_policy_cnn_blk + coloc.cuh) against the oracle, through the C ABI: integer
state, records and slot layout bit-exact, h', c', logits within 1 ulp, the kernel's own
sampled actions equal to the oracle's except at flagged near-ties."""
import numpy as np
import pytest

import oracle
import workloads
from harness import MAX_ULP_SEEN, compare_ints, compare_weights, gpu_world_state, lockstep_sampled

pytestmark = pytest.mark.gpu

sim = pytest.importorskip("paper_2302_09334_b200.sim")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device (no CPU fallback exists)")


def small(**kw):
    base = dict(rows=40, cols=60, slots=300, n_initial=150, repr_steps=20, seeds=(13,))
    base.update(kw)
    return workloads.paper_world_coloc().replace(**base)


def test_coloc_init_matches_oracle():
    wc = workloads.paper_world_coloc()
    with sim.World(wc) as world:
        g = gpu_world_state(world.get_state())
        o = oracle.OracleWorld(wc).state()
        compare_ints(g, o, "init")
        compare_weights(g["weights"], o["weights"], o["alive"] == 1, where="init")


@pytest.mark.parametrize("seed,density", [(1, 0.3), (2, 0.6), (3, 0.1)])
def test_coloc_stacked_random_states_one_step(seed, density):
    """Injected states with agents stacked up to several per cell (cells drawn WITH
    replacement from a small region, borders included), random timers and recurrent state:
    one step -- the counts channel, the lottery on shared resource cells, several children
    on one cell, slot-keyed mutation -- bit-exact."""
    wc = small(rows=30, cols=44, slots=400, seeds=(50 + seed,))
    st = workloads.random_state(wc, seed, n_alive=260, density=density, weight_std=0.3)
    rng = np.random.default_rng(seed)
    live = np.flatnonzero(st["alive"])
    ys = rng.integers(0, 12, live.size)
    xs = rng.integers(0, 16, live.size)
    st["cell"][live] = (ys * wc.cols + xs).astype(np.int32)  # ~1.4 agents per cell of the region
    st["ate"][live] = rng.integers(0, 2, live.size).astype(np.uint8)
    st["energy"][live] = rng.integers(1, 3001, live.size).astype(np.int32)
    st["repr"][live] = rng.integers(0, 2 * wc.repr_steps, live.size).astype(np.int32)
    st["age"] = np.minimum(st["age"], 600).astype(np.int32)
    world = sim.World(wc)
    world.set_state({k: (v[None] if isinstance(v, np.ndarray) else v) for k, v in st.items()})
    orc = oracle.OracleWorld(wc, state=st)
    flips, n, nulp = lockstep_sampled(world, orc, 1, check_weights_every=1)
    rec = world.step_log(st["t"], 1)[0, 0]
    print(f"stacked one step: {n} agents, births {int(rec['births'])}, eaten {int(rec['eaten'])}, "
          f"deferred {int(rec['deferred_capacity'])}, flips {flips}, max ulp {MAX_ULP_SEEN}")
    assert n == 260 and int(rec["births"]) > 0
    world.destroy()


def test_coloc_lockstep_small_world_300_steps():
    wc = small()
    world = sim.World(wc)
    orc = oracle.OracleWorld(wc)
    flips, n, nulp = lockstep_sampled(world, orc, 300, check_weights_every=50)
    log = world.step_log(0, 300)[:, 0]
    st = world.get_state(("alive", "cell"))
    c = np.bincount(st["cell"][0][st["alive"][0] == 1])
    print(f"coloc small world: {n} agent-steps, births {int(log['births'].sum())}, wall deaths "
          f"{int(log['deaths_wall'].sum())}, flips {flips}, max stack {c.max()}, max ulp {MAX_ULP_SEEN}")
    assert int(log["births"].sum()) > 0 and int(log["deaths_wall"].sum()) > 0
    world.destroy()


def test_coloc_paper_world_lockstep_400_steps():
    """workloads.paper_world_coloc: the paper's world, agents and reproduction at full size."""
    wc = workloads.paper_world_coloc()
    world = sim.World(wc)
    orc = oracle.OracleWorld(wc)
    flips, n, nulp = lockstep_sampled(world, orc, 400, check_weights_every=200)
    log = world.step_log(0, 400)[:, 0]
    print(f"coloc paper world: {n} agent-steps, births {int(log['births'].sum())}, timer deaths "
          f"{int(log['deaths_energy'].sum())}, wall deaths {int(log['deaths_wall'].sum())}, flips {flips}")
    assert int(log["births"].sum()) > 0
    world.destroy()


def test_coloc_batch_equals_single_worlds_and_instrumented_path():
    """Three worlds batched equal the single worlds bitwise (60 steps), and the graph path
    equals the one-kernel-per-phase instrumented path."""
    seeds = (31, 32, 33)
    wc = small(seeds=seeds)
    batch = sim.World(wc)
    batch.step(60)
    b = batch.get_state()
    for k, s in enumerate(seeds):
        one = sim.World(wc.replace(seeds=(s,)))
        if k == 0:
            for _ in range(60):
                one.step_timed()
        else:
            one.step(60)
        a = one.get_state()
        for f in sim.STATE_FIELDS:
            assert np.array_equal(np.asarray(a[f])[0], np.asarray(b[f])[k]), (s, f)
        one.destroy()
    batch.destroy()


@pytest.mark.parametrize("cfg", ["paper_world_cnn", "paper_world_coloc"])
def test_network1_determinism_resume_and_instrumented_path(cfg):
    """The paper's network, exclusive and co-located: two runs are bitwise equal; a run
    resumed by sim_set_state from its own state at t = 70 equals the uninterrupted run at
    t = 140 (every field, weights included); the instrumented path (one kernel per phase)
    equals the graph path."""
    wc = small() if cfg == "paper_world_coloc" else workloads.paper_world_cnn().replace(
        rows=40, cols=60, slots=300, n_initial=150, repr_steps=20, seeds=(17,))
    a, b = sim.World(wc), sim.World(wc)
    a.step(70)
    mid = a.get_state()
    a.step(70)
    for _ in range(70):
        b.step_timed()
    b.step(70)
    sa, sb = a.get_state(), b.get_state()
    for f in sim.STATE_FIELDS:
        assert np.array_equal(np.asarray(sa[f]), np.asarray(sb[f])), f
    c = sim.World(wc)
    c.set_state(mid)
    c.step(70)
    sc = c.get_state()
    for f in sim.STATE_FIELDS:
        assert np.array_equal(np.asarray(sa[f]), np.asarray(sc[f])), ("resume", f)
    for w in (a, b, c):
        w.destroy()
