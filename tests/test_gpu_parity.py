"""GPU parity: the CUDA library (through its C ABI) against the oracle on seeded inputs.

Integer state, step records and slot layout bit-exact; LSTM state within R27; weights
bit-exact up to counted 1-ulp differences (R29); argmax disagreements only at flagged
near-ties (R28).  Sizes span several tiles and ragged tails; the BASELINE configs at their
full sizes (8192x16384 regrowth, the 64-world ensemble, ensemble worlds at 8,192 slots) are
in test_gpu_fullsize.py.
"""
import numpy as np
import pytest

import oracle
import workloads
from harness import (MAX_ABS_SEEN, compare_floats, compare_ints, compare_record, compare_weights, gpu_world_state, lockstep)
from scenario import E, N, STAY, W, build_state, forced, small_config

pytestmark = pytest.mark.gpu

sim = pytest.importorskip("paper_2302_09334_b200.sim")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device (no CPU fallback exists)")


def gpu_state(world, w=0, weights=True):
    fields = sim.STATE_FIELDS if weights else tuple(f for f in sim.STATE_FIELDS if f != "weights")
    return gpu_world_state(world.get_state(fields), w)


# ----------------------------------------------------------------------------- init
@pytest.mark.parametrize("cfg", ["tiny", "paper", "odd", "paper_world"])
def test_init_matches_oracle(cfg):
    wc = {"tiny": workloads.tiny(), "paper": workloads.paper_scale(), "paper_world": workloads.paper_world(),
          "odd": workloads.tiny().replace(rows=37, cols=68, slots=100, n_initial=77, seeds=(12345678901,),
                                          hidden=16, obs_radius=3)}[cfg]
    with sim.World(wc) as world:
        g = gpu_state(world)
        o = oracle.OracleWorld(wc).state()
        compare_ints(g, o, "init")
        assert np.array_equal(g["last_action"], o["last_action"])
        live = o["alive"] == 1
        compare_weights(g["weights"], o["weights"], live, where="init")
        assert np.all(g["weights"][~live] == 0)
        assert np.all(g["h"] == 0) and np.all(g["c"] == 0)


def test_init_invalid_too_many_agents():
    wc = workloads.tiny().replace(init_resource_p=0.99, slots=900, n_initial=800)
    with pytest.raises(sim.SimError) as ei:
        sim.World(wc)
    assert ei.value.status == sim.SIM_E_INVALID and "n_initial" in str(ei.value)


# ------------------------------------------------------------------- regrowth-only
@pytest.mark.parametrize("rows,cols,steps,every", [(200, 400, 1000, 1), (37, 68, 300, 1), (2, 36, 200, 1),
                                                   (2048, 4096, 100, 10)])
def test_regrowth_only_bit_exact(rows, cols, steps, every):
    wc = workloads.regrowth_micro(rows, cols)
    world = sim.World(wc)
    R = oracle.OracleWorld(wc).st["resources"].copy()
    g = world.get_state(("resources",))["resources"][0]
    assert np.array_equal(g, R)
    for t in range(steps):
        R, grown = oracle.regrow(wc, t, R)
        world.step(1)
        rec = world.step_log(t, 1)[0, 0]
        assert rec["grown"] == grown and rec["resources"] == int(R.sum()), t
        if (t + 1) % every == 0 or t + 1 == steps:
            g = world.get_state(("resources",))["resources"][0]
            assert np.array_equal(g, R), f"step {t}"
    world.destroy()


@pytest.mark.parametrize("r2", [1, 2, 5, 8])
def test_regrowth_other_radii(r2):
    wc = workloads.regrowth_micro(45, 100).replace(regrow_r2=r2, f_class_min_k=(0, 1, 2, 4),
                                                  f_value=(0.0, 0.2, 0.4, 0.9))
    world = sim.World(wc)
    R = oracle.OracleWorld(wc).st["resources"].copy()
    for t in range(40):
        R, _ = oracle.regrow(wc, t, R)
    world.step(40)
    assert np.array_equal(world.get_state(("resources",))["resources"][0], R)


def test_regrowth_only_several_worlds_and_resume():
    """Agent-free worlds step with the regrowth kernel and the one-block bookkeeping kernel
    (k_advance_empty): three worlds in one handle against the oracle's regrowth world by
    world (grids, grown and resource counts of every record), and a resume from get_state."""
    seeds = (2, 3, 4)
    wc = workloads.regrowth_micro(70, 132).replace(seeds=seeds)
    world = sim.World(wc)
    Rs = [oracle.OracleWorld(wc.replace(seeds=(s_,))).st["resources"].copy() for s_ in seeds]
    for t in range(25):
        world.step(1)
        rec = world.step_log(t, 1)[0]
        for wi, s_ in enumerate(seeds):
            Rs[wi], grown = oracle.regrow(wc.replace(seeds=(s_,)), t, Rs[wi])
            assert rec[wi]["t"] == t and rec[wi]["grown"] == grown and rec[wi]["resources"] == int(Rs[wi].sum()), (t, s_)
            assert rec[wi]["population"] == 0 and rec[wi]["births"] == 0
    g = world.get_state(("resources",))["resources"]
    for wi in range(3):
        assert np.array_equal(g[wi], Rs[wi]), wi
    snap = world.get_state()
    other = sim.World(wc)
    other.set_state(snap)
    other.step(10)
    world.step(10)
    assert np.array_equal(other.get_state(("resources",))["resources"], world.get_state(("resources",))["resources"])
    assert np.array_equal(other.step_log(25, 10), world.step_log(25, 10))
    assert world.totals()["steps"] == 35
    world.destroy()
    other.destroy()


# --------------------------------------------------------------- full trajectories
def test_tiny_free_running_100_steps_bit_exact():
    """M1: the tiny config's 100 steps, free running on both sides."""
    wc = workloads.tiny()
    world = sim.World(wc)
    orc = oracle.OracleWorld(wc)
    near = 0
    for t in range(100):
        orec = orc.step()
        world.step(1)
        g = gpu_state(world, weights=False)
        o = orc.state()
        where = f"tiny step {t}"
        compare_ints(g, o, where)
        assert np.array_equal(g["last_action"][o["alive"] == 1], o["last_action"][o["alive"] == 1]), where
        compare_record(world.step_log(t, 1)[0, 0], orec, where)
        near += orec["near_ties"]
        live = np.flatnonzero(o["alive"] == 1)
        compare_floats(g, o, live, where)
    gw = world.get_state(("weights",))["weights"][0]
    compare_weights(gw, orc.st["weights"], orc.st["alive"] == 1, where="tiny end")
    print(f"tiny: {near} near-tie agent-steps flagged, trajectory bit-exact")


def test_tiny_lockstep_m2_m3():
    wc = workloads.tiny()
    world = sim.World(wc)
    orc = oracle.OracleWorld(wc)
    flips, n, nulp = lockstep(world, orc, 100, check_weights_every=25)
    assert n > 1000


def test_paper_scale_lockstep_200_steps():
    """C1 (configs[1]) first 200 steps: M2 + M3 every step."""
    wc = workloads.paper_scale()
    world = sim.World(wc)
    orc = oracle.OracleWorld(wc)
    flips, n, nulp = lockstep(world, orc, 200, check_weights_every=100)
    print(f"paper-scale: {n} agent-steps compared, {flips} near-tie disagreements, {nulp} one-ulp weights, "
          f"max |g-o| {MAX_ABS_SEEN}")
    assert n > 200000


def test_large_grid_lockstep():
    """C3 (configs[3]) parity scope on its 1600x3200 grid: M2 + M3 lock-step for 20 steps
    with 8,000 agents in 16,384 slots (the full 262,144-slot world would need 17.8 GB of
    fp32 weights on the oracle's host): large-grid indexing, the claims spread over the
    grid, births, and the oracle's exact integer state and records every step."""
    wc = workloads.large_world().replace(slots=16384, n_initial=8000, repr_steps=8, e_repr_gt=10400)
    world = sim.World(wc)
    orc = oracle.OracleWorld(wc)
    flips, n, nulp = lockstep(world, orc, 20, check_weights_every=10)
    log = world.step_log(0, 20)
    assert n > 100000 and int(log["births"].sum()) > 0
    world.destroy()


@pytest.mark.gpu
def test_many_slots_lockstep():
    """A world with more slots than ECO_HH_BIG_AGENTS (32,768) runs the graph path's second
    k_post variant (16 P warps per block): lock-step with the oracle for 8 steps, births
    included (33,000 agents in 33,792 slots on the 1600x3200 grid)."""
    wc = workloads.large_world().replace(slots=33792, n_initial=33000, repr_steps=4, e_repr_gt=10200)
    world = sim.World(wc)
    orc = oracle.OracleWorld(wc)
    flips, n, nulp = lockstep(world, orc, 8, check_weights_every=4)
    log = world.step_log(0, 8)
    assert n > 200000 and int(log["births"].sum()) > 0
    world.destroy()


@pytest.mark.parametrize("hidden,r", [(4, 1), (16, 2), (32, 0), (8, 3)])
def test_other_shapes_lockstep(hidden, r):
    wc = workloads.tiny().replace(rows=30, cols=72, slots=200, n_initial=90, hidden=hidden, obs_radius=r,
                                  repr_steps=5, e_repr_gt=10200, seeds=(77,))
    world = sim.World(wc)
    orc = oracle.OracleWorld(wc)
    flips, n, _ = lockstep(world, orc, 60, check_weights_every=30)
    assert n > 1000


# --------------------------------------------------------------- injected states (M3)
@pytest.mark.parametrize("cfg,seed", [("tiny", 1), ("tiny", 2), ("paper", 3), ("crowd", 4)])
def test_random_state_one_step(cfg, seed):
    if cfg == "paper":
        wc = workloads.paper_scale().replace(slots=2048)
        st = workloads.random_state(wc, seed, n_alive=1500, density=0.5)
    elif cfg == "crowd":
        # a crowded small world: many claims, births, deaths and capacity deferrals
        wc = workloads.tiny().replace(rows=16, cols=32, slots=300, mutation_std=0.05)
        st = workloads.random_state(wc, seed, n_alive=250, density=0.3)
    else:
        wc = workloads.tiny()
        st = workloads.random_state(wc, seed, n_alive=20, density=0.4)
    st["t"] = 1234 + seed
    for rep in range(3):
        world = sim.World(wc)
        world.set_state(st)
        orc = oracle.OracleWorld(wc, state=st)
        orec = orc.step()
        world.step(1)
        g = gpu_state(world)
        o = orc.state()
        compare_ints(g, o, f"{cfg} rep {rep}")
        compare_record(world.step_log(st["t"], 1)[0, 0], orec, cfg)
        live = np.flatnonzero((o["alive"] == 1) & (o["age"] > 0))
        compare_floats(g, o, live, cfg)
        compare_weights(g["weights"], o["weights"], o["alive"] == 1, where=cfg)
        world.destroy()
        st = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in o.items()}


# --------------------------------------------------------------------- scenarios
def run_both(wc, st, f):
    world = sim.World(wc)
    world.set_state(st)
    world.set_forced_actions(f)
    world.step(1)
    g = gpu_state(world)
    orc = oracle.OracleWorld(wc, state=st)
    orec = orc.step(f)
    compare_ints(g, orc.state(), "scenario")
    compare_record(world.step_log(st["t"], 1)[0, 0], orec, "scenario")
    return g, orec


def test_scenarios_s1_to_s13_match_oracle():
    wc = small_config()
    cases = [
        ([dict(slot=0, y=2, x=2), dict(slot=1, y=2, x=3)], None, {0: E, 1: W}),              # S1
        ([dict(slot=0, y=2, x=2), dict(slot=1, y=2, x=3)], None, {0: E, 1: E}),              # S2
        ([dict(slot=0, y=2, x=1), dict(slot=1, y=2, x=3)], None, {0: E, 1: W}),              # S3
        ([dict(slot=0, y=0, x=3)], None, {0: N}),                                            # S4
        ([dict(slot=0, y=3, x=3)], [(3, 4), (0, 0)], {0: E}),                                # S6
        ([dict(slot=0, y=3, x=3, energy=100)], None, {}),                                    # S11
        ([dict(slot=0, y=3, x=3, energy=50000, age=1000)], None, {}),                        # S12
        ([dict(slot=0, y=3, x=3, energy=11100, repr=7)], [(3, 3)], {}),                      # S13
        ([dict(slot=0, y=2, x=1, energy=20000, repr=19), dict(slot=1, y=2, x=3, energy=20000, repr=19)],
         [(1, 1), (3, 1), (2, 0), (1, 3), (3, 3), (2, 4)], {}),                              # S7
        ([dict(slot=0, y=0, x=0, energy=20000, repr=19), dict(slot=1, y=0, x=1), dict(slot=2, y=1, x=0)],
         None, {}),                                                                          # S8
    ]
    for t in range(0, 40, 7):
        for agents, res, acts in cases:
            st = build_state(wc, agents, resources=res, t=t)
            run_both(wc, st, forced(wc, acts))
    # S9 capacity and S10 slot reuse
    wc3 = small_config(rows=6, cols=8, slots=3)
    st = build_state(wc3, [dict(slot=i, y=1 + 2 * i, x=2 + 2 * i, energy=20000, repr=25) for i in range(3)])
    g, rec = run_both(wc3, st, forced(wc3, {}))
    assert rec["deferred_capacity"] == 3
    st = build_state(wc3, [dict(slot=0, y=1, x=1, energy=20000, repr=25), dict(slot=1, y=4, x=6, energy=100),
                           dict(slot=2, y=4, x=2, energy=20000)])
    g, rec = run_both(wc3, st, forced(wc3, {}))
    assert rec["births"] == 1 and g["alive"][1] == 1
    # S5 regrowth fills the cell under a staying agent
    wc5 = small_config(regrowth=True).replace(f_value=(0.0, 0.0, 0.0, 0.0), spontaneous=1.0)
    g, rec = run_both(wc5, build_state(wc5, [dict(slot=0, y=3, x=3)]), forced(wc5, {0: STAY}))
    assert g["ate"][0] == 1 and rec["eaten"] == 1


def test_scripted_walk_births_21_41_61_81_on_gpu():
    wc = small_config(rows=5, cols=120, slots=8)
    st = build_state(wc, [dict(slot=0, y=2, x=0)], resources=[(2, x) for x in range(1, 120)])
    world = sim.World(wc)
    world.set_state(st)
    world.set_forced_actions(forced(wc, {0: E}))
    world.step(100)
    log = world.step_log(0, 100)[:, 0]
    assert list(np.flatnonzero(log["births"])) == [21, 41, 61, 81]
    # walk (i): a never-eating agent dies at 0-based step 99
    world.set_state(build_state(wc, [dict(slot=0, y=2, x=0)]))
    world.set_forced_actions(forced(wc, {}))
    world.step(100)
    log = world.step_log(0, 100)[:, 0]
    assert list(np.flatnonzero(log["deaths_energy"])) == [99]


# ----------------------------------------------------------------------- ensemble
def test_ensemble_batch_equals_single_worlds_and_oracle():
    seeds = (100, 131, 163)
    wc = workloads.ensemble(seeds).replace(slots=4096)
    batched = sim.World(wc)
    batched.step(60)
    gb = batched.get_state()
    for wi, s in enumerate(seeds):
        single = sim.World(wc.replace(seeds=(s,)))
        single.step(60)
        g1 = single.get_state()
        for k in sim.STATE_FIELDS:
            assert np.array_equal(gb[k][wi], g1[k][0]), (s, k)
        single.destroy()
    log = batched.step_log(0, 60)
    assert log.shape == (60, 3)
    # worlds 100 and 163 against the oracle (lockstep, 40 steps each)
    for s in (100, 163):
        w1 = sim.World(wc.replace(seeds=(s,)))
        orc = oracle.OracleWorld(wc.replace(seeds=(s,)))
        lockstep(w1, orc, 40)
        w1.destroy()


def test_batched_uneven_worlds_equal_single_worlds():
    """40 worlds of very different populations in one handle (the several-world policy walks
    compacted tiles of the worlds' live list positions, the mutation one sequence over all
    worlds' children, the ranking blocks share the regrowth): empty worlds, 1, 2, 15..17
    agents (a tile boundary), a full slot table, worlds past the first 32 (the count chunks)
    -- every world bit-identical to the same state stepped alone, and to the oracle after
    one step."""
    n_w = 40
    wc1 = workloads.paper_scale().replace(rows=40, cols=80, slots=512, n_initial=100, seeds=(200,))
    counts = [0, 1, 2, 15, 16, 17, 511, 512, 0, 33] + [int(c) for c in np.random.default_rng(5).integers(0, 513, n_w - 10)]
    states = [workloads.random_state(wc1, 300 + w, n_alive=counts[w], density=0.3, t=77) for w in range(n_w)]
    wcb = wc1.replace(seeds=tuple(range(200, 200 + n_w)))
    stack = {k: (np.stack([st[k] for st in states]) if isinstance(v, np.ndarray) else v) for k, v in states[0].items()}
    batched = sim.World(wcb)
    batched.set_state(stack)
    batched.step(1)
    g1 = batched.get_state()
    for w in (0, 1, 5, 7, 33):  # against the oracle after one step
        orc = oracle.OracleWorld(wc1.replace(seeds=(200 + w,)), state=states[w])
        orec = orc.step()
        compare_ints(gpu_world_state(g1, w), orc.state(), f"uneven batch world {w}")
        compare_record(batched.step_log(77, 1)[0, w], orec, f"uneven batch world {w}")
    batched.step(5)
    gb = batched.get_state()
    births = batched.step_log(77, 6)["births"].sum(axis=0)
    assert (births > 0).sum() >= 20, births  # the mutation ran in many worlds at once
    for w in range(n_w):
        single = sim.World(wc1.replace(seeds=(200 + w,)))
        single.set_state(states[w])
        single.step(6)
        gs = single.get_state()
        live = gs["alive"][0] == 1
        for k in sim.STATE_FIELDS:
            if k == "weights":  # (a dead slot's weights are unspecified, sim.h)
                assert np.array_equal(gb[k][w][live], gs[k][0][live]), (w, counts[w], k)
            else:
                assert np.array_equal(gb[k][w], gs[k][0]), (w, counts[w], k)
        single.destroy()
    batched.destroy()


# --------------------------------------------------------------------- edge cases
def test_edge_empty_and_degenerate_worlds():
    # no agents at all, agents but zero initial, single-row-pair grid, W not a multiple of 32
    for wc in (workloads.tiny().replace(slots=0, n_initial=0),
               workloads.tiny().replace(n_initial=0),
               workloads.tiny().replace(rows=2, cols=36, slots=10, n_initial=6),
               workloads.tiny().replace(rows=9, cols=100, slots=64, n_initial=64)):
        world = sim.World(wc)
        orc = oracle.OracleWorld(wc)
        for t in range(30):
            orec = orc.step()
            world.step(1)
            compare_ints(gpu_state(world, weights=False), orc.state(), f"edge {wc.rows}x{wc.cols} step {t}")
            compare_record(world.step_log(t, 1)[0, 0], orec)
        world.destroy()


def test_extinction_and_step_zero():
    wc = workloads.no_regrowth(workloads.tiny()).replace(init_resource_p=0.0)
    world = sim.World(wc)
    world.step(0)
    world.step(101)
    log = world.step_log(0, 101)[:, 0]
    assert log["population"][-1] == 0 and world.totals()["steps"] == 101


def test_determinism_and_resume():
    wc = workloads.tiny().replace(rows=40, cols=80, slots=128, n_initial=60, seeds=(9,))
    a = sim.World(wc)
    a.step(150)
    sa = a.get_state()
    b = sim.World(wc)
    b.step(70)
    snap = b.get_state()
    c = sim.World(wc)
    c.set_state(snap)
    c.step(80)
    sc = c.get_state()
    b.step(80)
    sb = b.get_state()
    for k in sim.STATE_FIELDS:
        assert np.array_equal(sa[k], sb[k]), k
        assert np.array_equal(sa[k], sc[k]), k
    assert sa["t"] == sc["t"] == 150


def test_graph_path_equals_instrumented_path_long_run():
    """The fused graph step (cooperative k_post: flags, block-0 claims and rank, idle-block
    regrowth) and the instrumented step (one kernel per phase) must agree exactly over a
    long paper-scale run: an ordering race between the fused phases shows up as a first
    differing step (one such race first surfaced at step 1134)."""
    wc = workloads.paper_scale()
    K = 2000
    world = sim.World(wc, log_capacity=K + 16)
    world.step(5)
    snap = world.get_state()
    t0 = world.t
    world.step(K)
    log_g = world.step_log(t0, K)[:, 0]
    sg = world.get_state(("alive", "cell", "energy", "h", "weights"))
    world.set_state(snap)
    for _ in range(K):
        world.step_timed()
    log_t = world.step_log(t0, K)[:, 0]
    bad = [k for k in range(K) if log_g[k] != log_t[k]]
    assert not bad, f"first differing step {t0 + bad[0]}"
    st = world.get_state(("alive", "cell", "energy", "h", "weights"))
    for f in sg:
        if f != "t":
            assert np.array_equal(sg[f], st[f]), f
    world.destroy()


@pytest.mark.gpu
def test_graph_timed_step_equals_graph_step():
    """sim_step_graph_timed (the bench's per-kernel timing of the graph path) launches the
    graph's own two kernels directly: same trajectory and state as sim_step, and interleaving
    the two modes is seamless (the P rows and children counts carry over)."""
    wc = workloads.paper_scale()
    K = 300
    world = sim.World(wc, log_capacity=K + 16)
    world.step(5)
    snap = world.get_state()
    t0 = world.t
    world.step(K)
    log_g = world.step_log(t0, K)[:, 0]
    sg = world.get_state(("alive", "cell", "energy", "h", "c", "weights"))
    world.set_state(snap)
    for k in range(K):
        if k % 3 == 2:
            world.step(1)
        else:
            ms = world.step_graph_timed()
            assert ms["policy"] > 0 and ms["post"] > 0
    log_t = world.step_log(t0, K)[:, 0]
    bad = [k for k in range(K) if log_g[k] != log_t[k]]
    assert not bad, f"first differing step {t0 + bad[0]}"
    st = world.get_state(("alive", "cell", "energy", "h", "c", "weights"))
    for f in sg:
        if f != "t":
            assert np.array_equal(sg[f], st[f]), f
    world.destroy()


def _sharded_step(ranks):
    """One agent-sharded step of all ranks of a world on this GPU: the ranks' policies, the
    SUM-combine of their exchange buffers (what an NCCL allreduce does across GPUs; here the
    host sequences it, no kernel waits on another rank's), then every rank's dynamics."""
    import torch
    for r in ranks:
        r.step_policy()
    for r in ranks:
        r.synchronize()
    bufs = [r.exchange_tensors() for r in ranks]
    m = sum(b[0] for b in bufs)
    rec = sum(b[1] for b in bufs)
    for b in bufs:
        b[0].copy_(m)
        b[1].copy_(rec)
    torch.cuda.synchronize()
    for r in ranks:
        r.step_post()


@pytest.mark.parametrize("n_ranks", [2, 3])
def test_agent_sharded_world_equals_unsharded(n_ranks):
    """SURVEY.md §8(e) (agent-home variant): the world stepped as n_ranks ranks, each
    running the policy of its own slots and the dynamics of the whole world, reproduces the
    unsharded trajectory exactly: integer state and records bit-exact on every rank, and
    every live agent's weights, h and c bit-exact on some rank (its owner)."""
    wc = workloads.paper_scale().replace(slots=2048, n_initial=600)
    K = 150  # births from step ~21, slot reuse (a child in a slot last owned by another rank) later
    ref = sim.World(wc)
    ranks = [sim.World(wc) for _ in range(n_ranks)]
    for r, w in enumerate(ranks):
        w.shard(n_ranks, r)
    with pytest.raises(sim.SimError):
        ranks[0].step(1)  # a sharded handle steps only through the exchange protocol
    ref.step(K)
    for _ in range(K):
        _sharded_step(ranks)
    lr = ref.step_log(0, K)
    assert int(lr["births"].sum()) > 0  # the run exercised reproduction and mutation
    sr = ref.get_state()
    ints = ("resources", "alive", "cell", "energy", "age", "repr", "ate")
    states = [w.get_state() for w in ranks]
    for w, st in zip(ranks, states):
        assert np.array_equal(w.step_log(0, K), lr)
        for f in ints:
            assert np.array_equal(st[f], sr[f]), f
    live = np.flatnonzero(sr["alive"][0])
    for f in ("weights", "h", "c"):
        ok = np.zeros(len(live), bool)
        for st in states:
            ok |= np.all(st[f][0][live] == sr[f][0][live], axis=tuple(range(1, sr[f][0][live].ndim)))
        assert ok.all(), f"{f}: {int((~ok).sum())} live agents differ on every rank"
    for w in ranks + [ref]:
        w.destroy()


def test_record_mirror_and_async_log_equal_the_log():
    """sim_set_record_mirror (device-written mapped host ring) and sim_get_step_log_async
    deliver exactly the records sim_get_step_log returns."""
    import torch
    wc = workloads.tiny().replace(rows=40, cols=80, slots=128, n_initial=60, seeds=(4,))
    world = sim.World(wc)
    K, cap = 40, 16
    buf = torch.empty((cap, sim.RECORD_DTYPE.itemsize), dtype=torch.uint8, pin_memory=True).numpy()
    ring = buf.view(sim.RECORD_DTYPE).reshape(cap, 1)
    with pytest.raises(sim.SimError):
        world.set_record_mirror(ring[:12], 12)  # not a power of two
    world.set_record_mirror(ring, cap)
    abuf = torch.empty((K, sim.RECORD_DTYPE.itemsize), dtype=torch.uint8, pin_memory=True).numpy()
    alog = abuf.view(sim.RECORD_DTYPE).reshape(K, 1)
    for k in range(K):
        world.step(1)
        world.step_log_async(k, 1, alog[k:k + 1])
    world.synchronize()
    log = world.step_log(0, K)
    assert np.array_equal(alog, log)
    assert np.array_equal(ring[np.arange(K - cap, K) % cap], log[K - cap:])
    world.set_record_mirror(None)
    world.step(1)
    world.synchronize()
    assert np.array_equal(ring[np.arange(K - cap, K) % cap], log[K - cap:])  # no longer written
    world.destroy()


def test_set_state_rejects_bad_occupancy_and_nonfinite():
    wc = workloads.tiny()
    world = sim.World(wc)
    st = world.get_state()
    st2 = dict(st)
    st2["cell"] = st["cell"].copy()
    live = np.flatnonzero(st["alive"][0])
    st2["cell"][0, live[1]] = st["cell"][0, live[0]]
    with pytest.raises(sim.SimError):
        world.set_state(st2)
    st3 = dict(st)
    st3["weights"] = st["weights"].copy()
    st3["weights"][0, live[0], 3] = np.nan
    with pytest.raises(sim.SimError):
        world.set_state(st3)


@pytest.mark.parametrize("scatter", [False, True])
def test_set_state_from_pinned_memory(scatter):
    """sim_set_state from page-locked host buffers: the live rows' weights arrive by DMA runs
    (few runs) or are gathered in place from mapped memory (more than 64 runs); both paths
    give the same device state, and a non-finite weight in a live slot is refused either way."""
    import torch
    wc = workloads.paper_scale().replace(rows=60, cols=80, slots=600, n_initial=300)
    st = workloads.random_state(wc, 7, n_alive=300)
    if not scatter:  # live slots 0..299: one run
        order = np.argsort(-st["alive"], kind="stable")
        for k, v in list(st.items()):
            if isinstance(v, np.ndarray) and v.shape[:1] == (wc.slots,):
                st[k] = v[order].copy()
    live = np.flatnonzero(st["alive"])
    runs = 1 + int((np.diff(live) != 1).sum())
    assert (runs > 64) == scatter
    pinned = {}
    for k, v in st.items():
        if isinstance(v, np.ndarray):
            tt = torch.empty((1,) + v.shape, dtype=getattr(torch, str(v.dtype)), pin_memory=True)
            tt.numpy()[...] = v
            pinned[k] = tt.numpy()
        else:
            pinned[k] = v
    world = sim.World(wc)
    world.set_state(pinned)
    g = gpu_world_state(world.get_state())
    for f in ("alive", "cell", "energy", "h", "c"):
        assert np.array_equal(g[f][live], st[f][live]), f
    assert np.array_equal(g["weights"][live], st["weights"][live])
    pinned["weights"][0, live[5], 17] = np.inf
    with pytest.raises(sim.SimError):
        world.set_state(pinned)
    world.destroy()


def test_nonfinite_state_reported():
    wc = workloads.tiny()
    world = sim.World(wc)
    st = world.get_state()
    live = np.flatnonzero(st["alive"][0])[0]
    G = 4 * wc.hidden
    boff = G * wc.n_inputs + G * wc.hidden
    # bias 50 on every gate: i = f = o = 1, g = 1, so h' ~ tanh(2); W_out = 3e38 overflows the logits
    st["weights"][0, live, boff:boff + G] = 50.0
    st["weights"][0, live, boff + G:boff + G + 5 * wc.hidden] = 3.0e38
    st["c"][0, live, :] = 1.0
    world.set_state(st)
    with pytest.raises(sim.SimError) as ei:
        world.step(1)
        world.synchronize()
    assert ei.value.status == sim.SIM_E_NONFINITE


def test_large_world_full_size_graph_equals_instrumented_and_invariants():
    """BASELINE configs[3] at its full size (1600x3200, 262,144 slots, 64,000 agents) in the
    launch configuration bench.py times (the graph path, k_post with 16 P warps per block):
    two identically created worlds, one stepped through the graph and one through the
    instrumented phase kernels, agree exactly (records and integer state, h and c), and the
    properties that hold at any size hold (unique in-range cells of live agents, the
    population and resource balance of every record, the final resource plane's popcount)."""
    wc = workloads.large_world()
    K = 32  # the first births come after T_repr = 20 steps above the energy threshold
    a, b = sim.World(wc, log_capacity=64), sim.World(wc, log_capacity=64)
    a.step(K)
    for _ in range(K):
        b.step_timed()
    la, lb = a.step_log(0, K)[:, 0], b.step_log(0, K)[:, 0]
    assert np.array_equal(la, lb)
    fields = ("alive", "cell", "energy", "age", "repr", "h", "c", "resources")
    sa, sb = a.get_state(fields), b.get_state(fields)
    for f in fields:
        assert np.array_equal(sa[f], sb[f]), f
    alive = sa["alive"][0] == 1
    cells = sa["cell"][0][alive]
    assert cells.min() >= 0 and cells.max() < wc.rows * wc.cols and np.unique(cells).size == cells.size
    assert int(alive.sum()) == int(la["population"][-1])
    for k in range(1, K):
        assert la["agents_at_start"][k] == la["population"][k - 1]
        assert la["resources"][k] == la["resources"][k - 1] + la["grown"][k] - la["eaten"][k]
    assert la["population"][-1] == la["agents_at_start"][-1] - la["deaths_energy"][-1] - la["deaths_age"][-1] \
        + la["births"][-1]
    assert int(sa["resources"][0].astype(np.int64).sum()) == int(la["resources"][-1])
    assert int(la["births"].sum()) > 0
    a.destroy()
    b.destroy()


# ------------------------------------------------- Appendix C metrics
def _fold_run(world, orc, steps, forced_fn=None):
    """Step the oracle and the library together (the library forced to the oracle's actions
    when forced_fn is None) and fold the oracle's states into the Appendix C metrics."""
    from oracle import metrics
    fold = metrics.MetricsFold(world.wc.cols)
    for _ in range(steps):
        before = {k: orc.st[k].copy() for k in ("alive", "cell", "age")} | {"t": orc.t}
        if forced_fn is None:
            r = orc.step(return_actions=True)
            f = np.full((1, world.wc.slots), 255, np.uint8)
            f[0] = r["actions"]
        else:
            f = forced_fn()
            r = orc.step(forced=f)
            f = f[None]
        assert r["status"] == 0
        world.set_forced_actions(f)
        world.step(1)
        fold.feed(before, {k: orc.st[k] for k in ("alive", "cell", "age")} | {"t": orc.t})
    world.set_forced_actions(None)
    return fold


def _check_metrics(world, fold, t0, steps):
    log = world.step_log(t0, steps)[:, 0]
    for k in range(steps):
        assert int(log["death_age_sum"][k]) == fold.death_age_sum[t0 + k], f"step {t0 + k}"
    wins = sorted(fold.hist)
    got = world.move_hist(wins[0], len(wins))[:, 0]
    for i, k in enumerate(wins):
        assert np.array_equal(got[i], fold.hist[k]), (k, got[i], fold.hist[k])
    return got


def test_metrics_scripted_walk():
    from scenario import E, build_state, forced, small_config
    wc = small_config(rows=6, cols=60, slots=4)
    st = build_state(wc, [dict(slot=0, y=2, x=2), dict(slot=1, y=4, x=30), dict(slot=2, y=0, x=50, energy=1000)])
    world = sim.World(wc)
    world.set_state(st)
    orc = oracle.OracleWorld(wc, state=st)
    fold = _fold_run(world, orc, 50, forced_fn=lambda: forced(wc, {0: E}))
    got = _check_metrics(world, fold, 0, 50)
    assert got[0][16] == 1 and got[0][0] == 1 and got[0].sum() == 2
    assert int(world.step_log(9, 1)[0, 0]["death_age_sum"]) == 10


def test_metrics_match_the_oracle_tiny_and_paper_scale():
    """Movement histograms and ages at death equal the oracle fold: the tiny world over 150
    steps (three windows), the paper-scale world over 100 steps (two windows, thousands of
    agents, births and deaths); both forced to the oracle's actions (M2)."""
    for wc, steps in ((workloads.tiny(), 150), (workloads.paper_scale(), 100)):
        world = sim.World(wc)
        orc = oracle.OracleWorld(wc)
        fold = _fold_run(world, orc, steps)
        got = _check_metrics(world, fold, 0, steps)
        assert got.sum() > 0
        world.destroy()


def test_metrics_after_set_state_mid_window():
    """A run resumed at t = 25 does not measure window 0 (begun before the resume: all 0) and
    measures window 1 exactly."""
    wc = workloads.tiny()
    a = sim.World(wc)
    a.step(25)
    snap = a.get_state()
    world = sim.World(wc)
    world.set_state(snap)
    orc = oracle.OracleWorld(wc, state=snap)
    fold = _fold_run(world, orc, 75)
    assert world.move_hist(0, 1).sum() == 0
    assert np.array_equal(world.move_hist(1, 1)[0, 0], fold.hist[1])


# ------------------------------------------------- greediness and life expectancy (NEXT-3)
def test_greediness_counts_equal_oracle_fold():
    """T_r and C_r of every live agent after 200 tiny steps (10 windows; the GPU forced to
    the oracle's actions, M2) equal the oracle fold (oracle/metrics.py GreedinessFold)."""
    from oracle import metrics
    wc = workloads.tiny().replace(repr_steps=6, e_repr_gt=10300)  # births reuse slots
    world = sim.World(wc)
    orc = oracle.OracleWorld(wc)
    fold = metrics.GreedinessFold(wc)
    births = 0
    for t in range(200):
        before = orc.state()
        orec = orc.step(return_actions=True)
        fold.feed(before, orc.state())
        births += orec["births"]
        f = np.full((1, wc.slots), 255, np.uint8)
        f[0] = orec["actions"]
        world.set_forced_actions(f)
        world.step(1)
    world.set_forced_actions(None)
    g = gpu_state(world, weights=False)
    compare_ints(g, orc.state(), "greediness run end")
    T, C = world.greediness()
    live = orc.st["alive"] == 1
    assert births > 0 and int(fold.T[live].sum()) > 0 and int(fold.C[live].sum()) > 0
    assert np.array_equal(T[0][live], fold.T[live]) and np.array_equal(C[0][live], fold.C[live])
    world.destroy()


def test_banded_greediness_equals_unbanded_by_cell():
    wc = workloads.paper_scale()
    ref = sim.World(wc)
    ban = sim.World(wc, bands=dict(n_bands=4))
    ref.step(120)
    ban.step(120)
    out = []
    for w in (ref, ban):
        st = w.get_state(("alive", "cell"))
        T, C = w.greediness()
        live = np.flatnonzero(st["alive"][0])
        out.append(dict(zip(st["cell"][0][live].tolist(), zip(T[0][live].tolist(), C[0][live].tolist()))))
    assert out[0] == out[1] and sum(v[0] for v in out[0].values()) > 0
    ref.destroy()
    ban.destroy()


def test_life_windows_equal_the_records():
    """The device's 500-step windows of deaths and ages at death equal the sums of the step
    records (which are pinned against the oracle) over each window."""
    wc = workloads.paper_scale()
    world = sim.World(wc, log_capacity=2048)
    world.step(1100)
    d, a = world.life_windows(0, 2)
    log = world.step_log(0, 1000)[:, 0]
    for k in range(2):
        rk = log[500 * k:500 * (k + 1)]
        assert d[k, 0] == int(rk["deaths_energy"].sum() + rk["deaths_age"].sum())
        assert a[k, 0] == int(rk["death_age_sum"].sum())
    assert d[1, 0] > 0
    world.destroy()


# ---------------------------------------------- the paper's own world (NEXT-1, App. B.4)
def test_paper_world_lockstep_400_steps():
    """workloads.paper_world (exponential climate, 4-neighbour indicator regrowth, clipped
    energy, death timer, lethal walls, Hd = 4) in M2 + M3 lock-step with the oracle for 400
    steps: births from ~140 on, timer starvation from ~319, wall deaths."""
    wc = workloads.paper_world()
    world = sim.World(wc)
    orc = oracle.OracleWorld(wc)
    flips, n, nulp = lockstep(world, orc, 400, check_weights_every=200)
    log = world.step_log(0, 400)[:, 0]
    print(f"paper world: {n} agent-steps, births {int(log['births'].sum())}, timer deaths "
          f"{int(log['deaths_energy'].sum())}, wall deaths {int(log['deaths_wall'].sum())}")
    assert int(log["births"].sum()) > 0 and int(log["deaths_wall"].sum()) > 0
    world.destroy()


def test_paper_world_banded_equals_unbanded():
    wc = workloads.paper_world()
    ref = sim.World(wc)
    ban = sim.World(wc, bands=dict(n_bands=4))
    ref.step(400)
    ban.step(400)
    a, b = ref.get_state(), ban.get_state()
    for st in (a, b):
        live = np.flatnonzero(st["alive"][0])
        st["_by_cell"] = {int(st["cell"][0][i]): i for i in live}
    assert np.array_equal(a["resources"], b["resources"]) and a["_by_cell"].keys() == b["_by_cell"].keys()
    for c, i in a["_by_cell"].items():
        j = b["_by_cell"][c]
        for f in ("energy", "age", "repr", "low", "h", "c", "weights"):
            assert np.array_equal(a[f][0][i], b[f][0][j]), (c, f)
    la, lb = ref.step_log(0, 400)[:, 0], ban.step_log(0, 400)[:, 0]
    for f in sim.RECORD_FIELDS:
        assert np.array_equal(la[f], lb[f]), f
    ref.destroy()
    ban.destroy()
