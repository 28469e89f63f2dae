"""GPU parity of network 1, the paper's CNN-LSTM with softmax sampling (
SURVEY.md §8(f) NEXT-2; k_policy_cnn_blk) against the oracle, through the C ABI.

Integer state, step records and slot layout bit-exact; h', c', logits within R27; weights
bit-exact up to counted 1-ulp differences (R29); the kernel's own sampled actions
(sim_get_policy_actions) equal the oracle's except at flagged sampling near-ties (R38).
"""
import numpy as np
import pytest

import oracle
import workloads
from harness import MAX_ABS_SEEN, MAX_ULP_SEEN, compare_floats, compare_ints, compare_weights, gpu_world_state, lockstep_sampled

pytestmark = pytest.mark.gpu

sim = pytest.importorskip("paper_2302_09334_b200.sim")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device (no CPU fallback exists)")


def small(**kw):
    base = dict(rows=40, cols=60, slots=200, n_initial=120, repr_steps=20, seeds=(11,))
    base.update(kw)
    return workloads.paper_world_cnn().replace(**base)


def test_cnn_init_matches_oracle():
    wc = workloads.paper_world_cnn()
    with sim.World(wc) as world:
        g = gpu_world_state(world.get_state())
        o = oracle.OracleWorld(wc).state()
        compare_ints(g, o, "init")
        live = o["alive"] == 1
        assert g["weights"].shape == (wc.slots, 2445)
        compare_weights(g["weights"], o["weights"], live, where="init")
        assert np.all(g["weights"][~live] == 0)


@pytest.mark.parametrize("seed,wstd,density", [(1, 0.1, 0.3), (2, 0.5, 0.5), (3, 0.3, 0.1), (4, 1.0, 0.7)])
def test_cnn_one_step_random_states(seed, wstd, density):
    """Injected random states (agents everywhere, borders included, random h, c, previous
    actions, ate flags and weights up to std 1): one step, every agent's h', c', logits
    within R27, its own sampled action equal to the oracle's except at flagged near-ties,
    and the children's mutated weights (repr above T_repr for many parents) bit-exact."""
    wc = small(rows=37, cols=52, slots=300, seeds=(100 + seed,))
    st = workloads.random_state(wc, seed, n_alive=220, density=density, weight_std=wstd)
    rng = np.random.default_rng(seed)
    st["ate"][st["alive"] == 1] = rng.integers(0, 2, int(st["alive"].sum())).astype(np.uint8)
    st["energy"][st["alive"] == 1] = rng.integers(1, 3001, int(st["alive"].sum())).astype(np.int32)
    st["repr"][st["alive"] == 1] = rng.integers(0, 2 * wc.repr_steps, int(st["alive"].sum())).astype(np.int32)
    st["age"] = np.minimum(st["age"], 600).astype(np.int32)
    world = sim.World(wc)
    world.set_state({k: (v[None] if isinstance(v, np.ndarray) else v) for k, v in st.items()})
    orc = oracle.OracleWorld(wc, state=st)
    flips, n, nulp = lockstep_sampled(world, orc, 1, check_weights_every=1)
    assert n == 220
    births = int(world.step_log(st["t"], 1)[0, 0]["births"])
    print(f"one step: {n} agents, {births} births, {flips} flagged flips, {nulp} 1-ulp weights, "
          f"max |d| {MAX_ABS_SEEN}, max ulp {MAX_ULP_SEEN}")
    assert births > 0
    world.destroy()


def test_cnn_lockstep_small_world_300_steps():
    """A 40x60 paper world with the paper's network and T_repr = 20: births from step ~20,
    wall deaths, exact trajectories for 300 steps."""
    wc = small()
    world = sim.World(wc)
    orc = oracle.OracleWorld(wc)
    flips, n, nulp = lockstep_sampled(world, orc, 300, check_weights_every=50)
    log = world.step_log(0, 300)[:, 0]
    print(f"cnn small world: {n} agent-steps, births {int(log['births'].sum())}, wall deaths "
          f"{int(log['deaths_wall'].sum())}, {flips} flagged flips, {nulp} 1-ulp weights, max ulp {MAX_ULP_SEEN}")
    assert int(log["births"].sum()) > 0 and int(log["deaths_wall"].sum()) > 0
    world.destroy()


def test_cnn_paper_world_lockstep_400_steps():
    """workloads.paper_world_cnn: the paper's own world and agents (App. B.4-B.5) at full
    size (200x400, 1000 slots, 330 agents) for 400 steps: births from ~140, timer
    starvation from ~319, wall deaths."""
    wc = workloads.paper_world_cnn()
    world = sim.World(wc)
    orc = oracle.OracleWorld(wc)
    flips, n, nulp = lockstep_sampled(world, orc, 400, check_weights_every=200)
    log = world.step_log(0, 400)[:, 0]
    print(f"cnn paper world: {n} agent-steps, births {int(log['births'].sum())}, timer deaths "
          f"{int(log['deaths_energy'].sum())}, wall deaths {int(log['deaths_wall'].sum())}, flips {flips}")
    assert int(log["births"].sum()) > 0 and int(log["deaths_wall"].sum()) > 0
    world.destroy()


def test_cnn_batch_equals_single_worlds():
    """Three worlds batched on the device equal the same worlds run alone (bitwise), 60 steps."""
    seeds = (21, 22, 23)
    wc = small(seeds=seeds)
    batch = sim.World(wc)
    batch.step(60)
    b = batch.get_state()
    for k, s in enumerate(seeds):
        one = sim.World(wc.replace(seeds=(s,)))
        one.step(60)
        a = one.get_state()
        for f in sim.STATE_FIELDS:
            assert np.array_equal(np.asarray(a[f])[0], np.asarray(b[f])[k]), (s, f)
        one.destroy()
    batch.destroy()


def test_cnn_sampler_uniform_at_zero_weights():
    """All-zero weights give zero logits, a uniform softmax, so the kernel's
    own sampled actions are uniform over the 5 actions: 0.2 +- 0.01 over > 10^5 draws
    (SPEC.md:151), checked against the closed form, not against the oracle."""
    wc = small(rows=100, cols=200, slots=4000, n_initial=3000, repr_steps=10**6, seeds=(5,))
    world = sim.World(wc)
    st = world.get_state()
    st["weights"][:] = 0.0
    world.set_state(st)
    world.set_forced_actions(np.zeros((1, wc.slots), np.uint8))  # everyone stays: no deaths at walls
    counts = np.zeros(5, np.int64)
    for _ in range(40):
        alive = world.get_state(("alive",))["alive"][0] == 1
        world.step(1)
        own = world.policy_actions()[0][alive]
        counts += np.bincount(own, minlength=5)[:5]
    freq = counts / counts.sum()
    print("own action frequencies at zero weights:", freq, counts.sum())
    assert counts.sum() > 100_000 and np.all(np.abs(freq - 0.2) < 0.01)
    lg = world.get_state(("logits",))["logits"][0]
    assert np.all(lg == 0.0)
    world.destroy()
