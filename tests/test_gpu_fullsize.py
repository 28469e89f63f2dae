"""GPU parity at BASELINE.json's full sizes, in the launch
configuration bench.py / tools/bench_regrowth.py time (the graph path):

* configs[2]'s largest regrowth grid, 8192x16384 (134 M cells): bit-exact against the
  oracle for 10 steps from its initial grid (the growth phase) and for 5
  steps from a synthetic near-saturated grid injected at t = 900 (the saturated phase,
  where most 4-cell groups skip their draws);
* configs[4]'s ensemble worlds 100 and 163 at the full 8,192 slots, M2 + M3 lock-step with
  the oracle for 200 steps (SURVEY.md §8c C.6 "ensemble worlds 100 and 163");
* the 64-world batch of configs[4] (35.5 GB of weights on one GPU) equal, field by field, to
  the 64 worlds run one at a time.
"""
import numpy as np
import pytest

import oracle
import workloads
from harness import MAX_ABS_SEEN, lockstep

pytestmark = pytest.mark.gpu

sim = pytest.importorskip("paper_2302_09334_b200.sim")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device (no CPU fallback exists)")


def _regrow_steps_bit_exact(world, wc, R, t0, steps):
    for t in range(t0, t0 + steps):
        R, grown = oracle.regrow(wc, t, R)
        world.step(1)
        rec = world.step_log(t, 1)[0, 0]
        assert rec["grown"] == grown and rec["resources"] == int(R.sum()), f"step {t}"
        g = world.get_state(("resources",))["resources"][0]
        bad = np.argwhere(g != R)
        assert bad.size == 0, f"step {t}: {bad.shape[0]} cells differ, first {bad[:5].tolist()}"
    return R


def test_regrowth_8192x16384_growth_and_saturated_bit_exact():
    wc = workloads.regrowth_micro(8192, 16384)
    world = sim.World(wc)
    R = oracle.OracleWorld(wc).st["resources"].copy()
    assert np.array_equal(world.get_state(("resources",))["resources"][0], R)
    _regrow_steps_bit_exact(world, wc, R, 0, 10)
    # saturated phase: a seeded near-full grid (99.5 % resources) at t = 900
    st = workloads.random_state(wc, seed=900, n_alive=0, density=0.995, t=900)
    world.set_state({"t": 900, "resources": st["resources"]})
    R = st["resources"].copy()
    assert np.array_equal(world.get_state(("resources",))["resources"][0], R)
    _regrow_steps_bit_exact(world, wc, R, 900, 5)
    world.destroy()


@pytest.mark.parametrize("seed", [100, 163])
def test_ensemble_world_full_slots_lockstep_200_steps(seed):
    wc = workloads.ensemble((seed,))
    world = sim.World(wc)
    orc = oracle.OracleWorld(wc)
    flips, n, nulp = lockstep(world, orc, 200, check_weights_every=100)
    print(f"ensemble world {seed}: {n} agent-steps compared, {flips} near-tie disagreements, "
          f"{nulp} one-ulp weights, max |g-o| {MAX_ABS_SEEN}")
    assert n > 200000
    world.destroy()


def test_ensemble_64_batch_equals_single_worlds():
    """configs[4] whole (64 worlds x 8,192 slots): 40 steps batched equal the 64 worlds run
    alone, every non-weight field and record bitwise (h, c and logits bitwise as well: the
    children born from step 21 on act on their mutated weights, so a weight difference
    shows in their LSTM state)."""
    wc = workloads.ensemble()
    steps = 40
    fields = tuple(f for f in sim.STATE_FIELDS if f != "weights")
    batched = sim.World(wc, log_capacity=64)
    batched.step(steps)
    gb = batched.get_state(fields)
    lb = batched.step_log(0, steps)
    batched.destroy()
    assert int(lb["births"].sum()) > 0
    for wi, s in enumerate(wc.seeds):
        single = sim.World(wc.replace(seeds=(s,)), log_capacity=64)
        single.step(steps)
        g1 = single.get_state(fields)
        l1 = single.step_log(0, steps)
        single.destroy()
        assert np.array_equal(lb[:, wi], l1[:, 0]), f"world {s}: records differ"
        for k in fields:
            if k == "t":
                assert gb[k] == g1[k]
                continue
            a, b = gb[k][wi], g1[k][0]
            if k in ("h", "c", "logits", "cell", "energy", "age", "repr", "last_action", "ate"):
                live = g1["alive"][0] == 1
                a, b = a[live], b[live]
            assert np.array_equal(a, b), f"world {s}: {k} differs"
