"""Pins of the oracle's co-location mode (the paper's own
reproduction, "the off-spring appears on the same cell as its parent"; the
agent channel "including their number"; readings R43-R47 in DESIGN.md).

Anchored by SPEC.md's examples (3 agents stacked on a visible cell give 3 in the agent
channel; exactly one of the co-located agents consumes a resource, SPEC.md:273;
child position = parent position) and by hand-built scripted worlds whose
outcome follows from the rules alone: moves into occupied cells succeed, the lottery winner
is the agent with the largest key drawn from the pinned Philox (C.1), the offspring of the
lowest-slot parents take the lowest free slots, the mutation noise of a child is the pinned
Box-Muller sequence of its slot, and conservation holds over long runs.
"""
import numpy as np
import pytest

import oracle
import workloads
from scenario import E, N, STAY, W, build_state, forced

WC = workloads.paper_world_coloc()


def small(**kw):
    base = dict(rows=8, cols=10, slots=8, n_initial=0, f_value=(0.0, 0.0, 0.0, 0.0), spontaneous=0.0,
                mutation_std=0.0)
    base.update(kw)
    return WC.replace(**base)


def test_validation():
    assert oracle.validate(WC)[0] == 0
    assert oracle.validate(WC.replace(network=0, obs_radius=3, hidden=8))[0] != 0  # network 1 only
    assert oracle.validate(WC.replace(colocate=2))[0] != 0


def test_agent_channel_counts_stacked_agents():
    wc = WC.replace(rows=20, cols=24)
    R = np.zeros((20, 24), np.uint8)
    Ncount = np.zeros((20, 24), np.int32)
    Ncount[10, 12] = 1  # self
    Ncount[11, 14] = 3  # 3 agents stacked on one visible cell -> 3
    x = oracle.observe_paper(wc, R, Ncount, 10, 12)
    assert x[7, 7, 1] == 1.0 and x[8, 9, 1] == 3.0 and x[:, :, 1].sum() == 4.0


def test_moves_never_conflict():
    """Two agents stepping onto the same empty cell, and one onto an occupied cell, all arrive."""
    wc = small()
    st = build_state(wc, [dict(slot=0, y=3, x=3), dict(slot=1, y=3, x=5), dict(slot=2, y=5, x=4),
                          dict(slot=3, y=4, x=4)])
    w = oracle.OracleWorld(wc, state=st)
    w.step(forced(wc, {0: E, 1: W, 2: N, 3: STAY}))
    cells = w.st["cell"][:4]
    assert list(cells) == [3 * 10 + 4, 3 * 10 + 4, 4 * 10 + 4, 4 * 10 + 4]
    assert w.st["alive"][:4].all()


def lottery_key(seed, t, slot):
    w0 = oracle.draw4(seed, oracle.P_CONSUME, t, slot)[0]
    return (w0 << 32) | (0xFFFFFFFF - slot)


@pytest.mark.parametrize("t0", [0, 7, 123])
def test_one_agent_per_resource_cell_eats(t0):
    """exactly one co-located agent consumes; the winner is the largest
    (CONSUME draw of the slot, -slot) key; the others do not eat."""
    wc = small(seeds=(t0 + 5,))
    agents = [dict(slot=s, y=2, x=2, energy=2000) for s in (0, 3, 5)] + [dict(slot=6, y=6, x=7, energy=2000)]
    st = build_state(wc, agents, resources=[(2, 2)], t=t0)
    w = oracle.OracleWorld(wc, state=st)
    rec = w.step(forced(wc, {}))
    keys = {s: lottery_key(wc.seeds[0], t0, s) for s in (0, 3, 5)}
    win = max(keys, key=keys.get)
    assert rec["eaten"] == 1 and w.st["resources"][2, 2] == 0
    for s in (0, 3, 5, 6):
        assert w.st["ate"][s] == (1 if s == win else 0)
        assert w.st["energy"][s] == (2975 if s == win else 1975)  # 2.0 (+ 1) - 0.025


def test_lottery_is_fair():
    """Two agents sharing a resource cell over many independent steps win about equally often."""
    wins = np.zeros(2, int)
    wc = small()
    for t0 in range(2000):
        a, b = lottery_key(wc.seeds[0], t0, 1), lottery_key(wc.seeds[0], t0, 4)
        wins[0 if a > b else 1] += 1
    assert abs(wins[0] / wins.sum() - 0.5) < 0.05
    # and the oracle follows the same keys
    st = build_state(wc, [dict(slot=1, y=1, x=1, energy=1000), dict(slot=4, y=1, x=1, energy=1000)],
                     resources=[(1, 1)], t=17)
    w = oracle.OracleWorld(wc, state=st)
    w.step(forced(wc, {}))
    winner = 1 if lottery_key(wc.seeds[0], 17, 1) > lottery_key(wc.seeds[0], 17, 4) else 4
    assert w.st["ate"][winner] == 1 and w.st["ate"][5 - winner] == 0


def test_offspring_on_the_parents_cell_in_the_lowest_free_slots():
    """PAPER.md:297 / SPEC.md:337: child position = parent position; eligible parents in
    slot order take the free slots in ascending order; sigma = 0 gives a copy; the parent's
    repr resets; h = c = 0 and energy E0 for the child."""
    wc = small(repr_steps=5)
    st = build_state(wc, [dict(slot=2, y=4, x=4, repr=4), dict(slot=5, y=4, x=4, repr=4),
                          dict(slot=6, y=1, x=8, repr=0)], zero_weights=False)
    st["h"][2] = 0.5
    w = oracle.OracleWorld(wc, state=st)
    rec = w.step(forced(wc, {}))
    assert rec["births"] == 2 and rec["deferred_capacity"] == 0
    assert w.st["alive"][[0, 1]].all() and w.st["cell"][0] == w.st["cell"][1] == 44
    assert np.array_equal(w.st["weights"][0], st["weights"][2]) and np.array_equal(w.st["weights"][1], st["weights"][5])
    assert w.st["repr"][2] == 0 and w.st["repr"][5] == 0 and w.st["energy"][0] == wc.e_init
    assert np.all(w.st["h"][0] == 0) and np.all(w.st["c"][0] == 0)


def test_mutation_noise_is_keyed_by_the_child_slot():
    wc = small(repr_steps=3, mutation_std=0.02)
    st = build_state(wc, [dict(slot=3, y=2, x=2, repr=2), dict(slot=4, y=2, x=2, repr=2)], zero_weights=False, t=9)
    w = oracle.OracleWorld(wc, state=st)
    w.step(forced(wc, {}))
    for child, parent in ((0, 3), (1, 4)):
        z = oracle.gauss(wc.seeds[0], oracle.P_MUTATE, 9, child, wc.n_params)
        exp = st["weights"][parent] + (0.02 * z).astype(np.float32)
        assert np.array_equal(w.st["weights"][child], exp)
    # the two co-located children differ (keyed by slot, not by their shared cell)
    assert not np.array_equal(w.st["weights"][0] - st["weights"][3], w.st["weights"][1] - st["weights"][4])


def test_capacity_defers_the_highest_slots():
    wc = small(slots=5, repr_steps=3)
    st = build_state(wc, [dict(slot=s, y=3, x=s, repr=2) for s in range(4)])
    w = oracle.OracleWorld(wc, state=st)
    rec = w.step(forced(wc, {}))
    assert rec["births"] == 1 and rec["deferred_capacity"] == 3
    assert w.st["alive"][4] == 1 and w.st["cell"][4] == 3 * 10 + 0   # parent slot 0's child
    assert list(w.st["repr"][:4]) == [0, 3, 3, 3]                    # the deferred keep counting


def test_coloc_world_invariants():
    """Conservation every step of the paper's world with co-location, T_repr = 20 (births,
    stacking, wall deaths, starvation); per-cell stacking occurs."""
    wc = WC.replace(rows=40, cols=60, slots=300, n_initial=150, repr_steps=20)
    orc = oracle.OracleWorld(wc)
    res, pop = int(orc.st["resources"].sum()), int(orc.st["alive"].sum())
    tot = {"births": 0, "deaths_wall": 0, "deaths_energy": 0}
    stacked = 0
    for _ in range(400):
        r = orc.step()
        assert r["status"] == 0 and r["deferred_no_cell"] == 0 and r["deferred_claim"] == 0
        assert r["resources"] == res - r["eaten"] + r["grown"]
        assert r["population"] == pop + r["births"] - r["deaths_energy"] - r["deaths_age"] - r["deaths_wall"]
        res, pop = r["resources"], r["population"]
        for k in tot:
            tot[k] += r[k]
        live = orc.st["alive"] == 1
        stacked = max(stacked, int(np.bincount(orc.st["cell"][live]).max(initial=0)))
    assert tot["births"] > 0 and tot["deaths_wall"] > 0 and tot["deaths_energy"] > 0, tot
    assert stacked >= 2
