"""Pins for the oracle's movement, consumption, physiology, death and reproduction
(scenarios S1-S13).

Pinned by:
* a brute-force checker of the declarative movement rule (R14) on 3x3 worlds: an agent
  moves iff its action is non-stay, its target is in-grid and unoccupied at step start,
  and its key (MOVE draw, -cell) is the largest among all such claimants of the target;
* closed-form scripted single-agent walks (starvation at 0-based
  step 99, births at 21/41/61/81, age death at step 1000);
* hand-checkable scenarios S1-S13 whose outcome follows from the rules by hand;
* np.flatnonzero / sorting for the free-slot and birth ranking;
* sigma = 0 mutation giving a bit-identical child, and N(0,1) moments/KS of the deltas.
"""
import itertools
import math

import numpy as np
import pytest

import oracle
import workloads
from scenario import E, N, S, STAY, W, build_state, forced, small_config

DY = {0: 0, 1: -1, 2: 1, 3: 0, 4: 0}
DX = {0: 0, 1: 0, 2: 0, 3: 1, 4: -1}


def run1(wc, st, f=None):
    w = oracle.OracleWorld(wc, state=st)
    rec = w.step(f)
    return w.st, rec


# ----------------------------------------------------------------------------- movement
def declarative_moves(wc, st, actions, seed):
    """Independent statement of rule R14 (no claim buffer, no sequential pass)."""
    H, Wd = wc.rows, wc.cols
    occ = {int(st["cell"][s]) for s in range(wc.slots) if st["alive"][s]}
    claims = {}
    for s in range(wc.slots):
        if not st["alive"][s] or actions[s] == 0:
            continue
        y, x = divmod(int(st["cell"][s]), Wd)
        ty, tx = y + DY[int(actions[s])], x + DX[int(actions[s])]
        if not (0 <= ty < H and 0 <= tx < Wd) or ty * Wd + tx in occ:
            continue
        prio = oracle.draw4(seed, oracle.P_MOVE, int(st["t"]), int(st["cell"][s]))[0]
        claims.setdefault(ty * Wd + tx, []).append(((prio, -int(st["cell"][s])), s))
    final = {s: int(st["cell"][s]) for s in range(wc.slots) if st["alive"][s]}
    for tgt, cl in claims.items():
        final[max(cl)[1]] = tgt
    return final


def test_movement_bruteforce_3x3():
    rng = np.random.default_rng(0)
    wc = small_config(rows=3, cols=4, slots=9, e_init=50000)  # cols%4==0; use 3x3 region + a spare col
    n_cases = 0
    for n_agents in range(1, 10):
        for trial in range(300 if n_agents > 1 else 50):
            cells = rng.choice(9, n_agents, replace=False)
            agents = [dict(slot=i, y=int(c) // 3, x=int(c) % 3) for i, c in enumerate(cells)]
            st = build_state(wc, agents, t=int(rng.integers(0, 10**6)))
            acts = rng.integers(0, 5, wc.slots).astype(np.uint8)
            want = declarative_moves(wc, st, acts, wc.seeds[0])
            new, rec = run1(wc, st, acts)
            got = {s: int(new["cell"][s]) for s in range(wc.slots) if new["alive"][s]}
            assert got == want
            # invariants: exclusive occupancy; moves <= 1 cell; never into a start-occupied cell
            assert len(set(got.values())) == len(got)
            start = {int(st["cell"][s]) for s in want}
            for s, c in got.items():
                c0 = int(st["cell"][s])
                dy, dx = divmod(c, 4)[0] - divmod(c0, 4)[0], divmod(c, 4)[1] - divmod(c0, 4)[1]
                assert abs(dy) + abs(dx) <= 1
                if c != c0:
                    assert c not in start
            n_cases += 1
    assert n_cases > 2000


def test_swap_s1():
    wc = small_config()
    st = build_state(wc, [dict(slot=0, y=2, x=2), dict(slot=1, y=2, x=3)])
    new, _ = run1(wc, st, forced(wc, {0: E, 1: W}))
    assert new["cell"][0] == 2 * 8 + 2 and new["cell"][1] == 2 * 8 + 3


def test_chain_s2():
    wc = small_config()
    st = build_state(wc, [dict(slot=0, y=2, x=2), dict(slot=1, y=2, x=3)])
    new, _ = run1(wc, st, forced(wc, {0: E, 1: E}))
    assert new["cell"][0] == 2 * 8 + 2      # A's target was occupied at step start
    assert new["cell"][1] == 2 * 8 + 4      # B moved into an empty cell


def test_conflict_s3():
    wc = small_config()
    for t in range(50):
        st = build_state(wc, [dict(slot=0, y=2, x=1), dict(slot=1, y=2, x=3)], t=t)
        new, _ = run1(wc, st, forced(wc, {0: E, 1: W}))
        k0 = (oracle.draw4(0, oracle.P_MOVE, t, 2 * 8 + 1)[0], -(2 * 8 + 1))
        k1 = (oracle.draw4(0, oracle.P_MOVE, t, 2 * 8 + 3)[0], -(2 * 8 + 3))
        winner = 0 if k0 > k1 else 1
        assert new["cell"][winner] == 2 * 8 + 2
        assert new["cell"][1 - winner] == st["cell"][1 - winner]


def test_edge_blocked_s4():
    wc = small_config()
    st = build_state(wc, [dict(slot=0, y=0, x=3)])
    new, rec = run1(wc, st, forced(wc, {0: N}))
    assert new["alive"][0] == 1 and new["cell"][0] == 3
    assert new["energy"][0] == wc.e_init - wc.e_decay


# ------------------------------------------------------------------ consumption/physiology
def test_regrown_under_agent_is_eaten_s5():
    wc = small_config(regrowth=True).replace(f_value=(0.0, 0.0, 0.0, 0.0), spontaneous=1.0)
    st = build_state(wc, [dict(slot=0, y=3, x=3)])
    new, rec = run1(wc, st, forced(wc, {0: STAY}))
    assert new["ate"][0] == 1 and new["energy"][0] == wc.e_init + 900
    assert new["resources"][3, 3] == 0
    assert rec["eaten"] == 1 and rec["grown"] == 6 * 8


def test_move_onto_resource_s6():
    wc = small_config()
    st = build_state(wc, [dict(slot=0, y=3, x=3)], resources=[(3, 4), (0, 0)])
    new, rec = run1(wc, st, forced(wc, {0: E}))
    assert new["cell"][0] == 3 * 8 + 4 and new["ate"][0] == 1
    assert rec["eaten"] == 1 and new["resources"].sum() == 1 and rec["resources"] == 1


def test_starvation_s11_and_walk_i():
    wc = small_config()
    st = build_state(wc, [dict(slot=0, y=3, x=3, energy=100)])
    new, rec = run1(wc, st)
    assert new["alive"][0] == 0 and rec["deaths_energy"] == 1 and new["energy"][0] == 0
    # walk (i): never eats -> dies at 0-based step 99, the last step of the tiny run
    w = oracle.OracleWorld(wc, state=build_state(wc, [dict(slot=0, y=3, x=3)]))
    for t in range(100):
        r = w.step(forced(wc, {}))
        assert (r["deaths_energy"] == 1) == (t == 99)
    assert w.st["alive"][0] == 0


def test_age_death_s12():
    wc = small_config()
    st = build_state(wc, [dict(slot=0, y=3, x=3, energy=50000, age=1000)])
    new, rec = run1(wc, st)
    assert new["alive"][0] == 0 and rec["deaths_age"] == 1 and rec["deaths_energy"] == 0
    # energy takes precedence when both hold
    st = build_state(wc, [dict(slot=0, y=3, x=3, energy=100, age=1000)])
    _, rec = run1(wc, st)
    assert rec["deaths_energy"] == 1 and rec["deaths_age"] == 0


def test_repr_threshold_strict_s13():
    wc = small_config()
    st = build_state(wc, [dict(slot=0, y=3, x=3, energy=11100, repr=7)], resources=[(3, 3)])
    new, _ = run1(wc, st)
    assert new["energy"][0] == 12000 and new["repr"][0] == 0     # not > 12000
    st = build_state(wc, [dict(slot=0, y=3, x=3, energy=11101, repr=7)], resources=[(3, 3)])
    new, _ = run1(wc, st)
    assert new["repr"][0] == 8


def test_walk_ii_eats_every_step_births_at_21_41_61_81():
    wc = small_config(rows=5, cols=120, slots=8)
    st = build_state(wc, [dict(slot=0, y=2, x=0)], resources=[(2, x) for x in range(1, 120)])
    w = oracle.OracleWorld(wc, state=st)
    births = []
    for t in range(100):
        r = w.step(forced(wc, {0: E}))
        if r["births"]:
            births.append(t)
        assert w.st["ate"][0] == 1
    assert births == [21, 41, 61, 81]


def test_walk_iii_eats_every_10th_step_dies_of_age_at_1000():
    wc = small_config()
    w = oracle.OracleWorld(wc, state=build_state(wc, [dict(slot=0, y=3, x=3)]))
    max_e = 0
    for t in range(1001):
        if t % 10 == 9:
            w.st["resources"][3, 3] = 1
        r = w.step(forced(wc, {}))
        if t < 1000:
            assert w.st["alive"][0] == 1
            max_e = max(max_e, int(w.st["energy"][0]))
    assert r["deaths_age"] == 1 and w.st["alive"][0] == 0
    assert max_e == 10000 and r["births"] == 0


# ------------------------------------------------------------------------- reproduction
def test_shared_candidate_one_child_s7():
    wc = small_config(rows=6, cols=8)
    # parents at (2,1) and (2,3) — both eligible; the only free neighbour of each is (2,2)
    blockers = [(1, 1), (3, 1), (2, 0), (1, 3), (3, 3), (2, 4)]
    agents = [dict(slot=0, y=2, x=1, energy=20000, repr=19), dict(slot=1, y=2, x=3, energy=20000, repr=19)]
    for t in range(40):
        st = build_state(wc, agents, resources=blockers, t=t)
        new, rec = run1(wc, st, forced(wc, {}))
        # resources do not block themselves: blockers are resources, eaten? agents stay -> no
        assert rec["births"] == 1 and rec["deferred_claim"] == 1
        kids = [s for s in range(wc.slots) if new["alive"][s] and s > 1]
        assert kids == [2] and new["cell"][2] == 2 * 8 + 2
        k0 = (oracle.draw4(0, oracle.P_BIRTH, t, 2 * 8 + 1)[1], -(2 * 8 + 1))
        k1 = (oracle.draw4(0, oracle.P_BIRTH, t, 2 * 8 + 3)[1], -(2 * 8 + 3))
        win = 0 if k0 > k1 else 1
        assert new["repr"][win] == 0 and new["repr"][1 - win] == 20


def test_no_cell_s8():
    wc = small_config(rows=6, cols=8)
    agents = [dict(slot=0, y=0, x=0, energy=20000, repr=19), dict(slot=1, y=0, x=1), dict(slot=2, y=1, x=0)]
    st = build_state(wc, agents)
    new, rec = run1(wc, st, forced(wc, {}))
    assert rec["births"] == 0 and rec["deferred_no_cell"] == 1 and new["repr"][0] == 20
    # a resource also blocks the cell (R21: no resource after consumption)
    st = build_state(wc, [dict(slot=0, y=0, x=0, energy=20000, repr=19), dict(slot=1, y=0, x=1)],
                     resources=[(1, 0)])
    _, rec = run1(wc, st, forced(wc, {}))
    assert rec["deferred_no_cell"] == 1


def test_capacity_s9():
    wc = small_config(rows=6, cols=8, slots=3)
    agents = [dict(slot=i, y=1 + 2 * i, x=2 + 2 * i, energy=20000, repr=25) for i in range(3)]
    st = build_state(wc, agents)
    new, rec = run1(wc, st, forced(wc, {}))
    assert rec["births"] == 0 and rec["deferred_capacity"] == 3
    assert list(new["repr"]) == [26, 26, 26]
    assert new["alive"].sum() == 3


def test_death_frees_slot_for_birth_s10():
    wc = small_config(rows=6, cols=8, slots=3)
    agents = [dict(slot=0, y=1, x=1, energy=20000, repr=25), dict(slot=1, y=4, x=6, energy=100),
              dict(slot=2, y=4, x=2, energy=20000)]
    new, rec = run1(wc, build_state(wc, agents), forced(wc, {}))
    assert rec["deaths_energy"] == 1 and rec["births"] == 1
    assert new["alive"][1] == 1 and new["energy"][1] == wc.e_init and new["age"][1] == 0
    assert new["repr"][0] == 0


def test_birth_ranking_by_child_cell_into_ascending_free_slots():
    wc = small_config(rows=10, cols=16, slots=12)
    rng = np.random.default_rng(3)
    for trial in range(30):
        cells = rng.choice(10 * 16, 6, replace=False)
        parent_slots = rng.choice(12, 6, replace=False)
        agents = [dict(slot=int(s), y=int(c) // 16, x=int(c) % 16, energy=20000, repr=30)
                  for s, c in zip(parent_slots, cells)]
        st = build_state(wc, agents, t=trial)
        new, rec = run1(wc, st, forced(wc, {}))
        free = np.flatnonzero(st["alive"] == 0)
        newborn = [s for s in range(12) if new["alive"][s] and not st["alive"][s]]
        assert rec["births"] == len(newborn) == min(len(free), rec["births"] + rec["deferred_capacity"])
        # the k-th smallest child cell sits in the k-th smallest free slot
        child_cells = [int(new["cell"][s]) for s in newborn]
        assert newborn == list(free[:len(newborn)])
        assert child_cells == sorted(child_cells)


def test_mutation_sigma_zero_is_identity_and_parent_untouched():
    wc = small_config(rows=6, cols=8, slots=4).replace(mutation_std=0.0)
    st = build_state(wc, [dict(slot=1, y=2, x=2, energy=20000, repr=19)], zero_weights=False)
    parent_w = st["weights"][1].copy()
    new, rec = run1(wc, st, forced(wc, {}))
    assert rec["births"] == 1
    assert np.array_equal(new["weights"][0].view(np.uint32), parent_w.view(np.uint32))
    assert np.array_equal(new["weights"][1], parent_w)
    assert np.all(new["h"][0] == 0) and np.all(new["c"][0] == 0)


def test_mutation_deltas_are_gaussian():
    from scipy import stats
    wc = small_config(rows=6, cols=8, slots=8, hidden=32, obs_radius=3).replace(mutation_std=0.02)
    deltas = []
    for t in range(12):
        st = build_state(wc, [dict(slot=0, y=2, x=3, energy=20000, repr=19)], t=t)  # zero parent weights
        new, rec = run1(wc, st, forced(wc, {}))
        assert rec["births"] == 1
        deltas.append(new["weights"][1].astype(np.float64) / 0.02)
    z = np.concatenate(deltas)
    n = z.size
    assert abs(z.mean()) < 4 / math.sqrt(n)
    assert abs(z.var() - 1.0) < 4 * math.sqrt(2.0 / n) + 1e-6
    assert stats.kstest(z, "norm").pvalue > 1e-3
