"""Pins of the paper's own world in the oracle (App. B.4,
lines 311-338; workloads.paper_world): the exponential climate, the 4-neighbour indicator
regrowth with c = 5e-5, the clipped energy, the death timer, lethal walls.

Anchored by SPEC.md's worked values (climate 1.0 / 0.0099502 / 0.075334 and the ratio
100.5, regrowth 0.00005 / 0.00205, energy 2.975 / clip to 3.0) and closed forms of scripted
single-agent walks (starvation in step 319 under the death-timer reading R32: energy below
E_min = 0, i.e. <= -1 milli-unit, for T_death = 200 consecutive steps; an agent fed every 40
steps lives to the age cap, 651 > 650 in step 650)."""
import math

import numpy as np

import oracle
import workloads
from scenario import N, STAY, build_state, forced

TWO32 = 2.0 ** 32


def climate_cfg(rows):
    """f(class 1) = 1, no spontaneous growth: T[y][1] = floor(c(y) 2^32) exposes c(x)."""
    return workloads.paper_world().replace(rows=rows, f_value=(0.0, 1.0, 0.0, 0.0), spontaneous=0.0)


def test_climate_spec_values():
    T = oracle.thresholds(climate_cfg(201))
    c = T[:, 1].astype(np.float64) / TWO32
    assert T[200, 1] == 0xFFFFFFFF                       # x = 1 (bottom): c = 1.0 (clipped at 2^32-1)
    assert abs(c[0] - 2.0 / 201.0) < 1e-9                 # x = 0 (top): 0.0099502
    assert abs(c[0] - 0.0099502) < 1e-7
    assert abs(c[100] - (math.sqrt(200.0) + 1.0) / 201.0) < 1e-9  # x = 0.5: 0.075334
    assert abs(c[100] - 0.075334) < 1e-6
    assert abs(1.0 / c[0] - 100.5) < 1e-5                 # c(bottom) / c(top)
    assert np.all(np.diff(c) >= 0)                        # monotone towards the bottom


def test_regrowth_probabilities_spec_values():
    wc = workloads.paper_world()
    T = oracle.thresholds(wc)
    bottom, top = wc.rows - 1, 0
    assert T[bottom, 0] == math.floor(0.00005 * TWO32)              # n = 0: spontaneous only
    assert T[bottom, 1] == math.floor((0.002 * 1.0 + 0.00005) * TWO32)  # n >= 1, c = 1: 0.00205
    assert T[top, 1] == math.floor((0.002 * (2.0 / 201.0) + 0.00005) * TWO32)
    # the indicator over the 4 direct neighbours: class 1 iff k >= 1 (k <= 4 < 5)
    assert [oracle.class_of(wc, k) for k in range(5)] == [0, 1, 1, 1, 1]
    R = np.zeros((5, 5), np.uint8)
    R[1, 2] = R[2, 1] = R[3, 3] = 1  # two direct neighbours of (2, 2), one diagonal
    small = wc.replace(rows=5, cols=8)
    R8 = np.zeros((5, 8), np.uint8)
    R8[:, :5] = R
    assert oracle.neighbour_count(small, R8, 2, 2) == 2 and oracle.neighbour_count(small, R8, 4, 0) == 0


def walk(wc, st, steps, feed_every=0, act=STAY):
    w = oracle.OracleWorld(wc, state=st)
    recs = []
    for t in range(steps):
        if feed_every and t % feed_every == 0 and w.st["alive"][0]:
            c = int(w.st["cell"][0])
            w.st["resources"][c // wc.cols, c % wc.cols] = 1
        recs.append(w.step(forced(wc, {0: act})))
        if not w.st["alive"][0]:
            break
    return w, recs


def lone(wc):
    return wc.replace(rows=10, cols=12, slots=1, n_initial=0, f_value=(0.0, 0.0, 0.0, 0.0), spontaneous=0.0)


def test_energy_step_spec_values():
    wc = lone(workloads.paper_world())
    w, _ = walk(wc, build_state(wc, [dict(slot=0, y=5, x=5)]), 1)
    assert w.st["energy"][0] == 2975                      # (3.0, no eat) -> 2.975
    w, _ = walk(wc, build_state(wc, [dict(slot=0, y=5, x=5, energy=2500)], resources=[(5, 5)]), 1)
    assert w.st["energy"][0] == 3000                      # (2.5, eat) -> min(3, 3.475) = 3.0


def test_starvation_by_the_death_timer_in_step_319():
    wc = lone(workloads.paper_world())
    w, recs = walk(wc, build_state(wc, [dict(slot=0, y=5, x=5)]), 400)
    died = [i for i, r in enumerate(recs) if r["deaths_energy"]]
    assert died == [319] and len(recs) == 320
    assert w.st["energy"][0] == 3000 - 25 * 320           # it kept decaying below 0
    assert w.st["low"][0] == 200


def test_fed_every_40_steps_lives_to_the_age_cap():
    wc = lone(workloads.paper_world())
    w, recs = walk(wc, build_state(wc, [dict(slot=0, y=5, x=5)]), 700, feed_every=40)
    assert [i for i, r in enumerate(recs) if r["deaths_age"]] == [650]
    assert sum(r["deaths_energy"] for r in recs) == 0
    assert sum(r["deferred_capacity"] for r in recs) > 0  # eligible from step 139, but S = 1


def test_lethal_wall():
    wc = lone(workloads.paper_world())
    w, recs = walk(wc, build_state(wc, [dict(slot=0, y=0, x=5)]), 1, act=N)
    assert recs[0]["deaths_wall"] == 1 and w.st["alive"][0] == 0 and recs[0]["population"] == 0
    blocked = wc.replace(lethal_walls=0)
    w, recs = walk(blocked, build_state(blocked, [dict(slot=0, y=0, x=5)]), 1, act=N)
    assert recs[0]["deaths_wall"] == 0 and w.st["alive"][0] == 1 and w.st["cell"][0] == 5


def test_paper_world_invariants_300_steps():
    wc = workloads.paper_world()
    w = oracle.OracleWorld(wc)
    A = int(w.st["alive"].sum())
    R = int(w.st["resources"].sum())
    assert A == 330 and abs(R - 16000) < 4 * math.sqrt(80000 * 0.2 * 0.8)
    for _ in range(300):
        rec = w.step()
        A2, R2 = int(w.st["alive"].sum()), int(w.st["resources"].sum())
        assert A2 == A + rec["births"] - rec["deaths_energy"] - rec["deaths_age"] - rec["deaths_wall"]
        assert R2 == R + rec["grown"] - rec["eaten"] and A2 <= wc.slots
        cells = w.st["cell"][w.st["alive"] == 1]
        assert np.unique(cells).size == cells.size
        A, R = A2, R2
