"""Pins of the Appendix C metrics fold (oracle/metrics.py) — SPEC.md metrics examples and a
scripted oracle trajectory whose histogram and death ages follow from the rules by hand."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import oracle  # noqa: E402
from oracle import metrics  # noqa: E402
from scenario import E, build_state, forced, small_config  # noqa: E402


def test_movement_bin_spec_examples():
    # SPEC.md metrics.movement_bin: (0,0)->(0,0) bin 0; (0,0)->(3,4): d = 7 -> bin 2; d = 50 -> 16
    W = 100
    assert metrics.movement_bin(0, 0, W) == 0
    assert metrics.movement_bin(0, 3 * W + 4, W) == 2
    assert metrics.movement_bin(0, 20 * W + 30, W) == 16
    assert metrics.movement_bin(5 * W + 9, 5 * W + 6, W) == 1  # d = 3, either direction
    assert metrics.movement_bin(0, 2, W) == 0


def test_life_expectancy_spec_examples():
    assert metrics.life_expectancy([100, 200, 300]) == 200
    assert metrics.life_expectancy([]) is None
    assert metrics.life_expectancy([650]) == 650


def scripted_walk():
    """A walks east every step (d = 50 over window 0 -> bin 16), B stays (bin 0), C starves:
    10,000 - 100 per step with e_init lowered to 1,000 dies in step 9 at age 10."""
    wc = small_config(rows=6, cols=60, slots=4)
    st = build_state(wc, [dict(slot=0, y=2, x=2), dict(slot=1, y=4, x=30), dict(slot=2, y=0, x=50, energy=1000)])
    return wc, st


def run_oracle_fold(wc, st, steps):
    ow = oracle.OracleWorld(wc, state=st)
    fold = metrics.MetricsFold(wc.cols)
    f = forced(wc, {0: E})
    for _ in range(steps):
        before = {k: ow.st[k].copy() for k in ("alive", "cell", "age")} | {"t": ow.t}
        r = ow.step(forced=f)
        assert r["status"] == 0
        fold.feed(before, {k: ow.st[k] for k in ("alive", "cell", "age")} | {"t": ow.t})
    return ow, fold


def test_scripted_walk_histogram_and_death_age():
    wc, st = scripted_walk()
    ow, fold = run_oracle_fold(wc, st, 50)
    h = fold.hist[0]
    assert h[16] == 1 and h[0] == 1 and h.sum() == 2
    assert fold.death_age_sum[9] == 10 and fold.deaths[9] == 1
    assert sum(fold.deaths.values()) == 1
    assert ow.st["cell"][0] == 2 * wc.cols + 52
    assert fold.life_expectancy_windows()[0] == 10


# ------------------------------------------------------------------- greediness (NEXT-3)
def test_greediness_fold_scripted():
    """Regrowth off.  A stays 2 cells west of a resource (in its 5x5 field of view, never
    eats) for 40 steps: T_r = 2, C_r = 0.  B walks east onto a resource in step 5 (window 0)
    and then stays on the bare cell with nothing in view: T_r = 1 (window 0 only), C_r = 1.
    D has nothing in view at all: T_r = C_r = 0."""
    wc = small_config(rows=12, cols=60, slots=4).replace(obs_radius=2)
    st = build_state(wc, [dict(slot=0, y=2, x=5), dict(slot=1, y=8, x=20), dict(slot=2, y=8, x=50)])
    st["resources"][2, 7] = 1         # A's: 2 east, never reached
    st["resources"][8, 25] = 1        # B's: 5 east of B
    w = oracle.OracleWorld(wc, state=st)
    fold = metrics.GreedinessFold(wc)
    for t in range(40):
        acts = {1: E} if t < 5 else {}
        before = w.state()
        w.step(forced=forced(wc, acts))
        fold.feed(before, w.state())
    assert (fold.T[0], fold.C[0]) == (2, 0)
    assert (fold.T[1], fold.C[1]) == (1, 1)
    assert (fold.T[2], fold.C[2]) == (0, 0)
