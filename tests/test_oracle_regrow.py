"""Pins for the oracle's regrowth phase ("p(x,y) = p_I(x,y)*c(x) + c";
BASELINE configs[0] step function f and linear latitude).

Pinned by: closed-form thresholds, scipy's convolve2d for the
neighbour count, Monte Carlo growth frequencies within 3 sigma of the closed-form
probability, brute-force per-cell recomputation from independently pinned pieces, and the
worked regrowth-only trajectories of SURVEY.md §8c C.7.
"""
import json
import math
import os

import numpy as np
import pytest
from scipy.signal import convolve2d

import oracle
import workloads

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "contract_c7.json")))
M61 = 2**61 - 1


def disc(r2):
    k = np.zeros((7, 7), np.int64)
    for dy in range(-3, 4):
        for dx in range(-3, 4):
            if (dy, dx) != (0, 0) and dy * dy + dx * dx <= r2:
                k[dy + 3, dx + 3] = 1
    return k


def sig(R):
    idx = np.flatnonzero(R.ravel())
    return len(idx), int(sum(int(i) for i in idx) % M61)


def test_disc_has_12_cells():
    assert disc(4).sum() == 12       # Euclidean radius 2 (R4)
    assert disc(1).sum() == 4        # the paper's "4 direct neighbors"


@pytest.mark.parametrize("H", [20, 200, 1600, 2048, 8192])
def test_threshold_closed_form(H):
    T = oracle.thresholds(workloads.WorldConfig(rows=H, cols=40))
    th = GOLD["thresholds"]
    assert list(T[0]) == th["top_row"]
    assert list(T[H - 1]) == th["bottom_row"]
    # monotone in class and in latitude (lat grows towards the bottom row)
    assert np.all(np.diff(T.astype(np.int64), axis=1) >= 0)
    assert np.all(np.diff(T.astype(np.int64), axis=0) >= 0)
    # class 0 is spontaneous growth only: floor(1e-5 * 2^32)
    assert np.all(T[:, 0] == 42949)


def test_threshold_mid_rows():
    th = GOLD["thresholds"]
    assert list(oracle.thresholds(workloads.WorldConfig(rows=20, cols=40))[10]) == th["H20_y10"]
    assert list(oracle.thresholds(workloads.WorldConfig(rows=200, cols=40))[100]) == th["H200_y100"]


def test_threshold_saturates_at_p_one():
    wc = workloads.WorldConfig(rows=4, cols=8, f_value=(1.0, 1.0, 1.0, 1.0), spontaneous=0.0)
    assert np.all(oracle.thresholds(wc)[-1] == 0xFFFFFFFF)


@pytest.mark.parametrize("r2", [1, 2, 4, 5, 8])
def test_neighbour_count_matches_convolve2d(r2):
    rng = np.random.default_rng(r2)
    wc = workloads.WorldConfig(rows=13, cols=24, regrow_r2=r2)
    R = (rng.random((13, 24)) < 0.4).astype(np.uint8)
    K = convolve2d(R.astype(np.int64), disc(r2), mode="same", boundary="fill", fillvalue=0)
    for y in range(13):
        for x in range(24):
            assert oracle.neighbour_count(wc, R, y, x) == K[y, x]


def test_class_of_step_function():
    wc = workloads.tiny()
    # f(0)=0, f(1..2)=0.01, f(3..4)=0.05, f(>=5)=0.1  (BASELINE configs[0])
    assert [oracle.class_of(wc, k) for k in range(13)] == [0, 1, 1, 2, 2, 3, 3, 3, 3, 3, 3, 3, 3]


def test_regrow_bruteforce_per_cell():
    rng = np.random.default_rng(5)
    wc = workloads.WorldConfig(rows=17, cols=36, seeds=(99,))
    T = oracle.thresholds(wc)
    R = (rng.random((17, 36)) < 0.3).astype(np.uint8)
    K = convolve2d(R.astype(np.int64), disc(4), mode="same")
    for t in (0, 3, 1000):
        Rn, grown = oracle.regrow(wc, t, R)
        exp = R.copy()
        for y in range(17):
            for x in range(36):
                if R[y, x]:
                    continue
                k = K[y, x]
                cls = 0 if k == 0 else 1 if k <= 2 else 2 if k <= 4 else 3
                u = oracle.cell_draw(99, oracle.P_REGROW, t, y * 36 + x)
                exp[y, x] = 1 if u < T[y, cls] else 0
        assert np.array_equal(Rn, exp)
        assert grown == int(exp.sum() - R.sum())
        assert np.all(Rn >= R)  # regrowth never removes a resource


def test_monte_carlo_bottom_row_dense_neighbourhood():
    # bottom row (lat = 1.0); every empty target has k = 6 >= 5 -> p = 0.1 + 1e-5
    H, W = 5, 400
    R = np.ones((H, W), np.uint8)
    R[H - 1, 0::2] = 0
    R[H - 1, :2] = 1
    R[H - 1, -2:] = 1
    wc = workloads.WorldConfig(rows=H, cols=W, seeds=(3,))
    targets = np.flatnonzero(R[H - 1] == 0)
    for x in targets:
        assert oracle.neighbour_count(wc, R, H - 1, int(x)) >= 5
    hits = n = 0
    for t in range(2500):
        Rn, _ = oracle.regrow(wc, t, R)
        hits += int(Rn[H - 1, targets].sum())
        n += len(targets)
    p = (0.1 + 1e-5)
    p_eff = math.floor(p * 2**32) / 2**32
    sd = math.sqrt(n * p_eff * (1 - p_eff))
    assert abs(hits - n * p_eff) < 3 * sd


def test_monte_carlo_isolated_cells_spontaneous():
    # an empty world: every cell has k = 0 -> p = c = 1e-5 regardless of latitude
    wc = workloads.WorldConfig(rows=200, cols=400, seeds=(11,))
    R = np.zeros((200, 400), np.uint8)
    hits = n = 0
    for t in range(100):
        _, g = oracle.regrow(wc, t, R)
        hits += g
        n += R.size
    p_eff = 42949 / 2**32
    sd = math.sqrt(n * p_eff)
    assert abs(hits - n * p_eff) < 3 * sd


def test_regrow_only_trajectory_tiny_golden():
    wc = workloads.tiny().replace(slots=0, n_initial=0)
    w = oracle.OracleWorld(wc)
    R = w.st["resources"].copy()
    g = GOLD["tiny_seed0"]
    assert R.sum() == g["initial_resources"]
    assert "".join(map(str, R[0])) == g["row0_bits"]
    got = [[0, *sig(R)]]
    for t in range(5):
        R, _ = oracle.regrow(wc, t, R)
        got.append([t + 1, *sig(R)])
    assert got == g["regrow_only"]


def test_initial_resources_goldens():
    for seed, n in GOLD["initial_resources_200x400_rho0.1"].items():
        wc = workloads.regrowth_micro().replace(seeds=(int(seed),))
        assert oracle.OracleWorld(wc).st["resources"].sum() == n


def test_regrow_only_trajectory_200x400_golden():
    wc = workloads.regrowth_micro()
    R = oracle.OracleWorld(wc).st["resources"].copy()
    want = {t: (n, s) for t, n, s in GOLD["regrow_only_200x400_seed2"]}
    assert sig(R) == want[0]
    for t in range(1000):
        R, _ = oracle.regrow(wc, t, R)
        if t + 1 in want:
            assert sig(R) == want[t + 1], t + 1
