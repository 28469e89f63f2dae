"""Pins for the oracle's initialisation orc_init ("randomly placed",
"initialized randomly once"; readings R24 and C.1 in DESIGN.md §3).

Anchored outside orc_init:
* the worked values of SURVEY.md §8c C.7 (tests/golden/contract_c7.json, computed by the
  survey author's independent implementation): the initial cells in slot order and slot 0's
  first four weights, bit for bit;
* a restatement from the separately pinned primitives (the per-cell draw, pinned to cuRAND,
  and the INIT_W Gaussians, pinned by C.7's z values and by moments): the N0 smallest
  (INIT_PLACE draw, cell) keys among the empty cells in ascending order, and every initial
  weight w_j = (float)(0.1 * z_j) keyed by the agent's INITIAL cell (not its slot), with
  sigma a standard deviation.
A descending sort, slot-keyed draws or sigma taken as a variance each fail one of these.
"""
import json
import os

import numpy as np

import oracle
import workloads

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "contract_c7.json")))["tiny_seed0"]


def test_init_cells_and_first_weights_match_c7_golden():
    wc = workloads.tiny()
    st = oracle.OracleWorld(wc).state()
    n0 = wc.n_initial
    assert int(st["resources"].sum()) == GOLD["initial_resources"]
    assert "".join(str(int(v)) for v in st["resources"][0]) == GOLD["row0_bits"]
    assert st["alive"][:n0].tolist() == [1] * n0 and not st["alive"][n0:].any()
    assert st["cell"][:n0].tolist() == GOLD["initial_cells"]
    w = st["weights"][0, :4].astype(np.float32)
    assert w.tobytes() == np.asarray(GOLD["slot0_w0_3"], np.float32).tobytes()
    assert np.all(st["weights"][n0:] == 0)
    assert np.all(st["energy"][:n0] == wc.e_init) and np.all(st["age"] == 0) and np.all(st["repr"] == 0)
    assert np.all(st["h"] == 0) and np.all(st["c"] == 0)


def _placement_restated(wc, seed):
    """N0 smallest (draw(INIT_PLACE, 0, cell), cell) among empty cells, ascending (R24)."""
    R = oracle.OracleWorld(wc.replace(seeds=(seed,))).st["resources"]
    cells = np.flatnonzero(R.reshape(-1) == 0)
    keys = sorted((oracle.cell_draw(seed, oracle.P_INIT_PLACE, 0, int(c)), int(c)) for c in cells)
    return [c for _, c in keys[:wc.n_initial]]


def test_init_placement_restated_from_pinned_draws():
    for wc, seed in ((workloads.tiny(), 0), (workloads.tiny().replace(rows=24, cols=48, slots=64, n_initial=60), 7)):
        st = oracle.OracleWorld(wc.replace(seeds=(seed,))).state()
        assert st["cell"][:wc.n_initial].tolist() == _placement_restated(wc, seed)


def test_init_weights_restated_from_pinned_gaussians():
    wc = workloads.tiny()
    st = oracle.OracleWorld(wc).state()
    P = wc.n_params
    for i in range(wc.n_initial):
        z = oracle.gauss(0, oracle.P_INIT_W, 0, int(st["cell"][i]), P)  # keyed by the initial cell
        expect = (wc.init_weight_std * z).astype(np.float32)
        assert st["weights"][i].tobytes() == expect.tobytes(), f"slot {i}"
