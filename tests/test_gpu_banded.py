"""Banded mode (BASELINE configs[3]'s latitude bands): one world split
into G row bands on one GPU (the one-GPU band backend: the bands' exchanges are device
reads between the bands' buffers, in the same phase order the multi-GPU mode separates
with NCCL barriers).  The banded world must equal the unbanded one KEYED BY CELL (slot
layouts differ, SURVEY.md §8c C.6 "Multi-GPU"): the resource grid, the set of occupied
cells and, per agent, energy, age, repr, last action, ate, h, c, logits and weights bit for
bit, and the per-step records summed over the bands equal the unbanded records exactly.
Covered: G = 2, 4, 8 over 150+ steps of the paper-scale world (births, cross-band
migration), uneven band rows, a binding population cap (capacity deferrals decided across
bands), resume by set_state, and the local slot pool overflow error.
"""
import numpy as np
import pytest

import workloads

pytestmark = pytest.mark.gpu

sim = pytest.importorskip("paper_2302_09334_b200.sim")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device (no CPU fallback exists)")


AGENT_FIELDS = ("energy", "age", "repr", "last_action", "ate", "h", "c", "logits", "weights")


def by_cell(st, w=0):
    """{cell: slot} of the live agents of world w of a state dict."""
    alive = np.flatnonzero(st["alive"][w])
    return dict(zip(st["cell"][w][alive].tolist(), alive.tolist()))


def compare_by_cell(a, b, where=""):
    assert a["t"] == b["t"], where
    assert np.array_equal(a["resources"][0], b["resources"][0]), f"{where}: resources differ at " \
        f"{np.argwhere(a['resources'][0] != b['resources'][0])[:5].tolist()}"
    ca, cb = by_cell(a), by_cell(b)
    assert ca.keys() == cb.keys(), f"{where}: occupied cells differ: {sorted(set(ca) ^ set(cb))[:10]}"
    cells = sorted(ca)
    sa = np.array([ca[c] for c in cells], np.int64)
    sb = np.array([cb[c] for c in cells], np.int64)
    for f in AGENT_FIELDS:
        if f not in a:
            continue
        va, vb = a[f][0][sa], b[f][0][sb]
        same = np.array_equal(va.view(np.uint8), vb.view(np.uint8)) if va.dtype.kind == "f" else np.array_equal(va, vb)
        assert same, f"{where}: {f} differs (first cell {cells[int(np.flatnonzero((va != vb).reshape(len(cells), -1).any(axis=1))[0])]})"


def run_pair(wc, bands, steps, every, log_cap=4096, start_state=None):
    ref = sim.World(wc, log_capacity=log_cap)
    ban = sim.World(wc, log_capacity=log_cap, bands=bands)
    if start_state is not None:
        ref.set_state(start_state)
        ban.set_state(start_state)
    t0 = ref.t
    compare_by_cell(ref.get_state(), ban.get_state(), "start")
    done = 0
    while done < steps:
        k = min(every, steps - done)
        ref.step(k)
        ban.step(k)
        done += k
        compare_by_cell(ref.get_state(), ban.get_state(), f"t={t0 + done}")
    lr = ref.step_log(t0, steps)[:, 0]
    lb = ban.step_log(t0, steps)[:, 0]
    for f in sim.RECORD_FIELDS:
        assert np.array_equal(lr[f], lb[f]), f"record {f} differs at steps {np.flatnonzero(lr[f] != lb[f])[:5] + t0}"
    ref.destroy()
    ban.destroy()
    return lr


@pytest.mark.parametrize("G", [2, 4, 8])
def test_banded_paper_scale_equals_unbanded(G):
    wc = workloads.paper_scale()
    lr = run_pair(wc, dict(n_bands=G), steps=160, every=20)
    assert int(lr["births"].sum()) > 100
    print(f"G={G}: population {int(lr['population'][-1])} at t=160, {int(lr['births'].sum())} births")


def test_banded_uneven_rows_capped_population():
    """Uneven bands (3, 37, 60, 100 rows) and a population cap that binds: capacity
    deferrals are decided from every band's counts (R22 is global)."""
    wc = workloads.paper_scale().replace(slots=1300, n_initial=1000)
    lr = run_pair(wc, dict(n_bands=4, band_rows=[0, 3, 40, 100, 200]), steps=200, every=25)
    assert int(lr["deferred_capacity"].sum()) > 0 and int(lr["births"].sum()) > 0


def test_banded_resume_from_injected_state():
    """set_state of a mid-run unbanded state into a banded world (agents distributed by
    cell row), then both continue identically."""
    wc = workloads.paper_scale()
    src = sim.World(wc)
    src.step(90)
    st = src.get_state()
    src.destroy()
    run_pair(wc, dict(n_bands=3), steps=60, every=20, start_state=st)


def test_banded_tiny_world_hd8():
    """The lane-group policy kernel (Hd = 8) and a 5x5 window in 4 bands of a 20x40 grid."""
    wc = workloads.tiny().replace(slots=64, n_initial=40, repr_steps=5, e_repr_gt=10200)
    lr = run_pair(wc, dict(n_bands=4), steps=100, every=10)
    assert int(lr["births"].sum()) > 0


def test_banded_slot_pool_overflow_is_reported():
    wc = workloads.paper_scale()
    with pytest.raises(sim.SimError) as ei:
        w = sim.World(wc, bands=dict(n_bands=4, band_slots=100))
        w.step(1)
        w.synchronize()
    assert ei.value.status == sim.SIM_E_OOM


def test_banded_invalid_rows():
    wc = workloads.paper_scale()
    with pytest.raises(sim.SimError) as ei:
        sim.World(wc, bands=dict(n_bands=2, band_rows=[0, 2, 200]))
    assert ei.value.status == sim.SIM_E_INVALID


def test_banded_rebalance_continues_the_unbanded_trajectory():
    """banded.rebalanced(): equal rows for 80 steps, then agent-weighted rows (the population
    gathers at the rich bottom rows), 80 more steps -- keyed by cell equal to the unbanded
    world at every checkpoint, the records of the second half equal."""
    from paper_2302_09334_b200 import banded
    wc = workloads.paper_scale()
    ref = sim.World(wc)
    ban = sim.World(wc, bands=dict(n_bands=4))
    ref.step(80)
    ban.step(80)
    compare_by_cell(ref.get_state(), ban.get_state(), "t=80")
    ban = banded.rebalanced(ban)
    rows = ban.bands["band_rows"]
    assert rows != banded.equal_band_rows(wc.rows, 4)
    compare_by_cell(ref.get_state(), ban.get_state(), "rebalanced t=80")
    for k in range(4):
        ref.step(20)
        ban.step(20)
        compare_by_cell(ref.get_state(), ban.get_state(), f"t={100 + 20 * k}")
    lr, lb = ref.step_log(80, 80)[:, 0], ban.step_log(80, 80)[:, 0]
    for f in sim.RECORD_FIELDS:
        assert np.array_equal(lr[f], lb[f]), f
    ref.destroy()
    ban.destroy()


def test_banded_large_world_equals_unbanded():
    """BASELINE configs[3] itself (1600x3200, 64,000 initial agents, 262,144 slots) as 8
    latitude bands on this GPU (local slot pools of 56,000) against the unbanded world: 30
    steps, records equal every step, the state keyed by cell equal at the end (all fields but
    the 17.8 GB weight array)."""
    wc = workloads.large_world()
    ref = sim.World(wc)
    ban = sim.World(wc, bands=dict(n_bands=8, band_slots=56000))
    ref.step(30)
    ban.step(30)
    lr, lb = ref.step_log(0, 30)[:, 0], ban.step_log(0, 30)[:, 0]
    for f in sim.RECORD_FIELDS:
        assert np.array_equal(lr[f], lb[f]), f
    fields = tuple(f for f in sim.STATE_FIELDS if f != "weights")
    compare_by_cell(ref.get_state(fields), ban.get_state(fields), "large world t=30")
    assert int(lr["births"].sum()) > 0 or int(lr["population"][-1]) > 0
    ref.destroy()
    ban.destroy()
