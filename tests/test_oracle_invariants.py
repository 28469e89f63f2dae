"""Invariants of whole oracle trajectories:
R_{t+1} = R_t + grown - eaten, A_{t+1} = A_t + births - deaths, exclusive occupancy,
A <= S, determinism and exact resume.  Full trajectories themselves are "parity
unpinned" by the paper: these invariants, the per-phase pins and the
scripted walks are what pins them.
"""
import numpy as np
import pytest

import oracle
import workloads


def check_trajectory(wc, steps):
    w = oracle.OracleWorld(wc)
    R = int(w.st["resources"].sum())
    A = int(w.st["alive"].sum())
    recs = []
    for _ in range(steps):
        was_alive = w.st["alive"].copy() == 1
        r = w.step()
        assert r["status"] == 0
        R = R + r["grown"] - r["eaten"]
        A = A + r["births"] - r["deaths_energy"] - r["deaths_age"]
        assert R == r["resources"] == int(w.st["resources"].sum())
        assert A == r["population"] == int(w.st["alive"].sum())
        assert A <= wc.slots
        cells = w.st["cell"][w.st["alive"] == 1]
        assert len(np.unique(cells)) == len(cells)
        assert np.all((cells >= 0) & (cells < wc.rows * wc.cols))
        assert r["eaten"] == int(w.st["ate"][was_alive].sum())
        recs.append(r)
    return w, recs


def test_tiny_100_steps_invariants_and_golden_grown0():
    wc = workloads.tiny()
    w, recs = check_trajectory(wc, 100)
    assert recs[0]["grown"] == 3          # regrowth runs first
    assert w.t == 100


def test_paper_scale_first_steps_invariants():
    check_trajectory(workloads.paper_scale(), 25)


def test_determinism_and_resume():
    wc = workloads.tiny()
    a = oracle.OracleWorld(wc)
    b = oracle.OracleWorld(wc)
    for _ in range(40):
        a.step()
        b.step()
    snap = b.state()
    for _ in range(60):
        a.step()
    c = oracle.OracleWorld(wc, state=snap)
    for _ in range(60):
        c.step()
    for k in snap:
        if k == "t":
            assert a.t == c.t == 100
        else:
            assert np.array_equal(a.st[k], c.st[k]), k


def test_extinction_is_not_an_error():
    wc = workloads.no_regrowth(workloads.tiny()).replace(init_resource_p=0.0)
    w = oracle.OracleWorld(wc)
    for t in range(101):
        r = w.step()
        assert r["status"] == 0
    assert w.st["alive"].sum() == 0 and r["population"] == 0


def test_validation_rejects_bad_fields():
    wc = workloads.tiny()
    assert oracle.validate(wc)[0] == 0
    for kw, field in [(dict(rows=1), "rows"), (dict(cols=42), "cols"), (dict(init_resource_p=1.5), "init_resource_p"),
                      (dict(n_initial=40), "n_initial"), (dict(spontaneous=-0.1), "spontaneous"),
                      (dict(obs_radius=4), "obs_radius"), (dict(hidden=33), "hidden")]:
        rc, msg = oracle.validate(wc.replace(**kw))
        assert rc == oracle.E_INVALID and field in msg
    # more initial agents than empty cells is invalid
    with pytest.raises(ValueError):
        oracle.OracleWorld(wc.replace(init_resource_p=1.0))
