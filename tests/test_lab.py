"""Lab evaluation (§3.3; SPEC.md lab module): the host
statistics on scripted greediness (CPU) and a small batched lab run on the GPU."""
import numpy as np
import pytest

import workloads
from paper_2302_09334_b200 import lab


def test_classify_scripted_greediness():
    rng = np.random.default_rng(1)
    # always eats what it sees: G = 1 everywhere -> degenerate ANOVA, not adaptive (SPEC example)
    a = lab.classify({"low": np.ones(10), "medium": np.ones(10), "high": np.ones(10)})
    assert a["class"].startswith("opportunistic")
    # eats only when few resources are visible: G(low) clearly above G(high) -> sustainable
    b = lab.classify({"low": 0.9 + 0.05 * rng.random(10), "medium": 0.6 + 0.05 * rng.random(10),
                      "high": 0.2 + 0.05 * rng.random(10)})
    assert b["class"] == "sustainable forager" and b["anova_p"] < 1e-6
    # noise only -> no significant difference
    c = lab.classify({k: 0.5 + 0.1 * rng.standard_normal(10) for k in ("low", "medium", "high")})
    assert c["class"].startswith("opportunistic") or c["anova_p"] >= 0.05
    # the opposite direction is a difference, not a sustainable forager
    d = lab.classify({"low": np.full(10, 0.2), "medium": np.full(10, 0.5), "high": np.full(10, 0.9)})
    assert d["class"] == "other difference"
    # never saw a resource in a condition: excluded
    e = lab.classify({"low": np.full(10, np.nan), "medium": np.ones(10), "high": np.ones(10)})
    assert e["class"].startswith("excluded")


def test_greediness_and_config():
    g = lab.greediness(np.array([[4, 0], [2, 5]]), np.array([[2, 0], [2, 0]]))
    assert g[0, 0] == 0.5 and np.isnan(g[0, 1]) and g[1, 0] == 1.0 and g[1, 1] == 0.0
    wc = lab.lab_world_config(workloads.paper_scale(), lab.LabConfig(), 0.15, 30, 100, False)
    assert (wc.rows, wc.cols, wc.slots, wc.n_initial, wc.spontaneous) == (40, 40, 1, 0, 0.0)
    assert wc.f_value == (0.0, 0.0, 0.0, 0.0) and wc.seeds == tuple(range(100, 130)) and wc.repr_steps > 10**6
    wr = lab.lab_world_config(workloads.paper_scale(), lab.LabConfig(), 0.30, 4, 0, True)
    assert wr.repr_steps == 20 and wr.slots == 64


@pytest.mark.gpu
def test_lab_batch_on_gpu():
    """3 genomes sampled from a natural paper-scale run (t = 300) x 3 densities x 3 trials
    of 200 steps: the batch equals each world run alone, the genomes are unchanged (no
    reproduction, no mutation), regrowth off keeps the resources non-increasing, the
    greediness counts are consistent (C_r <= T_r <= 10 windows), and the pressure arms
    run (births only with reproduction on)."""
    from paper_2302_09334_b200 import sim
    base = workloads.paper_scale()
    nat = sim.World(base)
    nat.step(300)
    genomes = lab.sample_genomes(nat.get_state(), 3, seed=4)
    nat.destroy()
    cfg = lab.LabConfig(trial_steps=200, trials=3)
    r = lab.run_condition(base, genomes, cfg, 0.15, False, 1000)
    assert np.all(r["C_r"] <= r["T_r"]) and np.all(r["T_r"] <= 10) and int(r["T_r"].sum()) > 0
    for g in range(3):
        for k in range(3):
            if r["end_alive0"][g, k]:  # the focal agent is never mutated (no reproduction)
                assert r["end_weights0"][g, k].tobytes() == genomes[g].tobytes()
    assert np.all(np.diff(r["resources_series"], axis=2) <= 0)
    # batch invariance: world (g=1, k=2) alone
    wc1 = lab.lab_world_config(base, cfg, 0.15, 1, 1000 + 1 * 3 + 2, False)
    one = sim.World(wc1, log_capacity=cfg.trial_steps + 8)
    lab._inject(one, wc1, genomes[1:2], 1)
    one.step(cfg.trial_steps)
    T1, C1 = one.greediness()
    eaten1 = int(one.step_log(0, cfg.trial_steps)["eaten"].sum())
    one.destroy()
    assert (int(T1[0, 0]), int(C1[0, 0]), eaten1) == (int(r["T_r"][1, 2]), int(r["C_r"][1, 2]), int(r["eaten"][1, 2]))
    p = lab.pressure_experiment(base, genomes, cfg, densities=("high",))
    assert int(p["high"]["arms"]["off"]["births"].sum()) == 0
    assert p["high"]["mean_on"] >= 0 and p["high"]["mean_off"] >= 0


@pytest.mark.gpu
def test_lab_with_the_papers_agents():
    """The paper's pipeline end to end on the device: a natural run of the paper's world with
    its own network and same-cell reproduction (paper_world_coloc), genomes sampled from it,
    the greediness experiment over the three densities (each agent classified by ANOVA +
    Tukey, §3.3.1) and the peer-pressure arms (§3.3.2) -- with the 2,445-parameter
    CNN-LSTM genomes, sampled actions and co-location."""
    from paper_2302_09334_b200 import sim
    base = workloads.paper_world_coloc()
    nat = sim.World(base)
    nat.step(300)
    genomes = lab.sample_genomes(nat.get_state(), 3, seed=2)
    nat.destroy()
    assert genomes.shape == (3, 2445)
    cfg = lab.LabConfig(trial_steps=200, trials=3)
    res = lab.greediness_experiment(base, genomes, cfg)
    assert len(res["agents"]) == 3 and all("class" in a for a in res["agents"])
    p = lab.pressure_experiment(base, genomes, cfg, densities=("high",))
    assert int(p["high"]["arms"]["off"]["births"].sum()) == 0
