"""Lab-environment evaluation of evolved agents, batched on the device (SURVEY.md §8(f)
NEXT-4; §3.3 "Evaluation in lab environments", Appendix D.3).

* Greediness (§3.3.1, "Does the density of resources affect agents' greediness?"): a single
  agent that cannot reproduce, resource regeneration deactivated, three lab environments
  that differ in their initial resources; greediness G = C_r / T_r over non-overlapping
  20-step windows (sim_get_greediness).  Per agent, a one-way ANOVA over the three
  conditions (its trials as samples) and Tukey's HSD; an agent whose low- and high-density
  greediness differ significantly with G(low) > G(high) is a "sustainable forager", one
  with no significant difference an "opportunistic traveler" (§3.3.1).
* Peer pressure (§3.3.2, "Does peer-pressure lead to greediness?"): the high-density task
  with reproduction off and on (T_repr = 20); efficiency E = resources consumed per
  individual of the trial (the focal agent and its offspring), compared over agents and
  trials (and over all densities, Appendix D.3 Fig. 7).

Every trial is one world of a batched handle (n_worlds = genomes x trials per condition, one
handle per condition): the device steps them all at once; each world's seed is its trial
seed (the lab grid's Bernoulli resources come from it).  The focal agent is injected by
sim_set_state at the grid centre with the genome's weights and zero recurrent state.
Unstated lab parameters follow SPEC.md's lab module defaults (40x40 grid, densities 5 / 15 /
30 % of cells, 1000-step trials, 10 trials), all arguments here.
"""
from __future__ import annotations

import dataclasses

import numpy as np

from . import sim

DENSITIES = {"low": 0.05, "medium": 0.15, "high": 0.30}


@dataclasses.dataclass
class LabConfig:
    rows: int = 40
    cols: int = 40
    trial_steps: int = 1000
    trials: int = 10
    densities: tuple = (("low", 0.05), ("medium", 0.15), ("high", 0.30))
    seed: int = 7
    pressure_slots: int = 64  # population cap of a reproduction trial


def sample_genomes(state: dict, n: int, seed: int = 0) -> np.ndarray:
    """n genomes (canonical weights) drawn uniformly without replacement from the live agents
    of a (one-world) state, e.g. the end of a natural run."""
    st = {k: (v[0] if isinstance(v, np.ndarray) and v.ndim >= 2 and k != "resources" else v) for k, v in state.items()}
    alive = np.flatnonzero(st["alive"] == 1)
    rng = np.random.default_rng(seed)
    pick = rng.choice(alive, size=min(n, alive.size), replace=False)
    return np.ascontiguousarray(st["weights"][pick])


def lab_world_config(base, cfg: LabConfig, density: float, n_worlds: int, seed0: int, reproduce: bool):
    """The WorldConfig of a batch of lab trials: regrowth off, one focal agent, reproduction
    off (T_repr beyond the trial) or on (T_repr = 20 with the base physiology)."""
    return base.replace(rows=cfg.rows, cols=cfg.cols, init_resource_p=density,
                        f_value=(0.0, 0.0, 0.0, 0.0), spontaneous=0.0,
                        seeds=tuple(seed0 + k for k in range(n_worlds)),
                        slots=cfg.pressure_slots if reproduce else 1, n_initial=0,
                        repr_steps=20 if reproduce else 1 << 30, steps=cfg.trial_steps,
                        name="lab")


def _inject(world, wc, genomes: np.ndarray, trials: int):
    """World g * trials + k: genome g alone at the grid centre, recurrent state zero."""
    st = world.get_state()
    n = world.n_worlds
    st["alive"][:] = 0
    st["alive"][:, 0] = 1
    st["cell"][:, 0] = (wc.rows // 2) * wc.cols + wc.cols // 2
    st["energy"][:, 0] = wc.e_init
    for f in ("age", "repr"):
        st[f][:, 0] = 0
    for f in ("last_action", "ate"):
        st[f][:, 0] = 0
    st["h"][:] = 0
    st["c"][:] = 0
    st["logits"][:] = 0
    for w in range(n):
        st["weights"][w, 0] = genomes[w // trials]
    world.set_state(st)


def run_condition(base, genomes: np.ndarray, cfg: LabConfig, density: float, reproduce: bool, seed0: int,
                  device: int = 0) -> dict:
    """All trials of one condition as one batched handle: per world the greediness counts of
    the focal agent (reproduction off), the resources consumed, the individuals of the trial
    and the end state's weights (for the no-mutation invariant)."""
    G, K = genomes.shape[0], cfg.trials
    wc = lab_world_config(base, cfg, density, G * K, seed0, reproduce)
    world = sim.World(wc, device=device, log_capacity=cfg.trial_steps + 8)
    _inject(world, wc, genomes, K)
    res0 = world.get_state(("resources",))["resources"].reshape(G * K, -1).sum(axis=1)
    world.step(cfg.trial_steps)
    log = world.step_log(0, cfg.trial_steps)
    T, C = world.greediness()
    end = world.get_state(("alive", "weights", "resources"))
    world.destroy()
    eaten = log["eaten"].sum(axis=0)
    births = log["births"].sum(axis=0)
    return {"T_r": T[:, 0].reshape(G, K), "C_r": C[:, 0].reshape(G, K), "eaten": eaten.reshape(G, K),
            "individuals": (1 + births).reshape(G, K), "births": births.reshape(G, K),
            "resources_start": res0.reshape(G, K), "resources_series": log["resources"].T.reshape(G, K, -1),
            "end_weights0": end["weights"][:, 0].reshape(G, K, -1), "end_alive0": end["alive"][:, 0].reshape(G, K)}


def greediness(T: np.ndarray, C: np.ndarray) -> np.ndarray:
    """G = C_r / T_r (nan where the agent never saw a resource)."""
    T = np.asarray(T, np.float64)
    return np.where(T > 0, np.asarray(C, np.float64) / np.where(T > 0, T, 1.0), np.nan)


def classify(g_by_condition: dict, alpha: float = 0.05) -> dict:
    """One agent: ANOVA of its greediness over the conditions (trials as samples), Tukey's
    HSD, and the §3.3.1 classification.  g_by_condition: name -> per-trial G (nan = undefined)."""
    from scipy import stats
    names = list(g_by_condition)
    samples = [np.asarray(g_by_condition[k], np.float64) for k in names]
    samples = [s[~np.isnan(s)] for s in samples]
    if any(s.size < 2 for s in samples):
        return {"class": "excluded (greediness undefined)", "anova_p": None}
    if np.ptp(np.concatenate(samples)) == 0:  # identical greediness everywhere: ANOVA degenerate
        return {"class": "opportunistic traveler (no differences)", "anova_p": 1.0,
                "means": {k: float(s.mean()) for k, s in zip(names, samples)}}
    exact = all(s.std() == 0 for s in samples)  # no within-condition spread: any gap is certain
    p = 0.0 if exact else float(stats.f_oneway(*samples).pvalue)
    out = {"anova_p": p, "means": {k: float(s.mean()) for k, s in zip(names, samples)}}
    if p >= alpha:
        out["class"] = "opportunistic traveler (no differences)"
        return out
    lo, hi = names.index("low"), names.index("high")
    if exact:
        p_lh = 0.0 if samples[lo].mean() != samples[hi].mean() else 1.0
    else:
        p_lh = float(stats.tukey_hsd(*samples).pvalue[lo, hi])
    out["tukey_low_high_p"] = p_lh
    if p_lh < alpha and samples[lo].mean() > samples[hi].mean():
        out["class"] = "sustainable forager"
    else:
        out["class"] = "other difference"
    return out


def greediness_experiment(base, genomes: np.ndarray, cfg: LabConfig = LabConfig(), device: int = 0) -> dict:
    """§3.3.1 for every genome: per condition the trials' greediness, then the classification."""
    per = {}
    raw = {}
    for i, (name, dens) in enumerate(cfg.densities):
        r = run_condition(base, genomes, cfg, dens, False, cfg.seed * 1000003 + i * 100003, device)
        raw[name] = r
        per[name] = greediness(r["T_r"], r["C_r"])
    agents = [classify({k: per[k][g] for k in per}) for g in range(genomes.shape[0])]
    return {"greediness": per, "agents": agents, "raw": raw,
            "sustainable": sum(a["class"] == "sustainable forager" for a in agents)}


def pressure_experiment(base, genomes: np.ndarray, cfg: LabConfig = LabConfig(), device: int = 0,
                        densities=None) -> dict:
    """§3.3.2 (and Appendix D.3 over all densities): efficiency with reproduction off and on."""
    from scipy import stats
    out = {}
    for i, (name, dens) in enumerate(cfg.densities):
        if densities is not None and name not in densities:
            continue
        arms = {}
        for j, rep in enumerate((False, True)):
            r = run_condition(base, genomes, cfg, dens, rep, cfg.seed * 7919 + i * 104729 + j * 1299709, device)
            arms["on" if rep else "off"] = {"efficiency": r["eaten"] / r["individuals"], "births": r["births"],
                                            "raw": r}
        off, on = arms["off"]["efficiency"].mean(axis=1), arms["on"]["efficiency"].mean(axis=1)
        test = stats.ttest_rel(on, off) if off.size > 1 and np.any(on != off) else None
        out[name] = {"arms": arms, "mean_off": float(off.mean()), "mean_on": float(on.mean()),
                     "paired_p": None if test is None else float(test.pvalue)}
    return out
