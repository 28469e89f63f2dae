"""Seeded synthetic workloads shared by the CUDA path's harness and the CPU oracle.

This module holds ONLY inputs: the BASELINE.json configs written out as plain
parameter records, and seeded generators of random world states used to inject
states in parity tests.  It contains none of the method's arithmetic (no regrowth,
policy, movement, physiology or reproduction rule) and imports neither the product
package nor oracle/.

Config records follow BASELINE.json:configs[0..4].  Field names
match both C structs (include/sim.h `sim_config`, oracle/oracle.h `orc_config`).
"""
from __future__ import annotations

import dataclasses
from typing import Optional, Sequence

import numpy as np

INT32_MAX = 2**31 - 1


@dataclasses.dataclass
class WorldConfig:
    rows: int
    cols: int
    seeds: Sequence[int] = (0,)
    init_resource_p: float = 0.10
    regrow_r2: int = 4                       # Euclidean radius 2 -> 12-cell disc
    f_class_min_k: Sequence[int] = (0, 1, 3, 5)
    f_value: Sequence[float] = (0.0, 0.01, 0.05, 0.1)
    lat_top: float = 0.1
    lat_bottom: float = 1.0
    spontaneous: float = 1e-5
    slots: int = 0
    n_initial: int = 0
    obs_radius: int = 3
    hidden: int = 32
    n_actions: int = 5
    init_weight_std: float = 0.1
    mutation_std: float = 0.02
    e_init: int = 10000                      # milli-units: 10.0
    e_decay: int = 100                       # 0.1 per step
    e_gain: int = 1000                       # +1 per resource
    e_repr_gt: int = 12000                   # reproduce when energy > 12 ...
    e_death_le: int = 0                      # die when energy <= 0
    e_max: int = INT32_MAX                   # no clip
    repr_steps: int = 20                     # ... for 20 consecutive steps
    max_age: int = 1000
    # the paper's own world (App. B.4); BASELINE's world leaves them off
    climate_alpha: float = 0.0               # > 0: exponential climate (alpha^x + 1)/(alpha + 1)
    death_steps: int = 0                     # > 0: the death timer T_death (else immediate death)
    lethal_walls: int = 0                    # 1: moving off the grid kills
    network: int = 0                         # 1: the paper's CNN-LSTM, sampled (NEXT-2; r 7, Hd 4)
    colocate: int = 0                        # 1: co-location, offspring on the parent's cell (network 1)
    steps: int = 100                         # run length named by the config
    name: str = ""

    @property
    def n_worlds(self) -> int:
        return len(self.seeds)

    @property
    def n_inputs(self) -> int:
        if self.network == 1:
            return 15 * 15 * 3
        w = 2 * self.obs_radius + 1
        return 2 * w * w

    @property
    def n_params(self) -> int:
        if self.network == 1:  # the paper's count
            return 2445
        I, Hd, A = self.n_inputs, self.hidden, self.n_actions
        return 4 * Hd * I + 4 * Hd * Hd + 4 * Hd + A * Hd + A

    def replace(self, **kw) -> "WorldConfig":
        return dataclasses.replace(self, **kw)


def tiny() -> WorldConfig:
    """BASELINE.json configs[0]: 20x40, seed 0, rho 0.15, 32 slots / 16 agents, 5x5x2 obs, Hd 8, 100 steps."""
    return WorldConfig(rows=20, cols=40, seeds=(0,), init_resource_p=0.15, slots=32, n_initial=16,
                       obs_radius=2, hidden=8, steps=100, name="tiny")


def paper_scale() -> WorldConfig:
    """BASELINE.json configs[1]: 200x400, seed 1, rho 0.1, 8192 slots / 1000 agents, 7x7x2 obs, Hd 32, 10,000 steps."""
    return WorldConfig(rows=200, cols=400, seeds=(1,), init_resource_p=0.10, slots=8192, n_initial=1000,
                       obs_radius=3, hidden=32, steps=10000, name="paper_scale")


def paper_world() -> WorldConfig:
    """The paper's own natural environment (App. B.4; SURVEY.md §8(f)
    NEXT-1), on this build's mechanics: 400x200 read as H = 200 rows x W = 400 (R2); 1000
    slots, 330 initial agents; "16 0000" resources read as 16,000 = Bernoulli(0.2) of the
    80,000 cells; regrowth p = p_I c(x) + c with p_I = 0.002 * 1[I >= 1] over the 4 direct
    neighbours (the disc of r^2 = 1; class 1 iff k >= 1, SPEC's indicator reading of
    1_{I=1}), c(x) = (200^x + 1)/201 with x = 1 at the bottom row, c = 5e-5; E0 = E_max = 3,
    decay 0.025, +1 per resource (milli-units: 3000, 25, 1000, clip 3000); reproduction after
    T_repr = 140 steps above E_min = 0; death after T_death = 200 steps below 0 (energy <= -1
    milli-unit) or at age > 650; sigma = 0.02; lethal walls; an LSTM of hidden size 4.
    Deviations kept from this build's mechanics: exclusive occupancy with the
    child on an adjacent cell (the paper: the parent's cell), a 7x7x2 window (the paper:
    15x15 with walls) and the LSTM + linear head with argmax (the paper: a CNN-LSTM with
    softmax sampling, NEXT-2)."""
    return WorldConfig(rows=200, cols=400, seeds=(1,), init_resource_p=0.2, regrow_r2=1,
                       f_class_min_k=(0, 1, 5, 5), f_value=(0.0, 0.002, 0.0, 0.0), spontaneous=5e-5,
                       climate_alpha=200.0, slots=1000, n_initial=330, obs_radius=3, hidden=4,
                       mutation_std=0.02, e_init=3000, e_decay=25, e_gain=1000, e_repr_gt=0, e_death_le=-1,
                       e_max=3000, repr_steps=140, death_steps=200, max_age=650, lethal_walls=1,
                       steps=1_000_000, name="paper_world")


def paper_world_cnn() -> WorldConfig:
    """The paper's own world with the paper's own agents (SURVEY.md §8(f) NEXT-1 + NEXT-2):
    paper_world() with the CNN-LSTM of PAPER.md:346-350 -- a 15x15x3 window (resources,
    agents, walls), conv 3x3/2 (4) -> avgpool 2/1 -> conv 3x3/2 (8) -> avgpool 2/1 -> 72,
    ++ previous action (5) ++ ate (1) -> LSTM(4) -> [78 ++ 4] -> dense 8 tanh -> dense 5 ->
    softmax(50 logits), sampled; 2445 parameters per agent."""
    return paper_world().replace(network=1, obs_radius=7, hidden=4, name="paper_world_cnn")


def paper_world_coloc() -> WorldConfig:
    """The paper's world, agents and reproduction (SURVEY.md §8(f) NEXT-1 complete, with
    NEXT-2): paper_world_cnn() with co-location -- any number of agents per cell (the
    agent channel counts them, "including their number"), no collision
    exclusion, one agent per resource cell eats (a lottery), the offspring
    appears on its parent's cell."""
    return paper_world_cnn().replace(colocate=1, name="paper_world_coloc")


def regrowth_micro(rows: int = 200, cols: int = 400) -> WorldConfig:
    """BASELINE.json configs[2]: no agents, seed 2, rho 0.1; grids 200x400, 2048x4096, 8192x16384; 1000 steps."""
    return WorldConfig(rows=rows, cols=cols, seeds=(2,), init_resource_p=0.10, slots=0, n_initial=0,
                       obs_radius=3, hidden=32, steps=1000, name=f"regrowth_{rows}x{cols}")


REGROWTH_GRIDS = ((200, 400), (2048, 4096), (8192, 16384))


def large_world() -> WorldConfig:
    """BASELINE.json configs[3]: 1600x3200, seed 3, rho 0.1, 262,144 slots / 64,000 agents, 2000 steps."""
    return WorldConfig(rows=1600, cols=3200, seeds=(3,), init_resource_p=0.10, slots=262144, n_initial=64000,
                       obs_radius=3, hidden=32, steps=2000, name="large_world")


def ensemble(seeds: Optional[Sequence[int]] = None) -> WorldConfig:
    """BASELINE.json configs[4]: 64 independent 200x400 worlds, seeds 100-163, paper-scale parameters, 5000 steps."""
    seeds = tuple(range(100, 164)) if seeds is None else tuple(seeds)
    return WorldConfig(rows=200, cols=400, seeds=seeds, init_resource_p=0.10, slots=8192, n_initial=1000,
                       obs_radius=3, hidden=32, steps=5000, name="ensemble")


def ensemble_shard(n_ranks: int, rank: int, seeds: Optional[Sequence[int]] = None) -> Sequence[int]:
    """Contiguous split of the ensemble's seeds over ranks."""
    seeds = tuple(range(100, 164)) if seeds is None else tuple(seeds)
    n = len(seeds)
    lo = (n * rank) // n_ranks
    hi = (n * (rank + 1)) // n_ranks
    return seeds[lo:hi]


def no_regrowth(cfg: WorldConfig) -> WorldConfig:
    """Regrowth switched off (f = 0, spontaneous = 0), for scripted walks."""
    return cfg.replace(f_value=(0.0, 0.0, 0.0, 0.0), spontaneous=0.0)


# --------------------------------------------------------------------------------------
# Canonical state containers and seeded random states (for injection via set_state).
# --------------------------------------------------------------------------------------

def empty_state(cfg: WorldConfig) -> dict:
    """Zeroed canonical state arrays for one world (layout of include/sim.h `sim_state`)."""
    S, Hd, P, A = cfg.slots, cfg.hidden, cfg.n_params, cfg.n_actions
    return {
        "t": 0,
        "resources": np.zeros((cfg.rows, cfg.cols), np.uint8),
        "alive": np.zeros(S, np.uint8),
        "cell": np.zeros(S, np.int32),
        "energy": np.zeros(S, np.int32),
        "age": np.zeros(S, np.int32),
        "repr": np.zeros(S, np.int32),
        "last_action": np.zeros(S, np.uint8),
        "ate": np.zeros(S, np.uint8),
        "h": np.zeros((S, Hd), np.float32),
        "c": np.zeros((S, Hd), np.float32),
        "weights": np.zeros((S, P), np.float32),
        "logits": np.zeros((S, A), np.float32),
        "low": np.zeros(S, np.int32),
    }


def random_state(cfg: WorldConfig, seed: int, n_alive: Optional[int] = None, density: float = 0.5,
                 weight_std: float = 0.1, hc_std: float = 0.5, t: int = 0) -> dict:
    """A seeded random canonical state: Bernoulli(density) resources, n_alive agents on
    distinct random cells in random slots, N(0, weight_std^2) weights, random h/c, energy
    and ages.  Used by the one-step (M3) and scenario parity tests."""
    rng = np.random.default_rng(seed)
    st = empty_state(cfg)
    H, W, S = cfg.rows, cfg.cols, cfg.slots
    st["t"] = int(t)
    st["resources"][:] = (rng.random((H, W)) < density).astype(np.uint8)
    if n_alive is None:
        n_alive = S // 2
    n_alive = min(n_alive, S, H * W)
    slots = rng.choice(S, size=n_alive, replace=False) if n_alive else np.zeros(0, np.int64)
    cells = rng.choice(H * W, size=n_alive, replace=False) if n_alive else np.zeros(0, np.int64)
    st["alive"][slots] = 1
    st["cell"][slots] = cells.astype(np.int32)
    st["energy"][slots] = rng.integers(100, 20000, size=n_alive).astype(np.int32)
    st["age"][slots] = rng.integers(0, 1001, size=n_alive).astype(np.int32)
    st["repr"][slots] = rng.integers(0, 25, size=n_alive).astype(np.int32)
    st["last_action"][slots] = rng.integers(0, 5, size=n_alive).astype(np.uint8)
    st["h"][slots] = (rng.standard_normal((n_alive, cfg.hidden)) * hc_std).astype(np.float32).clip(-1, 1)
    st["c"][slots] = (rng.standard_normal((n_alive, cfg.hidden)) * hc_std * 2).astype(np.float32)
    st["weights"][:] = (rng.standard_normal((S, cfg.n_params)) * weight_std).astype(np.float32)
    return st
