"""Appendix C metrics of a trajectory, as plain folds over the oracle's per-step states.

TEST INFRASTRUCTURE ONLY: imported by tests/ (and nothing in the product path).  It reads
the oracle's canonical state before and after each step and shares no code with the CUDA
library (include/sim.h: sim_get_move_hist, sim_step_record.death_age_sum).

* Movement (Appendix C: "the Manhattan distance between the position at the last
  timestep of the window and the position at the beginning", "we then make 17 bins";
  SPEC.md metrics.movement_bin, d in [0, 50] -> floor(d / 3)).  Windows of 50 steps are
  aligned to multiples of 50 from step 0 (SPEC design decision); an agent counts in a window
  iff it is alive through it ("every agent alive during a time window"; born or dying
  inside it excludes it, SPEC design decision) — read off the state as: alive at the start
  of step 50k and at the end of step 50k+49 with its age grown by exactly 50.
* Greediness (§3.3 lab set-up: "non-overlapping fixed windows of 20 timesteps",
  T_r = windows with "at least one resource in its field of view", C_r = windows in which
  "the agent consumed at least one resource", G = C_r / T_r): windows aligned to multiples
  of 20 from step 0; the field of view is the agent's observation (its resource channel,
  after the step's regrowth, R10/R11) at every step of the window it is alive; a window is
  closed for the agents alive at the start of its last step; a newborn starts from zero.
* Life expectancy (Appendix C: "average of age of agent that died during a large
  time window of 500 timesteps"; SPEC.md metrics.life_expectancy): per step the sum of the
  ages at death (an agent that dies in step t was alive at its start and its age was
  incremented before the death test: age at death = age at step start + 1).
"""
import numpy as np

WINDOW, BINS, LIFE_WINDOW, GREED_WINDOW = 50, 17, 500, 20


def movement_bin(c0: int, c1: int, cols: int) -> int:
    """Bin of the Manhattan distance between cells c0 and c1 (row-major, `cols` wide)."""
    d = abs(c1 // cols - c0 // cols) + abs(c1 % cols - c0 % cols)
    return min(d // 3, BINS - 1)


def life_expectancy(ages):
    """Mean age at death, or None without deaths (SPEC.md metrics.life_expectancy)."""
    ages = list(ages)
    return sum(ages) / len(ages) if ages else None


class MetricsFold:
    """Feed (state before step t, state after it) for consecutive steps from a window start."""

    def __init__(self, cols: int):
        self.cols = cols
        self.hist = {}            # window k -> int64[17]
        self.death_age_sum = {}   # step t -> sum of ages at death
        self.deaths = {}          # step t -> number of deaths
        self._snap = None         # (alive mask, cells, ages) at the current window's start

    def feed(self, before: dict, after: dict):
        t = int(before["t"])
        a0, a1 = before["alive"] == 1, after["alive"] == 1
        age0, age1 = before["age"].astype(np.int64), after["age"].astype(np.int64)
        if t % WINDOW == 0:
            self._snap = (a0.copy(), before["cell"].astype(np.int64).copy(), age0.copy())
        died = a0 & (~a1 | (age1 != age0 + 1))
        self.death_age_sum[t] = int((age0[died] + 1).sum())
        self.deaths[t] = int(died.sum())
        if t % WINDOW == WINDOW - 1 and self._snap is not None:
            s_alive, s_cell, s_age = self._snap
            keep = s_alive & a1 & (age1 == s_age + WINDOW)
            h = np.zeros(BINS, np.int64)
            c1 = after["cell"].astype(np.int64)
            for i in np.flatnonzero(keep):
                h[movement_bin(int(s_cell[i]), int(c1[i]), self.cols)] += 1
            self.hist[t // WINDOW] = h

    def life_expectancy_windows(self):
        """Mean age at death per complete 500-step window (None for a window without deaths)."""
        out = {}
        for t, s in self.death_age_sum.items():
            k = t // LIFE_WINDOW
            tot, n = out.get(k, (0, 0))
            out[k] = (tot + s, n + self.deaths[t])
        return {k: (tot / n if n else None) for k, (tot, n) in out.items()}


class GreedinessFold:
    """Feed (state before step t, state after it) for consecutive steps; the oracle's own
    regrowth and observation functions give the field of view (test infrastructure)."""

    def __init__(self, wc):
        self.wc = wc
        S = wc.slots
        self.T = np.zeros(S, np.int64)
        self.C = np.zeros(S, np.int64)
        self.seen = np.zeros(S, bool)
        self.ate = np.zeros(S, bool)

    def feed(self, before: dict, after: dict):
        import oracle
        wc = self.wc
        t = int(before["t"])
        a0 = before["alive"] == 1
        Rp, _ = oracle.regrow(wc, t, before["resources"])  # R' of step t (what the policy sees)
        O = np.zeros((wc.rows, wc.cols), np.uint8)
        cells = before["cell"][a0]
        O.reshape(-1)[cells] = 1
        wd2 = (2 * wc.obs_radius + 1) ** 2
        for i in np.flatnonzero(a0):
            c = int(before["cell"][i])
            x = oracle.observe(wc, Rp, O, c // wc.cols, c % wc.cols)
            if x[:wd2].any():
                self.seen[i] = True
        # consumption of the agents alive at step start (a newborn in a freed slot has age 0)
        same = a0 & (after["alive"] == 1) & (after["age"] == before["age"] + 1)
        self.ate[same & (after["ate"] == 1)] = True
        if t % GREED_WINDOW == GREED_WINDOW - 1:
            self.T[a0] += self.seen[a0]
            self.C[a0] += self.ate[a0]
            self.seen[:] = False
            self.ate[:] = False
        born = (after["alive"] == 1) & (after["age"] == 0)
        self.T[born] = self.C[born] = 0
        self.seen[born] = self.ate[born] = False
