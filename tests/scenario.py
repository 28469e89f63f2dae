"""Helpers that build hand-made world states (scripted walks and the C.6b scenarios).

Pure input construction: no rule of the method is implemented here.  The same states
are fed to the oracle (CPU tests) and to the CUDA library (GPU tests).
"""
import numpy as np

import workloads


def small_config(rows=6, cols=8, slots=8, regrowth=False, seed=0, **kw):
    wc = workloads.tiny().replace(rows=rows, cols=cols, slots=slots, n_initial=0, seeds=(seed,), **kw)
    if not regrowth:
        wc = workloads.no_regrowth(wc)
    return wc


def build_state(wc, agents, resources=None, t=0, zero_weights=True, weight_seed=0):
    """agents: list of dicts {slot, y, x, energy?, age?, repr?}; resources: iterable of (y, x)."""
    st = workloads.empty_state(wc)
    st["t"] = t
    if resources is not None:
        for (y, x) in resources:
            st["resources"][y, x] = 1
    if not zero_weights:
        rng = np.random.default_rng(weight_seed)
        st["weights"][:] = (rng.standard_normal(st["weights"].shape) * 0.1).astype(np.float32)
    for a in agents:
        s = a["slot"]
        st["alive"][s] = 1
        st["cell"][s] = a["y"] * wc.cols + a["x"]
        st["energy"][s] = a.get("energy", wc.e_init)
        st["age"][s] = a.get("age", 0)
        st["repr"][s] = a.get("repr", 0)
    return st


def forced(wc, actions):
    """actions: dict slot -> action; every other slot forced to 0 (stay)."""
    f = np.zeros(wc.slots, np.uint8)
    for s, a in actions.items():
        f[s] = a
    return f


STAY, N, S, E, W = 0, 1, 2, 3, 4
