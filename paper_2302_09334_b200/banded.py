"""One world in latitude bands over several GPUs, one band per process (include/sim.h
"Banded mode"; BASELINE configs[3]).

Every rank (one process per GPU, an initialised torch.distributed group, rank = band index)
creates its band of the same world.  The ranks exchange their bands' IPC export blobs
(all_gather_object) so each band can pull its neighbours' halo rows, boundary claims and
outboxes directly over NVLink, and rank 0's NCCL unique id (broadcast_object_list) for the
library's own communicator, whose stream-ordered token exchanges separate the phases of a
step.  After that, step(n) on every rank runs n world steps with no host synchronisation.

The host-side helpers (row splits, splitting a whole-world state into bands, merging the
ranks' band states) are plain numpy and are what tests/test_multiproc.py checks with gloo on
CPU; the library's data path needs the GPUs.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import sim


def equal_band_rows(rows: int, n_bands: int) -> list:
    """The library's default split: band b owns rows [b*H//G, (b+1)*H//G)."""
    return [b * rows // n_bands for b in range(n_bands + 1)]


def agent_weighted_rows(agent_rows: np.ndarray, rows: int, n_bands: int, min_rows: int = 3) -> list:
    """Row boundaries giving each band about 1/G of the agents (agent_rows: the row of every
    live agent), each band at least `min_rows` rows (the halo depth)."""
    hist = np.bincount(np.asarray(agent_rows, np.int64), minlength=rows)[:rows]
    cum = np.cumsum(hist)
    tot = int(cum[-1]) if cum.size else 0
    b = [0]
    for k in range(1, n_bands):
        y = int(np.searchsorted(cum, tot * k / n_bands)) + 1 if tot else k * rows // n_bands
        y = max(y, b[-1] + min_rows)
        y = min(y, rows - (n_bands - k) * min_rows)
        b.append(y)
    b.append(rows)
    return b


def band_of_rows(band_rows, y: np.ndarray) -> np.ndarray:
    """The band owning each row in y."""
    return np.searchsorted(np.asarray(band_rows[1:]), np.asarray(y), side="right")


def split_state(state: dict, band_rows, band: int, cols: int) -> dict:
    """The share of a whole-world state (one world, canonical layout, leading world axis
    optional) a band holds: its rows of the resources (others 0) and its agents compacted
    into slots 0.. in ascending slot order — what sim_get_state returns for that band."""
    st = {k: (v[0] if isinstance(v, np.ndarray) and v.ndim >= 1 and k != "t" and v.shape[0] == 1 else v)
          for k, v in state.items()}
    y0, y1 = band_rows[band], band_rows[band + 1]
    out = {"t": st["t"]}
    res = np.zeros_like(st["resources"])
    res[y0:y1] = st["resources"][y0:y1]
    out["resources"] = res
    live = np.flatnonzero(st["alive"] == 1)
    mine = live[(st["cell"][live] // cols >= y0) & (st["cell"][live] // cols < y1)]
    for k, v in st.items():
        if k in ("t", "resources"):
            continue
        z = np.zeros_like(v)
        z[:mine.size] = v[mine]
        out[k] = z
    return out


def merge_band_states(states: list, band_rows, cols: int) -> dict:
    """The whole world from the bands' states (band order): resources from each band's rows,
    the live agents concatenated in band order into slots 0.. (cells are global, so the
    result equals the unbanded world keyed by cell)."""
    base = states[0]
    out = {"t": base["t"], "resources": np.zeros_like(base["resources"])}
    for b, st in enumerate(states):
        y0, y1 = band_rows[b], band_rows[b + 1]
        out["resources"][y0:y1] = st["resources"][y0:y1]
        assert st["t"] == base["t"], "bands at different steps"
    for k in base:
        if k in ("t", "resources"):
            continue
        parts = [st[k][st["alive"] == 1] for st in states]
        z = np.zeros_like(base[k])
        cat = np.concatenate(parts) if parts else z[:0]
        assert cat.shape[0] <= z.shape[0], "more agents than slots"
        z[:cat.shape[0]] = cat
        out[k] = z
    return out


def rebalanced(world, min_rows: int = 3, band_slots: int = 0):
    """Agent-weighted rebalancing of a banded world whose bands are all on this GPU (SURVEY.md
    §8(e) E.2 "rebalance by agent count"): the state is read out (sim_get_state merges the
    bands keyed by cell), a new banded handle is created with row boundaries giving every
    band about 1/G of the live agents (agent_weighted_rows) and the state is written in
    (sim_set_state splits it); the old handle is destroyed.  The trajectory continues
    exactly as the unbanded world's (cells, not slots, key every draw, R9).  The new handle's
    step log starts at the rebalancing step and the movement windows in progress are not
    measured (as after any sim_set_state).  Returns the new sim.World."""
    if not world.bands:
        raise ValueError("rebalanced() needs a banded world")
    G = int(world.bands["n_bands"])
    st = world.get_state()
    live = st["alive"][0] == 1
    rows = agent_weighted_rows(st["cell"][0][live] // world.wc.cols, world.wc.rows, G, min_rows)
    bands = dict(world.bands, band_rows=rows)
    if band_slots:
        bands["band_slots"] = band_slots
    new = sim.World(world.wc, device=world.device, stream=world.stream, log_capacity=world.log_capacity,
                    bands=bands)
    world.destroy()
    new.set_state(st)
    return new


class BandedWorld:
    """This rank's band of one world split over the ranks of `dist` (one band per GPU)."""

    def __init__(self, wc, dist, device: int, stream=None, band_rows=None, band_slots: int = 0,
                 log_capacity: int = 0, group=None):
        import torch
        self.dist, self.group = dist, group
        G = dist.get_world_size(group)
        b = dist.get_rank(group)
        self.n_bands, self.band = G, b
        self.band_rows = list(band_rows) if band_rows is not None else equal_band_rows(wc.rows, G)
        if stream is None:  # the library and NCCL's barriers share torch's current stream
            stream = torch.cuda.current_stream(device)
        self.stream = stream
        self.world = sim.World(wc, device=device, stream=stream, log_capacity=log_capacity,
                               bands=dict(n_bands=G, band_first=b, band_local=1, band_rows=self.band_rows,
                                          band_slots=band_slots))
        L = sim.lib()
        need = ctypes.c_size_t()
        sim._check(L.sim_band_export(self.world.handle, b, None, ctypes.byref(need)))
        blob = ctypes.create_string_buffer(need.value)
        sim._check(L.sim_band_export(self.world.handle, b, blob, ctypes.byref(need)))
        blobs = [None] * G
        dist.all_gather_object(blobs, bytes(blob.raw), group=group)
        for k, bl in enumerate(blobs):
            if k != b:
                buf = ctypes.create_string_buffer(bl, len(bl))
                sim._check(L.sim_band_import(self.world.handle, k, buf, len(bl)))
        uid = [None]
        if b == 0:
            raw = ctypes.create_string_buffer(128)
            sim._check(L.sim_band_nccl_id(raw))
            uid[0] = bytes(raw.raw)
        dist.broadcast_object_list(uid, src=0, group=group)
        idbuf = ctypes.create_string_buffer(uid[0], 128)
        sim._check(L.sim_band_nccl_init(self.world.handle, idbuf, G, b))

    @property
    def t(self):
        return self.world.t

    def step(self, n: int = 1):
        self.world.step(n)

    def get_state(self, fields=sim.STATE_FIELDS) -> dict:
        """This band's rows and agents (slots 0..)."""
        return self.world.get_state(fields)

    def gather_state(self, fields=sim.STATE_FIELDS) -> dict | None:
        """The whole world on rank 0 (None elsewhere): every band's state merged by cell."""
        st = sim.world_view(self.get_state(fields), 0)
        parts = [None] * self.n_bands
        self.dist.all_gather_object(parts, st, group=self.group)
        if self.band != 0:
            return None
        return merge_band_states(parts, self.band_rows, self.world.wc.cols)

    def __getattr__(self, name):  # step_log (this band's counters), synchronize, destroy, ...
        return getattr(self.world, name)
