"""Thin ctypes binding of libsim.so (include/sim.h).  Argument marshalling only: every
step of the world step runs in the library's CUDA kernels.  There is no CPU fallback —
if the extension cannot be loaded or no CUDA device is present, calls raise.

Names follow the C ABI: create / step / get_state / set_state / destroy, plus the test
and measurement hooks (forced actions, step log, totals, per-kernel timed step).
"""
from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from . import build as _build

_lock = threading.Lock()
_lib = None

SIM_OK, SIM_E_INVALID, SIM_E_CUDA, SIM_E_OOM, SIM_E_NCCL, SIM_E_NONFINITE, SIM_E_STATE = 0, -1, -2, -3, -4, -5, -6
ABI_VERSION = 1
INT32_MAX = 2**31 - 1
NUM_KERNELS = 7
KERNEL_NAMES = ("regrow", "policy", "move", "birth_claim", "birth_rank", "mutate", "hh")

EXPORTED = ("sim_create", "sim_step", "sim_get_state", "sim_set_state", "sim_destroy", "sim_last_error",
            "sim_validate", "sim_state_sizes", "sim_set_forced_actions", "sim_get_step_log", "sim_get_totals",
            "sim_step_timed", "sim_synchronize", "sim_kernels_per_step", "sim_get_phase_ns",
            "sim_shard", "sim_step_policy", "sim_step_post", "sim_exchange", "sim_get_step_log_async",
            "sim_set_record_mirror", "sim_step_graph_timed", "sim_get_move_hist",
            "sim_band_export", "sim_band_import", "sim_band_nccl_id", "sim_band_nccl_init", "sim_band_step_timed",
            "sim_get_greediness", "sim_get_life_windows", "sim_get_policy_actions")
GREED_WINDOW, LIFE_WINDOW = 20, 500  # include/sim.h: SIM_GREED_WINDOW, SIM_LIFE_WINDOW
BAND_PHASES = ("halo_x1", "policy", "merge_x2", "move", "arrive_x3", "live", "prep_p", "halo_x4a", "claims",
               "merge_x4b", "rank", "mutate", "regrow")  # include/sim.h: SIM_BAND_PHASES
POST_PHASES = ("move", "birth_claim", "birth_rank+regrow_next", "mutate",
               "reserved4", "reserved5", "reserved6", "reserved7",
               "claim.warp_sum_b0", "regrow.warp_sum_b1")  # summed over the warps of block 0 / block 1


class SimError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"libsim status {status}: {msg}")
        self.status = status


class SimConfig(ctypes.Structure):
    _fields_ = [
        ("abi_version", ctypes.c_uint32), ("struct_size", ctypes.c_uint32),
        ("rows", ctypes.c_int32), ("cols", ctypes.c_int32),
        ("n_worlds", ctypes.c_int32), ("device", ctypes.c_int32),
        ("seeds", ctypes.POINTER(ctypes.c_uint64)),
        ("init_resource_p", ctypes.c_double),
        ("regrow_r2", ctypes.c_int32),
        ("f_class_min_k", ctypes.c_int32 * 4),
        ("f_value", ctypes.c_double * 4),
        ("lat_top", ctypes.c_double), ("lat_bottom", ctypes.c_double),
        ("spontaneous", ctypes.c_double),
        ("slots", ctypes.c_int32), ("n_initial", ctypes.c_int32),
        ("obs_radius", ctypes.c_int32), ("hidden", ctypes.c_int32),
        ("n_actions", ctypes.c_int32), ("log_capacity", ctypes.c_int32),
        ("init_weight_std", ctypes.c_double), ("mutation_std", ctypes.c_double),
        ("e_init", ctypes.c_int32), ("e_decay", ctypes.c_int32), ("e_gain", ctypes.c_int32),
        ("e_repr_gt", ctypes.c_int32), ("e_death_le", ctypes.c_int32), ("e_max", ctypes.c_int32),
        ("repr_steps", ctypes.c_int32), ("max_age", ctypes.c_int32),
        ("cuda_stream", ctypes.c_void_p),
        # banded mode (include/sim.h: one world in latitude bands)
        ("n_bands", ctypes.c_int32), ("band_first", ctypes.c_int32), ("band_local", ctypes.c_int32),
        ("band_rows", ctypes.POINTER(ctypes.c_int32)), ("band_slots", ctypes.c_int32),
        # the paper's own world (include/sim.h)
        ("climate_alpha", ctypes.c_double), ("death_steps", ctypes.c_int32), ("lethal_walls", ctypes.c_int32),
        ("network", ctypes.c_int32), ("colocate", ctypes.c_int32),
    ]


class SimState(ctypes.Structure):
    _fields_ = [("t", ctypes.c_int64)] + [(f, ctypes.c_void_p) for f in (
        "resources", "alive", "cell", "energy", "age", "repr", "last_action", "ate", "h", "c", "weights",
        "logits", "low")]


RECORD_FIELDS = ("t", "agents_at_start", "grown", "eaten", "births", "deaths_energy", "deaths_age",
                 "deferred_no_cell", "deferred_claim", "deferred_capacity", "population", "resources",
                 "near_ties", "obs_nnz", "death_age_sum", "deaths_wall")
MOVE_WINDOW, MOVE_BINS = 50, 17  # include/sim.h: SIM_MOVE_WINDOW, SIM_MOVE_BINS
RECORD_DTYPE = np.dtype([(f, np.int64) for f in RECORD_FIELDS])
TOTALS_FIELDS = ("steps", "agent_steps", "cell_updates", "births", "deaths", "eaten", "grown")


class SimTotals(ctypes.Structure):
    _fields_ = [(f, ctypes.c_int64) for f in TOTALS_FIELDS]


class SimStateSizes(ctypes.Structure):
    _fields_ = [("cells", ctypes.c_int64), ("slots", ctypes.c_int64), ("hidden", ctypes.c_int32),
                ("inputs", ctypes.c_int32), ("params", ctypes.c_int32), ("n_actions", ctypes.c_int32),
                ("device_bytes", ctypes.c_int64)]


class SimStepTiming(ctypes.Structure):
    _fields_ = [("step_ms", ctypes.c_float), ("kernel_ms", ctypes.c_float * NUM_KERNELS)]


def lib():
    """Load (building first if stale) the in-tree libsim.so.  Raises if it cannot."""
    global _lib
    with _lock:
        if _lib is None:
            path = os.environ.get("ECO_LIBSIM_OVERRIDE") or _build.LIB  # diagnostics: alternative build
            if path == _build.LIB and (not os.path.exists(path) or _build._stale()):
                _build.build()
            L = ctypes.CDLL(path)
            H = ctypes.c_void_p
            L.sim_create.argtypes = [ctypes.POINTER(SimConfig), ctypes.POINTER(H)]
            L.sim_step.argtypes = [H, ctypes.c_int64]
            L.sim_get_state.argtypes = [H, ctypes.POINTER(SimState)]
            L.sim_set_state.argtypes = [H, ctypes.POINTER(SimState)]
            L.sim_destroy.argtypes = [H]
            L.sim_last_error.restype = ctypes.c_char_p
            L.sim_validate.argtypes = [ctypes.POINTER(SimConfig)]
            L.sim_state_sizes.argtypes = [ctypes.POINTER(SimConfig), ctypes.POINTER(SimStateSizes)]
            L.sim_set_forced_actions.argtypes = [H, ctypes.c_void_p]
            L.sim_get_policy_actions.argtypes = [H, ctypes.c_void_p]
            L.sim_get_step_log.argtypes = [H, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p]
            if hasattr(L, "sim_get_step_log_async"):
                L.sim_get_step_log_async.argtypes = [H, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p]
            if hasattr(L, "sim_set_record_mirror"):
                L.sim_set_record_mirror.argtypes = [H, ctypes.c_void_p, ctypes.c_int64]
            L.sim_get_totals.argtypes = [H, ctypes.POINTER(SimTotals)]
            L.sim_step_timed.argtypes = [H, ctypes.POINTER(SimStepTiming)]
            if hasattr(L, "sim_get_move_hist"):
                L.sim_get_move_hist.argtypes = [H, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p]
            if hasattr(L, "sim_step_graph_timed"):
                L.sim_step_graph_timed.argtypes = [H, ctypes.c_void_p]
            L.sim_synchronize.argtypes = [H]
            L.sim_kernels_per_step.restype = ctypes.c_int32
            L.sim_get_phase_ns.argtypes = [H, ctypes.c_void_p, ctypes.c_int32]
            if hasattr(L, "sim_shard"):  # (an ECO_LIBSIM_OVERRIDE build may predate the sharded mode)
                L.sim_shard.argtypes = [H, ctypes.c_int32, ctypes.c_int32]
                L.sim_step_policy.argtypes = [H]
                L.sim_step_post.argtypes = [H]
                L.sim_exchange.argtypes = [H, ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_size_t),
                                           ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_size_t)]
            if hasattr(L, "sim_band_export"):
                L.sim_band_export.argtypes = [H, ctypes.c_int32, ctypes.c_void_p, ctypes.POINTER(ctypes.c_size_t)]
                L.sim_band_import.argtypes = [H, ctypes.c_int32, ctypes.c_void_p, ctypes.c_size_t]
                L.sim_band_nccl_id.argtypes = [ctypes.c_void_p]
                L.sim_band_nccl_init.argtypes = [H, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32]
                L.sim_band_step_timed.argtypes = [H, ctypes.c_void_p, ctypes.c_int32]
            if hasattr(L, "sim_get_greediness"):
                L.sim_get_greediness.argtypes = [H, ctypes.c_void_p, ctypes.c_void_p]
                L.sim_get_life_windows.argtypes = [H, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
            for f in EXPORTED:
                if f not in ("sim_last_error", "sim_kernels_per_step") and hasattr(L, f):
                    getattr(L, f).restype = ctypes.c_int
            _lib = L
    return _lib


def _check(rc: int):
    if rc != SIM_OK:
        raise SimError(rc, lib().sim_last_error().decode())


def _stream_handle(stream) -> int:
    if stream is None:
        return 0
    if isinstance(stream, int):
        return stream
    return int(stream.cuda_stream)  # torch.cuda.Stream


def make_config(wc, device: int = 0, stream=None, log_capacity: int = 0, bands=None):
    """SimConfig from a workloads.WorldConfig (or any object with the same fields).
    `bands` (banded mode): dict(n_bands=G, band_first=0, band_local=G, band_rows=None,
    band_slots=0).  Returns (config, keep-alive arrays) — keep them while the config is used."""
    seeds = np.ascontiguousarray(np.array([int(s) & 0xFFFFFFFFFFFFFFFF for s in wc.seeds], dtype=np.uint64))
    c = SimConfig()
    c.abi_version, c.struct_size = ABI_VERSION, ctypes.sizeof(SimConfig)
    c.rows, c.cols, c.n_worlds, c.device = wc.rows, wc.cols, len(seeds), device
    c.seeds = seeds.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))
    c.init_resource_p, c.regrow_r2 = wc.init_resource_p, wc.regrow_r2
    for i in range(4):
        c.f_class_min_k[i] = int(wc.f_class_min_k[i])
        c.f_value[i] = float(wc.f_value[i])
    c.lat_top, c.lat_bottom, c.spontaneous = wc.lat_top, wc.lat_bottom, wc.spontaneous
    c.slots, c.n_initial = wc.slots, wc.n_initial
    c.obs_radius, c.hidden, c.n_actions = wc.obs_radius, wc.hidden, wc.n_actions
    c.log_capacity = log_capacity
    c.init_weight_std, c.mutation_std = wc.init_weight_std, wc.mutation_std
    c.e_init, c.e_decay, c.e_gain = wc.e_init, wc.e_decay, wc.e_gain
    c.e_repr_gt, c.e_death_le, c.e_max = wc.e_repr_gt, wc.e_death_le, wc.e_max
    c.repr_steps, c.max_age = wc.repr_steps, wc.max_age
    c.cuda_stream = _stream_handle(stream)
    c.climate_alpha = float(getattr(wc, "climate_alpha", 0.0))
    c.death_steps = int(getattr(wc, "death_steps", 0))
    c.lethal_walls = int(getattr(wc, "lethal_walls", 0))
    c.network = int(getattr(wc, "network", 0))
    c.colocate = int(getattr(wc, "colocate", 0))
    keep = [seeds]
    if bands:
        G = int(bands["n_bands"])
        c.n_bands = G
        c.band_first = int(bands.get("band_first", 0))
        c.band_local = int(bands.get("band_local", G - c.band_first))
        c.band_slots = int(bands.get("band_slots", 0))
        if bands.get("band_rows") is not None:
            rows = np.ascontiguousarray(np.asarray(bands["band_rows"], np.int32))
            c.band_rows = rows.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
            keep.append(rows)
    return c, keep


def validate(wc, bands=None) -> None:
    c, _seeds = make_config(wc, bands=bands)
    _check(lib().sim_validate(ctypes.byref(c)))


def state_sizes(wc) -> dict:
    c, _seeds = make_config(wc)
    s = SimStateSizes()
    _check(lib().sim_state_sizes(ctypes.byref(c), ctypes.byref(s)))
    return {f: int(getattr(s, f)) for f, _ in SimStateSizes._fields_}


STATE_FIELDS = ("resources", "alive", "cell", "energy", "age", "repr", "last_action", "ate", "h", "c",
                "weights", "logits", "low")


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


class World:
    """One handle of libsim.so: n_worlds independent worlds batched on one GPU."""

    def __init__(self, wc, device: int = 0, stream=None, log_capacity: int = 0, bands=None):
        """bands: banded mode (one world in latitude bands, include/sim.h), e.g.
        dict(n_bands=4) for four bands on this GPU (see paper_2302_09334_b200.banded)."""
        self.wc = wc
        self.device = device
        self.stream = stream
        self.n_worlds = len(wc.seeds)
        self.bands = dict(bands) if bands else None
        self._cfg, self._seeds = make_config(wc, device, stream, log_capacity, bands)
        self.log_capacity = log_capacity or 4096
        h = ctypes.c_void_p()
        _check(lib().sim_create(ctypes.byref(self._cfg), ctypes.byref(h)))
        self._h = h
        self._t = 0

    # -- lifecycle ------------------------------------------------------------------
    def destroy(self):
        if getattr(self, "_h", None):
            lib().sim_destroy(self._h)
            self._h = None

    close = destroy

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.destroy()

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    @property
    def t(self) -> int:
        return self._t

    def step(self, n: int = 1):
        _check(lib().sim_step(self._h, int(n)))
        self._t += int(n)

    # -- agent-sharded mode (include/sim.h: sim_shard) --------------------------------
    def shard(self, n_ranks: int, rank: int):
        """Own slots s with s % n_ranks == rank; step with step_policy / exchange / step_post."""
        _check(lib().sim_shard(self._h, int(n_ranks), int(rank)))

    def step_policy(self):
        _check(lib().sim_step_policy(self._h))

    def step_post(self):
        _check(lib().sim_step_post(self._h))
        self._t += 1

    def exchange_buffers(self):
        """(move-record pointer, bytes, record pointer, bytes): the device buffers to
        SUM-allreduce over the ranks between step_policy and step_post."""
        mp, mb, rp, rb = ctypes.c_void_p(), ctypes.c_size_t(), ctypes.c_void_p(), ctypes.c_size_t()
        _check(lib().sim_exchange(self._h, ctypes.byref(mp), ctypes.byref(mb), ctypes.byref(rp), ctypes.byref(rb)))
        return mp.value, mb.value, rp.value, rb.value

    def exchange_tensors(self):
        """The exchange buffers as torch CUDA tensors aliasing the library's memory (int32
        move records, int64 policy counters), for torch.distributed.all_reduce."""
        import torch
        mp, mb, rp, rb = self.exchange_buffers()
        dev = torch.device("cuda", self.device)

        class _View:  # __cuda_array_interface__ over a device pointer owned by the handle
            def __init__(self, ptr, n, typestr):
                self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False),
                                                 "version": 3, "strides": None}

        m = torch.as_tensor(_View(mp, mb // 4, "<i4"), device=dev)
        r = torch.as_tensor(_View(rp, rb // 8, "<i8"), device=dev)
        return m, r

    def step_timed(self) -> dict:
        tm = SimStepTiming()
        _check(lib().sim_step_timed(self._h, ctypes.byref(tm)))
        self._t += 1
        return {"step_ms": float(tm.step_ms), **{k: float(tm.kernel_ms[i]) for i, k in enumerate(KERNEL_NAMES)}}

    def band_step_timed(self) -> np.ndarray:
        """Banded handle: one step with events around every local band's phases (bands one
        after the other): float [band_local][len(BAND_PHASES)] milliseconds."""
        nl = int(self.bands.get("band_local", self.bands["n_bands"] - self.bands.get("band_first", 0)))
        out = np.zeros((nl, len(BAND_PHASES)), np.float32)
        _check(lib().sim_band_step_timed(self._h, _ptr(out), len(BAND_PHASES)))
        self._t += 1
        return out

    def step_graph_timed(self) -> dict:
        """One step through graph mode's two kernels, each bracketed by CUDA events (ms)."""
        out = (ctypes.c_float * 2)()
        _check(lib().sim_step_graph_timed(self._h, out))
        self._t += 1
        return {"policy": float(out[0]), "post": float(out[1])}

    def synchronize(self):
        _check(lib().sim_synchronize(self._h))

    # -- state ----------------------------------------------------------------------
    def state_shapes(self) -> dict:
        """field -> (shape, dtype) of the canonical state arrays (leading world axis)."""
        wc, nw = self.wc, self.n_worlds
        S, Hd, P = wc.slots, wc.hidden, wc.n_params
        return {
            "resources": ((nw, wc.rows, wc.cols), np.uint8), "alive": ((nw, S), np.uint8),
            "cell": ((nw, S), np.int32), "energy": ((nw, S), np.int32), "age": ((nw, S), np.int32),
            "repr": ((nw, S), np.int32), "last_action": ((nw, S), np.uint8), "ate": ((nw, S), np.uint8),
            "h": ((nw, S, Hd), np.float32), "c": ((nw, S, Hd), np.float32),
            "weights": ((nw, S, P), np.float32), "logits": ((nw, S, 5), np.float32),
            "low": ((nw, S), np.int32),
        }

    def empty_state(self, fields=STATE_FIELDS) -> dict:
        shapes = self.state_shapes()
        return {f: np.zeros(*shapes[f]) for f in fields}

    def get_state(self, fields=STATE_FIELDS) -> dict:
        """Canonical state (include/sim.h sim_state) as numpy arrays with a leading world axis."""
        out = self.empty_state(fields)
        st = SimState()
        for f in fields:
            setattr(st, f, _ptr(out[f]))
        _check(lib().sim_get_state(self._h, ctypes.byref(st)))
        out["t"] = int(st.t)
        self._t = int(st.t)
        return out

    def set_state(self, state: dict):
        """Inject canonical state (fields missing from `state` keep their device values).
        Per-field arrays may omit the world axis when n_worlds == 1."""
        st = SimState()
        keep = []
        shapes = self.state_shapes()  # (no host allocation: the weights alone are 0.5 GB at paper scale)
        for f in STATE_FIELDS:
            if f not in state:
                continue
            a = np.ascontiguousarray(np.asarray(state[f]).reshape(shapes[f][0]), dtype=shapes[f][1])
            keep.append(a)
            setattr(st, f, _ptr(a))
        st.t = int(state.get("t", self._t))
        _check(lib().sim_set_state(self._h, ctypes.byref(st)))
        self._t = int(st.t)

    def set_forced_actions(self, actions):
        """actions: [n_worlds][S] (or [S]) uint8, 255 = policy; None clears."""
        if actions is None:
            _check(lib().sim_set_forced_actions(self._h, None))
            return
        a = np.ascontiguousarray(np.asarray(actions, dtype=np.uint8).reshape(self.n_worlds, self.wc.slots))
        _check(lib().sim_set_forced_actions(self._h, _ptr(a)))

    def policy_actions(self) -> np.ndarray:
        """[n_worlds][S]: the policy's own action of each slot in the last forced step."""
        out = np.full((self.n_worlds, self.wc.slots), 255, np.uint8)
        _check(lib().sim_get_policy_actions(self._h, _ptr(out)))
        return out

    def step_log(self, first: int, n: int) -> np.ndarray:
        """Records of steps [first, first+n): structured array of shape [n, n_worlds]."""
        out = np.zeros((n, self.n_worlds), RECORD_DTYPE)
        _check(lib().sim_get_step_log(self._h, int(first), int(n), _ptr(out)))
        return out

    def step_log_async(self, first: int, n: int, out: np.ndarray):
        """Enqueue the copy of the records of steps [first, first+n) into `out` (a structured
        array of RECORD_DTYPE, shape [n, n_worlds], ideally in pinned memory) without waiting;
        `out` is valid after the next synchronize()."""
        assert out.dtype == RECORD_DTYPE and out.shape == (n, self.n_worlds) and out.flags.c_contiguous
        _check(lib().sim_get_step_log_async(self._h, int(first), int(n), _ptr(out)))

    def set_record_mirror(self, buf, capacity: int = 0):
        """Mirror each step's record into `buf` (RECORD_DTYPE [capacity][n_worlds], page-locked
        mapped host memory, e.g. a numpy view of a torch pin_memory tensor); None stops."""
        if buf is None:
            _check(lib().sim_set_record_mirror(self._h, None, 0))
            self._mirror = None
            return
        assert buf.dtype == RECORD_DTYPE and buf.shape == (capacity, self.n_worlds) and buf.flags.c_contiguous
        _check(lib().sim_set_record_mirror(self._h, _ptr(buf), int(capacity)))
        self._mirror = buf  # the device writes into it: keep it alive

    def phase_ns(self, reset: bool = False) -> dict:
        """Summed k_post phase durations (ns, block-0 view) since the last reset."""
        out = np.zeros(len(POST_PHASES), np.int64)
        _check(lib().sim_get_phase_ns(self._h, _ptr(out), int(reset)))
        return dict(zip(POST_PHASES, out.tolist()))

    def move_hist(self, first: int, n: int) -> np.ndarray:
        """Movement histograms of windows [first, first+n): int32 [n, n_worlds, 17]
        (include/sim.h: sim_get_move_hist)."""
        out = np.zeros((n, self.n_worlds, MOVE_BINS), np.int32)
        _check(lib().sim_get_move_hist(self._h, int(first), int(n), _ptr(out)))
        return out

    def greediness(self):
        """(T_r, C_r) int32 [n_worlds][S] (include/sim.h sim_get_greediness); G = C_r / T_r."""
        T = np.zeros((self.n_worlds, self.wc.slots), np.int32)
        C = np.zeros((self.n_worlds, self.wc.slots), np.int32)
        _check(lib().sim_get_greediness(self._h, _ptr(T), _ptr(C)))
        return T, C

    def life_windows(self, first: int, n: int):
        """(deaths, age_sum) int64 [n][n_worlds] of 500-step windows [first, first+n)."""
        d = np.zeros((n, self.n_worlds), np.int64)
        a = np.zeros((n, self.n_worlds), np.int64)
        _check(lib().sim_get_life_windows(self._h, int(first), int(n), _ptr(d), _ptr(a)))
        return d, a

    def totals(self) -> dict:
        tt = SimTotals()
        _check(lib().sim_get_totals(self._h, ctypes.byref(tt)))
        return {f: int(getattr(tt, f)) for f in TOTALS_FIELDS}


def world_view(state: dict, w: int) -> dict:
    """One world's slice of a batched state dict."""
    return {k: (v[w] if isinstance(v, np.ndarray) else v) for k, v in state.items()}
