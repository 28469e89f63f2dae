"""CPU oracle for the world step — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / ``--impl reference``
legs may import this package.  The product path (paper_2302_09334_b200/) never imports
it and shares no code with it.

A ctypes wrapper over oracle/liboracle.so (plain C99, oracle/oracle.c), which follows
PAPER.md App. B (lines 248-350) under the BASELINE.json configs and the readings in
DESIGN.md §3.  Parity pins live in tests/test_oracle_*.py.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

OK, E_INVALID, E_NONFINITE = 0, -1, -5
P_INIT_RES, P_INIT_PLACE, P_INIT_W, P_REGROW, P_MOVE, P_BIRTH, P_MUTATE, P_ACTION, P_CONSUME = range(1, 10)


def build(force: bool = False) -> str:
    """Compile oracle.c into liboracle.so (gcc -O2 -ffp-contract=off)."""
    src = os.path.join(_HERE, "oracle.c")
    hdr = os.path.join(_HERE, "oracle.h")
    if (not force and os.path.exists(_LIB_PATH)
            and os.path.getmtime(_LIB_PATH) >= max(os.path.getmtime(src), os.path.getmtime(hdr))):
        return _LIB_PATH
    tmp = _LIB_PATH + f".tmp{os.getpid()}"
    subprocess.check_call(["gcc", "-O2", "-std=c99", "-Wall", "-ffp-contract=off", "-fPIC", "-shared",
                           src, "-o", tmp, "-lm"])
    os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


class Config(ctypes.Structure):
    _fields_ = [
        ("rows", ctypes.c_int32), ("cols", ctypes.c_int32),
        ("seed", ctypes.c_uint64),
        ("init_resource_p", ctypes.c_double),
        ("regrow_r2", ctypes.c_int32),
        ("f_class_min_k", ctypes.c_int32 * 4),
        ("f_value", ctypes.c_double * 4),
        ("lat_top", ctypes.c_double), ("lat_bottom", ctypes.c_double),
        ("spontaneous", ctypes.c_double),
        ("slots", ctypes.c_int32), ("n_initial", ctypes.c_int32),
        ("obs_radius", ctypes.c_int32), ("hidden", ctypes.c_int32), ("n_actions", ctypes.c_int32),
        ("init_weight_std", ctypes.c_double), ("mutation_std", ctypes.c_double),
        ("e_init", ctypes.c_int32), ("e_decay", ctypes.c_int32), ("e_gain", ctypes.c_int32),
        ("e_repr_gt", ctypes.c_int32), ("e_death_le", ctypes.c_int32), ("e_max", ctypes.c_int32),
        ("repr_steps", ctypes.c_int32), ("max_age", ctypes.c_int32),
        ("climate_alpha", ctypes.c_double), ("death_steps", ctypes.c_int32), ("lethal_walls", ctypes.c_int32),
        ("network", ctypes.c_int32), ("colocate", ctypes.c_int32),
    ]


class State(ctypes.Structure):
    _fields_ = [
        ("t", ctypes.c_int64),
        ("resources", ctypes.c_void_p), ("alive", ctypes.c_void_p), ("cell", ctypes.c_void_p),
        ("energy", ctypes.c_void_p), ("age", ctypes.c_void_p), ("repr", ctypes.c_void_p),
        ("last_action", ctypes.c_void_p), ("ate", ctypes.c_void_p),
        ("h", ctypes.c_void_p), ("c", ctypes.c_void_p), ("weights", ctypes.c_void_p),
        ("logits", ctypes.c_void_p), ("low", ctypes.c_void_p),
    ]


RECORD_FIELDS = ("t", "grown", "eaten", "births", "deaths_energy", "deaths_age", "deferred_no_cell",
                 "deferred_claim", "deferred_capacity", "population", "resources", "near_ties", "deaths_wall")


class Record(ctypes.Structure):
    _fields_ = [(f, ctypes.c_int64) for f in RECORD_FIELDS]

    def as_dict(self) -> dict:
        return {f: int(getattr(self, f)) for f in RECORD_FIELDS}


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB_PATH)
            u32p = ctypes.POINTER(ctypes.c_uint32)
            L.orc_philox4x32_10.argtypes = [u32p, u32p, u32p]
            L.orc_draw4.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
                                    ctypes.c_uint32, u32p]
            L.orc_cell_draw.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32]
            L.orc_cell_draw.restype = ctypes.c_uint32
            L.orc_box_muller.argtypes = [ctypes.c_uint32, ctypes.c_uint32, ctypes.POINTER(ctypes.c_double),
                                         ctypes.POINTER(ctypes.c_double)]
            L.orc_gauss.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
                                    ctypes.c_int32, ctypes.c_void_p]
            cp = ctypes.POINTER(Config)
            L.orc_param_count.argtypes = [cp]
            L.orc_param_count.restype = ctypes.c_int32
            L.orc_input_count.argtypes = [cp]
            L.orc_input_count.restype = ctypes.c_int32
            L.orc_validate.argtypes = [cp, ctypes.c_char_p, ctypes.c_int]
            L.orc_thresholds.argtypes = [cp, ctypes.c_void_p]
            L.orc_neighbour_count.argtypes = [cp, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32]
            L.orc_neighbour_count.restype = ctypes.c_int32
            L.orc_class_of.argtypes = [cp, ctypes.c_int32]
            L.orc_class_of.restype = ctypes.c_int32
            L.orc_regrow.argtypes = [cp, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
            L.orc_regrow.restype = ctypes.c_int64
            L.orc_observe.argtypes = [cp, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32,
                                      ctypes.c_void_p]
            L.orc_policy.argtypes = [cp, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                     ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                     ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_double)]
            L.orc_observe_paper.argtypes = [cp, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32,
                                            ctypes.c_void_p]
            L.orc_conv3x3_s2_same.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                              ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p]
            L.orc_avgpool2_s1.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                          ctypes.c_void_p]
            L.orc_policy_cnn.argtypes = [cp, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32,
                                         ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                         ctypes.c_void_p, ctypes.c_void_p]
            L.orc_sample_action.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_void_p,
                                            ctypes.c_void_p, ctypes.POINTER(ctypes.c_double)]
            L.orc_sample_action.restype = ctypes.c_int32
            L.orc_init.argtypes = [cp, ctypes.POINTER(State)]
            L.orc_step.argtypes = [cp, ctypes.POINTER(State), ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(Record)]
            _lib = L
    return _lib


def _ptr(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.c_void_p)


def make_config(wc, world: int = 0) -> Config:
    """orc_config from a workloads.WorldConfig (world = index into its seeds)."""
    c = Config()
    c.rows, c.cols = wc.rows, wc.cols
    c.seed = int(wc.seeds[world]) & 0xFFFFFFFFFFFFFFFF
    c.init_resource_p = wc.init_resource_p
    c.regrow_r2 = wc.regrow_r2
    for i in range(4):
        c.f_class_min_k[i] = int(wc.f_class_min_k[i])
        c.f_value[i] = float(wc.f_value[i])
    c.lat_top, c.lat_bottom, c.spontaneous = wc.lat_top, wc.lat_bottom, wc.spontaneous
    c.slots, c.n_initial = wc.slots, wc.n_initial
    c.obs_radius, c.hidden, c.n_actions = wc.obs_radius, wc.hidden, wc.n_actions
    c.init_weight_std, c.mutation_std = wc.init_weight_std, wc.mutation_std
    c.e_init, c.e_decay, c.e_gain = wc.e_init, wc.e_decay, wc.e_gain
    c.e_repr_gt, c.e_death_le, c.e_max = wc.e_repr_gt, wc.e_death_le, wc.e_max
    c.repr_steps, c.max_age = wc.repr_steps, wc.max_age
    c.climate_alpha = float(getattr(wc, "climate_alpha", 0.0))
    c.death_steps = int(getattr(wc, "death_steps", 0))
    c.lethal_walls = int(getattr(wc, "lethal_walls", 0))
    c.network = int(getattr(wc, "network", 0))
    c.colocate = int(getattr(wc, "colocate", 0))
    return c


# ------------------------------------------------------------------ primitives
def philox(ctr, key):
    L = lib()
    c = (ctypes.c_uint32 * 4)(*[int(v) & 0xFFFFFFFF for v in ctr])
    k = (ctypes.c_uint32 * 2)(*[int(v) & 0xFFFFFFFF for v in key])
    o = (ctypes.c_uint32 * 4)()
    L.orc_philox4x32_10(c, k, o)
    return tuple(int(v) for v in o)


def draw4(seed, purpose, step, entity, sub=0):
    o = (ctypes.c_uint32 * 4)()
    lib().orc_draw4(seed, purpose, step, entity, sub, o)
    return tuple(int(v) for v in o)


def cell_draw(seed, purpose, step, cell):
    return int(lib().orc_cell_draw(seed, purpose, step, cell))


def box_muller(wa, wb):
    za, zb = ctypes.c_double(), ctypes.c_double()
    lib().orc_box_muller(wa, wb, ctypes.byref(za), ctypes.byref(zb))
    return za.value, zb.value


def gauss(seed, purpose, step, entity, n):
    z = np.zeros(n, np.float64)
    lib().orc_gauss(seed, purpose, step, entity, n, _ptr(z))
    return z


def param_count(wc) -> int:
    return int(lib().orc_param_count(ctypes.byref(make_config(wc))))


def validate(wc, world: int = 0):
    msg = ctypes.create_string_buffer(128)
    rc = lib().orc_validate(ctypes.byref(make_config(wc, world)), msg, 128)
    return rc, msg.value.decode()


def thresholds(wc) -> np.ndarray:
    T = np.zeros((wc.rows, 4), np.uint32)
    lib().orc_thresholds(ctypes.byref(make_config(wc)), _ptr(T))
    return T


def neighbour_count(wc, R: np.ndarray, y: int, x: int) -> int:
    R = np.ascontiguousarray(R, np.uint8)
    return int(lib().orc_neighbour_count(ctypes.byref(make_config(wc)), _ptr(R), y, x))


def class_of(wc, k: int) -> int:
    return int(lib().orc_class_of(ctypes.byref(make_config(wc)), k))


def regrow(wc, t: int, R: np.ndarray, world: int = 0):
    R = np.ascontiguousarray(R, np.uint8)
    Rn = np.zeros_like(R)
    grown = lib().orc_regrow(ctypes.byref(make_config(wc, world)), t, _ptr(R), _ptr(Rn))
    return Rn, int(grown)


def observe(wc, R: np.ndarray, O: np.ndarray, y: int, x: int) -> np.ndarray:
    R = np.ascontiguousarray(R, np.uint8)
    O = np.ascontiguousarray(O, np.uint8)
    out = np.zeros(wc.n_inputs, np.float64)
    lib().orc_observe(ctypes.byref(make_config(wc)), _ptr(R), _ptr(O), y, x, _ptr(out))
    return out


def policy(wc, w: np.ndarray, x: np.ndarray, h: np.ndarray, c: np.ndarray):
    """One agent's LSTM + head + argmax; returns (h', c', logits, action, margin, status)."""
    w = np.ascontiguousarray(w, np.float32)
    x = np.ascontiguousarray(x, np.float64)
    h = np.ascontiguousarray(h, np.float32)
    c = np.ascontiguousarray(c, np.float32)
    ho = np.zeros(wc.hidden, np.float32)
    co = np.zeros(wc.hidden, np.float32)
    lg = np.zeros(8, np.float32)
    a = ctypes.c_int32()
    m = ctypes.c_double()
    rc = lib().orc_policy(ctypes.byref(make_config(wc)), _ptr(w), _ptr(x), _ptr(h), _ptr(c), _ptr(ho),
                          _ptr(co), _ptr(lg), ctypes.byref(a), ctypes.byref(m))
    return ho, co, lg[:wc.n_actions].copy(), int(a.value), float(m.value), int(rc)


# ------------------------------------------- network 1: the paper's CNN-LSTM (NEXT-2)
def observe_paper(wc, R: np.ndarray, O: np.ndarray, y: int, x: int) -> np.ndarray:
    """The 15x15x3 window (HWC: resources, agents, walls) around (y, x); O: agents per cell."""
    R = np.ascontiguousarray(R, np.uint8)
    O = np.ascontiguousarray(O, np.int32)
    out = np.zeros((15, 15, 3), np.float64)
    lib().orc_observe_paper(ctypes.byref(make_config(wc)), _ptr(R), _ptr(O), y, x, _ptr(out))
    return out


def conv3x3_s2_same(x: np.ndarray, w: np.ndarray, b: np.ndarray) -> np.ndarray:
    """x [H][W][cin] fp64, w [cout][3][3][cin] fp32, b [cout] fp32 -> [ceil(H/2)][ceil(W/2)][cout]."""
    x = np.ascontiguousarray(x, np.float64)
    w = np.ascontiguousarray(w, np.float32)
    b = np.ascontiguousarray(b, np.float32)
    H, W, cin = x.shape
    cout = w.shape[0]
    out = np.zeros(((H + 1) // 2, (W + 1) // 2, cout), np.float64)
    lib().orc_conv3x3_s2_same(_ptr(x), H, W, cin, _ptr(w), _ptr(b), cout, _ptr(out))
    return out


def avgpool2_s1(x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float64)
    H, W, C = x.shape
    out = np.zeros((H - 1, W - 1, C), np.float64)
    lib().orc_avgpool2_s1(_ptr(x), H, W, C, _ptr(out))
    return out


def policy_cnn(wc, w: np.ndarray, obs: np.ndarray, last_action: int, ate: int, h: np.ndarray, c: np.ndarray):
    """One agent's CNN-LSTM forward; returns (h', c', logits, embedding[78], status)."""
    w = np.ascontiguousarray(w, np.float32)
    obs = np.ascontiguousarray(obs, np.float64)
    h = np.ascontiguousarray(h, np.float32)
    c = np.ascontiguousarray(c, np.float32)
    ho, co = np.zeros(4, np.float32), np.zeros(4, np.float32)
    lg = np.zeros(5, np.float32)
    emb = np.zeros(78, np.float64)
    rc = lib().orc_policy_cnn(ctypes.byref(make_config(wc)), _ptr(w), _ptr(obs), last_action, ate, _ptr(h), _ptr(c),
                              _ptr(ho), _ptr(co), _ptr(lg), _ptr(emb))
    return ho, co, lg, emb, int(rc)


def sample_action(seed: int, step: int, cell: int, logits: np.ndarray):
    """softmax(50 logits) sampled with the (ACTION, step, cell) draw: (action, probs, margin)."""
    lg = np.ascontiguousarray(logits, np.float32)
    probs = np.zeros(5, np.float64)
    m = ctypes.c_double()
    a = lib().orc_sample_action(int(seed) & 0xFFFFFFFFFFFFFFFF, step, cell, _ptr(lg), _ptr(probs), ctypes.byref(m))
    return int(a), probs, float(m.value)


# ------------------------------------------------------------------ world
class OracleWorld:
    """One world of the oracle; state arrays are numpy (canonical layout)."""

    def __init__(self, wc, world: int = 0, state: dict | None = None):
        import workloads  # the shared input module (no method arithmetic)
        self.wc = wc
        self.world = world
        self.cfg = make_config(wc, world)
        self.st = workloads.empty_state(wc)
        self._cst = State()
        if state is None:
            rc = lib().orc_init(ctypes.byref(self.cfg), self._bind())
            if rc != OK:
                raise ValueError(f"orc_init failed: {rc} {validate(wc, world)[1]}")
        else:
            self.set_state(state)

    def _bind(self):
        s = self._cst
        s.t = int(self.st["t"])
        for f in ("resources", "alive", "cell", "energy", "age", "repr", "last_action", "ate", "h", "c",
                  "weights", "logits", "low"):
            setattr(s, f, _ptr(self.st[f]))
        return ctypes.byref(s)

    def set_state(self, state: dict):
        for k, v in state.items():
            if k == "t":
                self.st["t"] = int(v)
            elif k in self.st:
                self.st[k][...] = v

    @property
    def t(self) -> int:
        return int(self.st["t"])

    def step(self, forced: np.ndarray | None = None, return_actions: bool = False) -> dict:
        """One oracle step.  With return_actions, d["actions"] holds the action every slot
        alive at step start used (255 elsewhere)."""
        rec = Record()
        ref = self._bind()
        fp = None
        if forced is not None:
            forced = np.ascontiguousarray(forced, np.uint8)
            fp = _ptr(forced)
        acts = np.full(self.wc.slots, 255, np.uint8) if return_actions else None
        rc = lib().orc_step(ctypes.byref(self.cfg), ref, fp, _ptr(acts) if return_actions else None,
                            ctypes.byref(rec))
        self.st["t"] = int(self._cst.t)
        d = rec.as_dict()
        d["status"] = int(rc)
        if return_actions:
            d["actions"] = acts
        return d

    def state(self) -> dict:
        return {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in self.st.items()}
