"""Pins for the oracle's RNG contract: Philox4x32-10, counter layout,
per-cell word selection and fp64 Box-Muller.

Pinned against things other than the oracle itself:
* cuRAND's own Philox block function (curand_philox4x32_x.h compiled for the host) on
  random counters/keys, and the Random123 known-answer vectors;
* the cuRAND host generator (libcurand, CURAND_RNG_PSEUDO_PHILOX4_32_10): output block i
  equals philox((0,0,i,0), seed);
* closed forms of Box-Muller at its end points, and normal moments / KS;
* the worked values of SURVEY.md §8c C.7 (tests/golden/contract_c7.json).
"""
import ctypes
import json
import math
import os
import shutil
import subprocess

import numpy as np
import pytest

import oracle

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "contract_c7.json")))
CUDA_INC = "/usr/local/cuda/include"
CURAND_LIB = "/usr/local/cuda/lib64/libcurand.so"


@pytest.fixture(scope="module")
def curand_pin(tmp_path_factory):
    if not (shutil.which("g++") and os.path.exists(os.path.join(CUDA_INC, "curand_philox4x32_x.h"))):
        pytest.skip("g++ or cuRAND headers unavailable")
    out = str(tmp_path_factory.mktemp("pin") / "libpin.so")
    subprocess.check_call(["g++", "-x", "c++", "-O1", "-shared", "-fPIC", f"-I{CUDA_INC}",
                           os.path.join(HERE, "pins", "curand_philox_pin.c"), "-o", out])
    L = ctypes.CDLL(out)
    u = ctypes.POINTER(ctypes.c_uint32)
    L.pin_philox.argtypes = [u, u, u]

    def f(ctr, key):
        c = (ctypes.c_uint32 * 4)(*ctr)
        k = (ctypes.c_uint32 * 2)(*key)
        o = (ctypes.c_uint32 * 4)()
        L.pin_philox(c, k, o)
        return tuple(int(v) for v in o)
    return f


def test_philox_known_answer_vectors():
    for case in GOLD["random123_kat_philox4x32_10"]["cases"]:
        ctr = [int(v, 16) for v in case["ctr"]]
        key = [int(v, 16) for v in case["key"]]
        assert oracle.philox(ctr, key) == tuple(int(v, 16) for v in case["out"])


def test_philox_matches_curand_block_function(curand_pin):
    rng = np.random.default_rng(1234)
    for _ in range(2000):
        ctr = [int(v) for v in rng.integers(0, 2**32, 4, dtype=np.uint64)]
        key = [int(v) for v in rng.integers(0, 2**32, 2, dtype=np.uint64)]
        assert oracle.philox(ctr, key) == curand_pin(ctr, key)
    # each counter word separately (catches swapped counter words / multipliers)
    for pos in range(4):
        for v in (1, 0x80000000, 0xFFFFFFFF):
            ctr = [0, 0, 0, 0]
            ctr[pos] = v
            assert oracle.philox(ctr, [7, 9]) == curand_pin(ctr, [7, 9])


@pytest.mark.parametrize("seed", [0, 1, 0x123456789ABCDEF0])
def test_philox_matches_curand_host_generator(seed):
    if not os.path.exists(CURAND_LIB):
        pytest.skip("libcurand unavailable")
    L = ctypes.CDLL(CURAND_LIB)
    g = ctypes.c_void_p()
    assert L.curandCreateGeneratorHost(ctypes.byref(g), 161) == 0  # PHILOX4_32_10
    try:
        assert L.curandSetPseudoRandomGeneratorSeed(g, ctypes.c_ulonglong(seed)) == 0
        n = 4 * 256
        out = np.zeros(n, np.uint32)
        assert L.curandGenerate(g, out.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(n)) == 0
    finally:
        L.curandDestroyGenerator(g)
    key = (seed & 0xFFFFFFFF, seed >> 32)
    for i in range(256):
        assert oracle.philox((0, 0, i, 0), key) == tuple(int(v) for v in out[4 * i:4 * i + 4]), i


def test_counter_layout_goldens():
    g = GOLD
    assert [oracle.cell_draw(0, oracle.P_REGROW, 0, c) for c in range(8)] == g["regrow_draws_seed0_t0_cells0_7"]
    w = oracle.draw4(1, oracle.P_MOVE, 5, 123, 0)
    assert w == tuple(int(v, 16) for v in g["philox_0_123_5_MOVE_seed1"])
    b = oracle.draw4(1, oracle.P_BIRTH, 5, 123, 0)
    assert b[0] & 3 == g["birth_t5_cell123_seed1"]["first_dir"]
    assert b[1] == g["birth_t5_cell123_seed1"]["priority"]


def test_cell_draw_word_selection():
    # one Philox call serves 4 horizontally adjacent cells: word cell&3 of entity cell>>2
    for cell in (0, 1, 2, 3, 4, 77, 12345, 2**31 - 1):
        words = oracle.draw4(42, oracle.P_REGROW, 9, cell >> 2, 0)
        assert oracle.cell_draw(42, oracle.P_REGROW, 9, cell) == words[cell & 3]
    # purposes and steps give distinct streams
    assert oracle.draw4(5, 1, 0, 10) != oracle.draw4(5, 2, 0, 10)
    assert oracle.draw4(5, 4, 0, 10) != oracle.draw4(5, 4, 1, 10)


def test_box_muller_closed_forms():
    # wa = 2^32-1 -> u1 = 1 -> radius 0
    assert oracle.box_muller(0xFFFFFFFF, 12345) == (0.0, 0.0)
    # wa = 0 -> u1 = 2^-32 -> r = sqrt(64 ln 2); wb = 0 -> theta = 0 -> (r, 0)
    r = math.sqrt(64.0 * math.log(2.0))
    za, zb = oracle.box_muller(0, 0)
    assert za == pytest.approx(r, rel=1e-15) and zb == 0.0
    # wb = 2^30 -> theta = pi/2 -> (~0, r)
    za, zb = oracle.box_muller(0, 2**30)
    assert abs(za) < 1e-14 and zb == pytest.approx(r, rel=1e-15)
    # wb = 2^31 -> theta = pi -> (-r, ~0)
    za, zb = oracle.box_muller(0, 2**31)
    assert za == pytest.approx(-r, rel=1e-15) and abs(zb) < 1e-14


def test_gauss_pairing_golden():
    z = oracle.gauss(0, oracle.P_INIT_W, 0, GOLD["tiny_seed0"]["initial_cells"][0], 4)
    assert list(z) == pytest.approx(GOLD["tiny_seed0"]["slot0_z0_3"], rel=1e-15, abs=0)


def test_gauss_moments_and_ks():
    from scipy import stats
    z = np.concatenate([oracle.gauss(7, oracle.P_MUTATE, t, 1000 + t, 50000) for t in range(20)])
    n = z.size
    assert abs(z.mean()) < 4 / math.sqrt(n)
    assert abs(z.var() - 1.0) < 4 * math.sqrt(2.0 / n)
    assert stats.kstest(z, "norm").pvalue > 1e-3
