"""Pins for the oracle's observation gather and policy (SURVEY.md §8c
C.3.2-C.3.3, R10-R13, R28).

Pinned by: np.pad + slicing for the observation; torch.nn.LSTMCell + nn.Linear in float64
for the LSTM and head; special cases S14 (corner agent) and S15 (all-zero weights);
exact ties resolving to the lowest index; non-finite detection.
"""
import numpy as np
import pytest
import torch

import oracle
import workloads


def np_window(plane, y, x, r):
    p = np.pad(plane, r)
    return p[y:y + 2 * r + 1, x:x + 2 * r + 1]


@pytest.mark.parametrize("r", [0, 1, 2, 3])
def test_observe_matches_pad_and_slice(r):
    rng = np.random.default_rng(r)
    wc = workloads.WorldConfig(rows=9, cols=12, obs_radius=r)
    R = (rng.random((9, 12)) < 0.5).astype(np.uint8)
    O = (rng.random((9, 12)) < 0.3).astype(np.uint8)
    for y in range(9):
        for x in range(12):
            got = oracle.observe(wc, R, O, y, x)
            want = np.concatenate([np_window(R, y, x, r).ravel(), np_window(O, y, x, r).ravel()])
            assert np.array_equal(got, want.astype(np.float64))


def test_observe_corner_agent_s14():
    # S14: an agent at (0,0) with r=3: zeros at rows/cols -3..-1, centre of channel 1 = 1 (self)
    wc = workloads.WorldConfig(rows=10, cols=12, obs_radius=3)
    R = np.ones((10, 12), np.uint8)
    O = np.zeros((10, 12), np.uint8)
    O[0, 0] = 1
    x = oracle.observe(wc, R, O, 0, 0).reshape(2, 7, 7)
    assert np.all(x[:, :3, :] == 0) and np.all(x[:, :, :3] == 0)
    assert np.all(x[0, 3:, 3:] == 1)
    assert x[1, 3, 3] == 1 and x[1].sum() == 1


def split(wc, w):
    I, Hd, A = wc.n_inputs, wc.hidden, wc.n_actions
    G = 4 * Hd
    o = 0
    W_ih = w[o:o + G * I].reshape(G, I); o += G * I
    W_hh = w[o:o + G * Hd].reshape(G, Hd); o += G * Hd
    b = w[o:o + G]; o += G
    W_out = w[o:o + A * Hd].reshape(A, Hd); o += A * Hd
    b_out = w[o:o + A]; o += A
    assert o == wc.n_params
    return W_ih, W_hh, b, W_out, b_out


def torch_reference(wc, w, x, h, c):
    W_ih, W_hh, b, W_out, b_out = split(wc, w.astype(np.float64))
    cell = torch.nn.LSTMCell(wc.n_inputs, wc.hidden, dtype=torch.float64)
    head = torch.nn.Linear(wc.hidden, wc.n_actions, dtype=torch.float64)
    with torch.no_grad():
        cell.weight_ih.copy_(torch.from_numpy(W_ih))
        cell.weight_hh.copy_(torch.from_numpy(W_hh))
        cell.bias_ih.copy_(torch.from_numpy(b))
        cell.bias_hh.zero_()
        head.weight.copy_(torch.from_numpy(W_out))
        head.bias.copy_(torch.from_numpy(b_out))
        hn, cn = cell(torch.from_numpy(x)[None], (torch.from_numpy(h.astype(np.float64))[None],
                                                  torch.from_numpy(c.astype(np.float64))[None]))
        h32 = hn[0].numpy().astype(np.float32)
        logits = head(torch.from_numpy(h32.astype(np.float64))[None])[0].numpy()
    return hn[0].numpy(), cn[0].numpy(), logits


@pytest.mark.parametrize("cfg", ["tiny", "paper"])
def test_policy_matches_torch_lstmcell(cfg):
    wc = workloads.tiny() if cfg == "tiny" else workloads.paper_scale()
    rng = np.random.default_rng(17)
    for trial in range(20):
        w = (rng.standard_normal(wc.n_params) * 0.3).astype(np.float32)
        x = (rng.random(wc.n_inputs) < 0.4).astype(np.float64)
        h = rng.uniform(-1, 1, wc.hidden).astype(np.float32)
        c = (rng.standard_normal(wc.hidden) * 2).astype(np.float32)
        ho, co, lg, a, margin, rc = oracle.policy(wc, w, x, h, c)
        assert rc == oracle.OK
        th, tc, tl = torch_reference(wc, w, x, h, c)
        # the oracle stores h', c' rounded to fp32 (R12); the head reads h'_fp32
        assert np.array_equal(ho, th.astype(np.float32))
        assert np.array_equal(co, tc.astype(np.float32))
        assert np.array_equal(lg, tl.astype(np.float32))
        assert a == int(np.argmax(tl.astype(np.float32)))
        s = np.sort(lg.astype(np.float64))
        assert margin == pytest.approx(s[-1] - s[-2], abs=0)


def test_policy_all_zero_weights_s15():
    wc = workloads.tiny()
    w = np.zeros(wc.n_params, np.float32)
    x = np.ones(wc.n_inputs)
    h = np.linspace(-1, 1, wc.hidden).astype(np.float32)
    c = np.linspace(-2, 2, wc.hidden).astype(np.float32)
    ho, co, lg, a, margin, rc = oracle.policy(wc, w, x, h, c)
    # z = 0: every gate 0.5, g = 0 -> c' = 0.5 c, h' = 0.5 tanh(c'); logits 0 -> action 0
    assert np.array_equal(co, (0.5 * c.astype(np.float64)).astype(np.float32))
    assert np.array_equal(ho, (0.5 * np.tanh(0.5 * c.astype(np.float64))).astype(np.float32))
    assert np.all(lg == 0) and a == 0 and margin == 0.0


def test_policy_exact_tie_lowest_index():
    wc = workloads.tiny()
    w = np.zeros(wc.n_params, np.float32)
    b_out = w[-5:]
    b_out[:] = [0.1, 0.3, 0.2, 0.3, -1.0]
    _, _, lg, a, margin, _ = oracle.policy(wc, w, np.zeros(wc.n_inputs), np.zeros(8, np.float32),
                                           np.zeros(8, np.float32))
    assert a == 1 and margin == 0.0


def test_policy_nonfinite_flag():
    wc = workloads.tiny()
    w = np.zeros(wc.n_params, np.float32)
    w[0] = np.nan
    x = np.zeros(wc.n_inputs)
    x[0] = 1.0
    *_, rc = oracle.policy(wc, w, x, np.zeros(8, np.float32), np.zeros(8, np.float32))
    assert rc == oracle.E_NONFINITE


def test_param_counts():
    # 1,933 (tiny) and 16,933 (Hd=32, I=98)
    assert oracle.param_count(workloads.tiny()) == 1933 == workloads.tiny().n_params
    assert oracle.param_count(workloads.paper_scale()) == 16933 == workloads.paper_scale().n_params
