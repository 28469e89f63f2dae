"""Pins of the oracle's network 1, the paper's CNN-LSTM with softmax sampling
(App. B.5; R38-R42).

What fixes it from outside the oracle:
  * the paper's parameter count, 2445, and SPEC's per-layer audit
    112 + 296 + 1328 + 664 + 45;
  * the convolution, pooling, LSTM cell and dense layers against torch's CPU library
    routines (F.conv2d with TF-style SAME padding, F.avg_pool2d, nn.LSTMCell, F.linear) in
    fp64 on random inputs: the whole forward composed from those routines must equal the
    oracle's (a transposed kernel, a wrong padding side, a dropped bias or a swapped gate
    fails here);
  * zero weights give a uniform softmax; a one-hot logit of 1 gives action 0
    with probability 1 - 4/(e^50 + 4); uniform logits sample each action
    with frequency 0.2 +- 0.01 over 10^5 draws; the inverse CDF against
    numpy's searchsorted on the same Philox words;
  * the observation's channels on hand-built worlds (walls off the grid, self in the
    agent channel, HWC order).
"""
import math

import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle
import workloads

WC = workloads.paper_world_cnn()


def split_params(w):
    """Canonical order of network 1 (oracle.h / sim.h): shapes by the paper's architecture."""
    shapes = [("c1w", (4, 3, 3, 3)), ("c1b", (4,)), ("c2w", (8, 3, 3, 4)), ("c2b", (8,)),
              ("W_ih", (16, 78)), ("W_hh", (16, 4)), ("b", (16,)), ("W_d", (8, 82)), ("b_d", (8,)),
              ("W_o", (5, 8)), ("b_o", (5,))]
    out, k = {}, 0
    for name, shp in shapes:
        n = int(np.prod(shp))
        out[name] = w[k:k + n].reshape(shp)
        k += n
    assert k == w.size
    return out


def test_param_count_is_the_papers():
    # "In total the agent neural network is very small with only 2445 parameters"
    assert oracle.param_count(WC) == 2445 == WC.n_params
    # conv1 112, conv2 296, LSTM 1328, dense 664, out 45
    assert 3 * 3 * 3 * 4 + 4 == 112 and 3 * 3 * 4 * 8 + 8 == 296
    assert 16 * (78 + 4) + 16 == 1328 and 82 * 8 + 8 == 664 and 8 * 5 + 5 == 45
    assert oracle.validate(WC)[0] == 0
    assert oracle.validate(WC.replace(obs_radius=3))[0] != 0  # the architecture fixes w_o = 15
    assert oracle.validate(WC.replace(hidden=8))[0] != 0      # and the LSTM size 4


def same_pad(n, k=3, s=2):
    out = -(-n // s)
    tot = max((out - 1) * s + k - n, 0)
    return tot // 2, tot - tot // 2


def torch_conv_same_s2(x, w, b):
    """x [H][W][C], w [cout][3][3][cin] -> TF/JAX 'SAME' stride-2 convolution via F.conv2d."""
    xt = torch.from_numpy(np.ascontiguousarray(x.transpose(2, 0, 1)))[None].double()
    py, px = same_pad(x.shape[0]), same_pad(x.shape[1])
    xt = F.pad(xt, (px[0], px[1], py[0], py[1]))
    wt = torch.from_numpy(np.ascontiguousarray(w.transpose(0, 3, 1, 2))).double()
    y = F.conv2d(xt, wt, torch.from_numpy(b).double(), stride=2)
    return y[0].numpy().transpose(1, 2, 0)


def torch_pool(x):
    xt = torch.from_numpy(np.ascontiguousarray(x.transpose(2, 0, 1)))[None].double()
    return F.avg_pool2d(xt, 2, stride=1)[0].numpy().transpose(1, 2, 0)


@pytest.mark.parametrize("H,W,cin,cout", [(15, 15, 3, 4), (7, 7, 4, 8), (8, 8, 2, 3), (6, 9, 1, 2)])
def test_conv_same_stride2_against_torch(H, W, cin, cout):
    rng = np.random.default_rng(H * 100 + W)
    x = rng.standard_normal((H, W, cin))
    w = rng.standard_normal((cout, 3, 3, cin)).astype(np.float32)
    b = rng.standard_normal(cout).astype(np.float32)
    got = oracle.conv3x3_s2_same(x, w, b)
    exp = torch_conv_same_s2(x, w.astype(np.float64), b.astype(np.float64))
    assert got.shape == exp.shape == ((H + 1) // 2, (W + 1) // 2, cout)
    np.testing.assert_allclose(got, exp, rtol=1e-12, atol=1e-12)


def test_shapes_of_the_pipeline():
    # 15x15x3 -> 8x8x4 -> 7x7x4 -> 4x4x8 -> 3x3x8 = 72
    x = np.zeros((15, 15, 3))
    a1 = oracle.conv3x3_s2_same(x, np.zeros((4, 3, 3, 3), np.float32), np.zeros(4, np.float32))
    p1 = oracle.avgpool2_s1(a1)
    a2 = oracle.conv3x3_s2_same(p1, np.zeros((8, 3, 3, 4), np.float32), np.zeros(8, np.float32))
    p2 = oracle.avgpool2_s1(a2)
    assert (a1.shape, p1.shape, a2.shape, p2.shape) == ((8, 8, 4), (7, 7, 4), (4, 4, 8), (3, 3, 8))


def test_avgpool_against_torch():
    x = np.random.default_rng(3).standard_normal((8, 8, 4))
    np.testing.assert_allclose(oracle.avgpool2_s1(x), torch_pool(x), rtol=1e-14, atol=1e-14)


def torch_forward(w, obs, last_action, ate, h, c):
    """The whole network composed from torch library routines in fp64."""
    p = {k: v.astype(np.float64) for k, v in split_params(w).items()}
    a1 = torch_conv_same_s2(obs, p["c1w"], p["c1b"])
    a2 = torch_conv_same_s2(torch_pool(a1), p["c2w"], p["c2b"])
    feat = torch_pool(a2).reshape(-1)  # HWC flatten, 72
    e = np.concatenate([feat, np.eye(5)[last_action], [float(ate)]])
    cell = torch.nn.LSTMCell(78, 4).double()
    with torch.no_grad():
        cell.weight_ih.copy_(torch.from_numpy(p["W_ih"]))
        cell.weight_hh.copy_(torch.from_numpy(p["W_hh"]))
        cell.bias_ih.copy_(torch.from_numpy(p["b"]))
        cell.bias_hh.zero_()
        hn, cn = cell(torch.from_numpy(e)[None], (torch.from_numpy(h.astype(np.float64))[None],
                                                  torch.from_numpy(c.astype(np.float64))[None]))
    hn32 = hn[0].numpy().astype(np.float32)
    z = np.concatenate([e, hn32.astype(np.float64)])
    d = torch.tanh(F.linear(torch.from_numpy(z), torch.from_numpy(p["W_d"]), torch.from_numpy(p["b_d"])))
    lg = F.linear(d, torch.from_numpy(p["W_o"]), torch.from_numpy(p["b_o"])).numpy()
    return hn[0].numpy(), cn[0].numpy(), lg, e


@pytest.mark.parametrize("seed", range(6))
def test_forward_against_torch_composition(seed):
    rng = np.random.default_rng(seed)
    w = (rng.standard_normal(2445) * (0.1 if seed < 3 else 0.5)).astype(np.float32)
    obs = (rng.random((15, 15, 3)) < 0.3).astype(np.float64)
    if seed % 2:
        obs = rng.standard_normal((15, 15, 3))  # the network is defined on any input
    la, ate = int(rng.integers(0, 5)), int(rng.integers(0, 2))
    h = rng.standard_normal(4).astype(np.float32) * 0.5
    c = rng.standard_normal(4).astype(np.float32)
    ho, co, lg, emb, rc = oracle.policy_cnn(WC, w, obs, la, ate, h, c)
    assert rc == 0
    th, tc, tl, te = torch_forward(w, obs, la, ate, h, c)
    np.testing.assert_allclose(emb, te, rtol=1e-12, atol=1e-12)
    # the oracle stores h', c', logits as fp32 (one rounding)
    np.testing.assert_allclose(ho, th, rtol=1e-7, atol=1e-7)
    np.testing.assert_allclose(co, tc, rtol=1e-7, atol=1e-7)
    np.testing.assert_allclose(lg, tl, rtol=2e-6, atol=2e-7)


def test_zero_weights_give_uniform_softmax():
    # all-zero params, any observation -> uniform probabilities (0.2 each)
    obs = (np.random.default_rng(1).random((15, 15, 3)) < 0.5).astype(np.float64)
    ho, co, lg, emb, rc = oracle.policy_cnn(WC, np.zeros(2445, np.float32), obs, 3, 1,
                                             np.ones(4, np.float32), np.ones(4, np.float32))
    assert rc == 0 and np.all(lg == 0.0)
    # h' = sigmoid(0) * tanh(sigmoid(0) * c + sigmoid(0) * tanh(0)) = 0.5 tanh(0.5)
    np.testing.assert_allclose(co, 0.5, rtol=1e-7)
    np.testing.assert_allclose(ho, 0.5 * math.tanh(0.5), rtol=1e-7)
    _, probs, _ = oracle.sample_action(7, 0, 0, lg)
    np.testing.assert_allclose(probs, 0.2, rtol=1e-15)


def test_sampling_closed_forms():
    # logits (1,0,0,0,0) -> P(0) = e^50 / (e^50 + 4)
    lg = np.array([1, 0, 0, 0, 0], np.float32)
    a, probs, _ = oracle.sample_action(5, 3, 11, lg)
    assert a == 0
    np.testing.assert_allclose(probs[0], 1.0 - 4.0 / (math.exp(50.0) + 4.0), rtol=0, atol=1e-300)
    np.testing.assert_allclose(probs[1:], 1.0 / (math.exp(50.0) + 4.0), rtol=1e-12)
    # temperature 1/50: logits 0.02 apart are softmax(1, 0) apart
    a, probs, _ = oracle.sample_action(5, 3, 11, np.array([0.02, 0, 0, 0, 0], np.float32))
    np.testing.assert_allclose(probs[0] / probs[1], math.exp(50.0 * float(np.float32(0.02))), rtol=1e-12)


def test_sampling_inverse_cdf_and_frequencies():
    rng = np.random.default_rng(9)
    seed = 1234
    counts = np.zeros(5, np.int64)
    n = 100_000
    lg_u = np.zeros(5, np.float32)
    for cell in range(n):
        a, _, m = oracle.sample_action(seed, 17, cell, lg_u)
        counts[a] += 1
    # uniform probs, 10^5 samples -> each frequency 0.2 +- 0.01
    assert np.all(np.abs(counts / n - 0.2) < 0.01), counts
    for k in range(300):
        lg = (rng.standard_normal(5) * 0.05).astype(np.float32)
        cell, step = int(rng.integers(0, 80000)), int(rng.integers(0, 10**6))
        a, probs, m = oracle.sample_action(seed, step, cell, lg)
        z = 50.0 * lg.astype(np.float64)
        p = np.exp(z - z.max())
        p /= p.sum()
        np.testing.assert_allclose(probs, p, rtol=1e-12)
        u = oracle.draw4(seed, oracle.P_ACTION, step, cell)[0] / 2.0**32
        cum = np.cumsum(p)[:4]
        assert a == int(np.searchsorted(cum, u, side="right"))
        assert m == pytest.approx(np.min(np.abs(u - cum)), rel=1e-9, abs=1e-15)


def test_observation_channels():
    wc = WC.replace(rows=20, cols=24)
    R = np.zeros((20, 24), np.uint8)
    O = np.zeros((20, 24), np.uint8)
    R[2, 5] = 1
    O[0, 0] = 1
    O[3, 1] = 1
    x = oracle.observe_paper(wc, R, O, 0, 0)  # agent at the top-left corner
    assert x.shape == (15, 15, 3)
    walls = np.ones((15, 15))
    walls[7:, 7:] = 0.0  # rows y-7..y+7, cols x-7..x+7: on the grid from offset +0
    assert np.array_equal(x[:, :, 2], walls)
    assert x[7, 7, 1] == 1.0          # self, at the centre
    assert x[7 + 3, 7 + 1, 1] == 1.0  # the other agent at (+3, +1)
    assert x[7 + 2, 7 + 5, 0] == 1.0  # the resource at (+2, +5)
    assert x[:, :, 0].sum() == 1 and x[:, :, 1].sum() == 2
    R[3, 5] = 1
    x = oracle.observe_paper(wc, R, O, 10, 12)  # interior: no walls
    assert x[:, :, 2].sum() == 0
    assert x[:, :, 0].sum() == 1 and x[7 + (3 - 10), 7 + (5 - 12), 0] == 1.0  # (2, 5) is 8 rows up: out of view
    assert x[:, :, 1].sum() == 0  # (3, 1) is 11 columns left: out of view; O holds no self here


def test_step_uses_the_sampled_policy():
    """The world step of network 1 decides each agent's action by orc_policy_cnn +
    orc_sample_action on its own window (checked by recomputing them for every agent)."""
    wc = WC.replace(rows=30, cols=40, slots=64, n_initial=40)
    orc = oracle.OracleWorld(wc)
    for _ in range(3):
        orc.step()
    st = orc.state()
    t = orc.t
    rec = orc.step(return_actions=True)
    Rn, _ = oracle.regrow(wc, t, st["resources"])
    O = np.zeros((wc.rows, wc.cols), np.uint8)
    live = np.flatnonzero(st["alive"])
    O.flat[st["cell"][live]] = 1
    for i in live:
        y, x = divmod(int(st["cell"][i]), wc.cols)
        obs = oracle.observe_paper(wc, Rn, O, y, x)
        ho, co, lg, _, rc = oracle.policy_cnn(wc, st["weights"][i], obs, int(st["last_action"][i]),
                                              int(st["ate"][i]), st["h"][i], st["c"][i])
        a, _, _ = oracle.sample_action(wc.seeds[0], t, int(st["cell"][i]), lg)
        assert rec["actions"][i] == a


def test_cnn_world_invariants():
    """Conservation (north_star): resources(t+1) = resources(t) - eaten + grown and
    agents(t+1) = agents(t) + births - deaths, every step of a small paper world with the
    paper's network, with births, starvation and wall deaths."""
    wc = WC.replace(rows=40, cols=60, slots=200, n_initial=120, repr_steps=20)
    orc = oracle.OracleWorld(wc)
    res, pop = int(orc.st["resources"].sum()), int(orc.st["alive"].sum())
    tot = {"births": 0, "deaths_wall": 0, "deaths_energy": 0}
    for _ in range(400):  # starvation: 120 steps to reach 0, then the 200-step timer
        r = orc.step()
        assert r["status"] == 0
        assert r["resources"] == res - r["eaten"] + r["grown"]
        assert r["population"] == pop + r["births"] - r["deaths_energy"] - r["deaths_age"] - r["deaths_wall"]
        res, pop = r["resources"], r["population"]
        for k in tot:
            tot[k] += r[k]
    assert tot["births"] > 0 and tot["deaths_wall"] > 0 and tot["deaths_energy"] > 0, tot
