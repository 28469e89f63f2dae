"""Comparison protocol between the CUDA library and the oracle (SURVEY.md
§8c C.6): integer state bit-exact, fp32 LSTM state within |g - o| <= 1e-5 |o| + 2e-6
(R27: north_star's "1e-5 relative" plus an absolute floor of 2e-6 = about twice the
largest fp32-vs-fp64 difference measured near zero, 4.8e-7 .. 1e-6: fp32 summation of
~130 products cannot be relative near 0), weights bit-exact up to counted 1-ulp
differences (R29), argmax disagreements only at flagged near-ties (margin < 1e-4, R28)."""
import numpy as np

import oracle

REL, ABS = 1e-5, 2e-6
MAX_ABS_SEEN = {"h": 0.0, "c": 0.0, "logits": 0.0}  # largest |g - o| compared (reported by tests)
INT_FIELDS = ("cell", "energy", "age", "repr", "ate", "low")
REC_EXACT = ("grown", "eaten", "births", "deaths_energy", "deaths_age", "deferred_no_cell", "deferred_claim",
             "deferred_capacity", "population", "resources", "deaths_wall")


def gpu_world_state(gs: dict, w: int = 0) -> dict:
    return {k: (v[w] if isinstance(v, np.ndarray) else v) for k, v in gs.items()}


def close(g, o, rel=REL, abs_=ABS):
    g = np.asarray(g, np.float64)
    o = np.asarray(o, np.float64)
    return np.abs(g - o) <= rel * np.abs(o) + abs_


def ulp_diff(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    ia = a.astype(np.float32).view(np.int32).astype(np.int64)
    ib = b.astype(np.float32).view(np.int32).astype(np.int64)
    ia = np.where(ia < 0, -(ia & 0x7FFFFFFF), ia)
    ib = np.where(ib < 0, -(ib & 0x7FFFFFFF), ib)
    return np.abs(ia - ib)


def compare_ints(g: dict, o: dict, where: str = ""):
    """alive mask over all slots, integer fields over live slots, resources everywhere."""
    assert g["t"] == o["t"], f"{where}: t {g['t']} != {o['t']}"
    assert np.array_equal(g["resources"], o["resources"]), f"{where}: resources differ at " \
        f"{np.argwhere(g['resources'] != o['resources'])[:5].tolist()}"
    assert np.array_equal(g["alive"], o["alive"]), f"{where}: alive differs at slots " \
        f"{np.flatnonzero(g['alive'] != o['alive'])[:10].tolist()}"
    live = o["alive"] == 1
    for f in INT_FIELDS:
        bad = np.flatnonzero(g[f][live] != o[f][live])
        assert bad.size == 0, f"{where}: {f} differs at live slots {np.flatnonzero(live)[bad][:10].tolist()}"


def compare_floats(g: dict, o: dict, slots, where: str = ""):
    for f in ("h", "c", "logits"):
        d = np.abs(np.asarray(g[f][slots], np.float64) - o[f][slots])
        if d.size:
            MAX_ABS_SEEN[f] = max(MAX_ABS_SEEN[f], float(d.max()))
        ok = close(g[f][slots], o[f][slots])
        assert ok.all(), (f"{where}: {f} out of tolerance at slots "
                          f"{np.asarray(slots)[np.flatnonzero(~ok.all(axis=1))][:5].tolist()}: "
                          f"max |d| {np.max(np.abs(g[f][slots].astype(np.float64) - o[f][slots])):.3g}")


def compare_weights(g: np.ndarray, o: np.ndarray, live, max_ulp_frac=1e-6, where: str = ""):
    """Bit-exact except counted 1-ulp differences (fp64 transcendentals, R29)."""
    d = ulp_diff(g[live], o[live])
    assert d.max(initial=0) <= 1, f"{where}: weights differ by {d.max()} ulp"
    n1 = int((d == 1).sum())
    assert n1 <= max(2, max_ulp_frac * d.size), f"{where}: {n1} one-ulp weight differences"
    return n1


def argmax_with_margin(logits: np.ndarray):
    a = np.argmax(logits, axis=-1)
    s = np.sort(logits.astype(np.float64), axis=-1)
    return a, s[..., -1] - s[..., -2]


def compare_record(grec, orec, where=""):
    for f in REC_EXACT:
        assert int(grec[f]) == int(orec[f]), f"{where}: record {f} gpu {int(grec[f])} oracle {int(orec[f])}"


def lockstep(world, orc: "oracle.OracleWorld", steps: int, check_weights_every: int = 0, sync_floats: bool = True,
             w: int = 0, fields_no_weights=True):
    """M2 + M3 protocol: every step the oracle takes the GPU's h, c (one-step float check,
    M3), decides actions with its own policy, the GPU is forced to the oracle's actions
    (M2), then integer state and step records must be bit-exact and floats within R27.
    The GPU's own argmax must equal the oracle's except at flagged near-ties.
    Returns (near_tie_disagreements, n_compared_agent_steps, one_ulp_weights)."""
    from paper_2302_09334_b200.sim import STATE_FIELDS
    fields = tuple(f for f in STATE_FIELDS if f != "weights") if fields_no_weights else STATE_FIELDS
    nw = world.n_worlds
    flips = 0
    n_cmp = 0
    n_ulp = 0
    for step in range(steps):
        g0 = gpu_world_state(world.get_state(("h", "c", "alive")), w)
        if sync_floats:
            live0 = g0["alive"] == 1
            orc.st["h"][live0] = g0["h"][live0]
            orc.st["c"][live0] = g0["c"][live0]
        alive_start = orc.st["alive"].copy() == 1
        orec = orc.step(return_actions=True)
        assert orec["status"] == 0
        acts = orec["actions"]
        forced = np.full((nw, world.wc.slots), 255, np.uint8)
        forced[w] = acts
        world.set_forced_actions(forced)
        world.step(1)
        g = gpu_world_state(world.get_state(fields), w)
        o = orc.st
        where = f"step {orec['t']}"
        compare_ints(g, {**o, "t": orc.t}, where)
        grec = world.step_log(orec["t"], 1)[0, w]
        compare_record(grec, orec, where)
        # floats: agents alive at start and not replaced by a newborn in their slot
        keep = alive_start & (o["alive"] == 1) & (o["age"] > 0)
        slots = np.flatnonzero(keep)
        if slots.size:
            compare_floats(g, o, slots, where)
            ga, gm = argmax_with_margin(g["logits"][slots])
            oa, om = argmax_with_margin(o["logits"][slots])
            dis = ga != acts[slots]
            if dis.any():
                near = (gm[dis] < 1e-4) | (om[dis] < 1e-4)
                assert near.all(), f"{where}: unflagged argmax disagreement at slots {slots[dis][~near][:5]}"
                flips += int(dis.sum())
            n_cmp += slots.size
        if check_weights_every and (step + 1) % check_weights_every == 0:
            gw = world.get_state(("weights",))["weights"][w]
            n_ulp += compare_weights(gw, o["weights"], o["alive"] == 1, where=where)
    world.set_forced_actions(None)
    return flips, n_cmp, n_ulp


MAX_ULP_SEEN = {"h": 0, "c": 0, "logits": 0}


def lockstep_sampled(world, orc: "oracle.OracleWorld", steps: int, check_weights_every: int = 0, w: int = 0,
                     max_ulp: int = 1):
    """The M2 + M3 protocol for network 1, whose actions are SAMPLED (R38):
    every step the oracle takes the GPU's h, c, samples its own actions, the GPU is forced
    to them; integer state and records bit-exact, floats within R27; and the GPU's OWN
    sampled action of every agent alive at the step's start (sim_get_policy_actions) equals
    the oracle's except where either side's sampling margin |u - CDF| is below 1e-4.
    k_policy_cnn_blk evaluates the network in fp64 like the oracle (only the summation order
    differs), so beyond R27 its stored h', c' and logits must be within `max_ulp` fp32 ulps.
    Returns (near_tie_disagreements, n_compared_agent_steps, one_ulp_weights)."""
    from paper_2302_09334_b200.sim import STATE_FIELDS
    fields = tuple(f for f in STATE_FIELDS if f != "weights")
    seed = int(world.wc.seeds[w])
    nw = world.n_worlds
    flips = n_cmp = n_ulp = 0
    for step in range(steps):
        g0 = gpu_world_state(world.get_state(("h", "c", "alive")), w)
        live0 = g0["alive"] == 1
        orc.st["h"][live0] = g0["h"][live0]
        orc.st["c"][live0] = g0["c"][live0]
        alive_start = orc.st["alive"].copy() == 1
        cells_start = orc.st["cell"].copy()
        t = orc.t
        orec = orc.step(return_actions=True)
        assert orec["status"] == 0
        acts = orec["actions"]
        forced = np.full((nw, world.wc.slots), 255, np.uint8)
        forced[w] = acts
        world.set_forced_actions(forced)
        world.step(1)
        g = gpu_world_state(world.get_state(fields), w)
        o = orc.st
        where = f"step {orec['t']}"
        compare_ints(g, {**o, "t": orc.t}, where)
        compare_record(world.step_log(orec["t"], 1)[0, w], orec, where)
        keep = alive_start & (o["alive"] == 1) & (o["age"] > 0)
        slots = np.flatnonzero(keep)
        if slots.size:
            compare_floats(g, o, slots, where)
            for f in ("h", "c", "logits"):
                u = ulp_diff(g[f][slots], o[f][slots])
                MAX_ULP_SEEN[f] = max(MAX_ULP_SEEN[f], int(u.max()))
                assert u.max() <= max_ulp, f"{where}: {f} differs by {int(u.max())} ulp (fp64 evaluation on both sides)"
        own = world.policy_actions()[w]
        start = np.flatnonzero(alive_start)
        dis = start[own[start] != acts[start]]
        for i in dis:
            if o["alive"][i] == 1 and o["age"][i] == 0:
                continue  # died and its slot was reused by a newborn: the step's logits are gone
            ent = int(i) if getattr(world.wc, "colocate", 0) else int(cells_start[i])  # R47 / R38
            _, _, mo = oracle.sample_action(seed, t, ent, o["logits"][i])
            _, _, mg = oracle.sample_action(seed, t, ent, g["logits"][i])
            assert min(mo, mg) < 1e-4, f"{where}: unflagged sampling disagreement at slot {i} (margins {mo}, {mg})"
        flips += int(dis.size)
        n_cmp += int(start.size)
        if check_weights_every and (step + 1) % check_weights_every == 0:
            gw = world.get_state(("weights",))["weights"][w]
            n_ulp += compare_weights(gw, o["weights"], o["alive"] == 1, where=where)
    world.set_forced_actions(None)
    return flips, n_cmp, n_ulp
