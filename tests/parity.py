"""Parity helpers: run the CUDA path (through the C-ABI binding) and the fp64 oracle on the same
seeded inputs and compare element by element.

Contract:
* bit-exact: Philox-driven integers and every decision -- delay bits, p-index, force threshold,
  dropout timers, has_last, k_f, episode counters, `prev` (a copy of the input), integer stats;
* floats: |gpu - oracle| / max(|oracle|, floor) <= 1e-6 with a per-channel floor;
* backlash rail knife-edges: where the oracle's fp64 rail margin |s + a d dt - sgn(a)| is below
  KNIFE_TAU, fp32 and fp64 may legitimately take different sides of the clamp; that actuator is
  excused until both sides agree again, and such events are counted.
"""
from __future__ import annotations

import numpy as np

TOL = 1e-6
KNIFE_TAU = 1e-5

OUT_FLOORS = {"out_actions": 1.0, "out_dt": 0.008}


def rel_err(g, o, floor):
    g = np.asarray(g, dtype=np.float64)
    o = np.asarray(o, dtype=np.float64)
    return np.abs(g - o) / np.maximum(np.abs(o), floor)


def assert_close(name, g, o, floor, tol=TOL, mask=None):
    e = rel_err(g, o, floor)
    if mask is not None:
        e = np.where(mask, e, 0.0)
    bad = e > tol
    if bad.any():
        idx = np.argwhere(bad)[:5]
        detail = [(tuple(i), float(np.asarray(g)[tuple(i)]), float(np.asarray(o)[tuple(i)])) for i in idx]
        raise AssertionError(f"{name}: {bad.sum()} elements beyond {tol} (max {e.max():.3g}); first {detail}")
    return float(e.max()) if e.size else 0.0


def compare_obs(g_obs, o_obs, t=None):
    """out_obs: rel goal (floor 1) w >= 0 canonical -- compare up to sign when |w| ~ 0 [Q16];
    tips and object (floor 0.1 m)."""
    rel_g, rel_o = g_obs[:, 0:4], o_obs[:, 0:4]
    flip = (np.abs(rel_o[:, 0]) < 1e-6) & (np.sum(rel_g * rel_o, axis=1) < 0)
    rel_g = np.where(flip[:, None], -rel_g, rel_g)
    m1 = assert_close(f"out_obs.rel_goal t={t}", rel_g, rel_o, 1.0)
    m2 = assert_close(f"out_obs.tips t={t}", g_obs[:, 4:19], o_obs[:, 4:19], 0.1)
    m3 = assert_close(f"out_obs.obj t={t}", g_obs[:, 19:22], o_obs[:, 19:22], 0.1)
    return max(m1, m2, m3)


class KnifeTracker:
    """Per-(env, actuator) excusal of backlash rail knife-edges."""

    def __init__(self, n, tau=None):
        self.tau = KNIFE_TAU if tau is None else tau
        self.excused = np.zeros((n, 20), dtype=bool)
        self.events = 0
        self.excused_mismatches = 0

    def update_before_compare(self, margin):
        k = margin < self.tau
        self.events += int(k.sum())
        self.excused |= k

    def compare_actions(self, g, o, t=None):
        e = rel_err(g, o, 1.0)
        bad = e > TOL
        unexcused = bad & ~self.excused
        if unexcused.any():
            idx = np.argwhere(unexcused)[:5]
            raise AssertionError(f"out_actions t={t}: {unexcused.sum()} mismatches, first "
                                 f"{[(tuple(i), float(g[tuple(i)]), float(o[tuple(i)])) for i in idx]}")
        self.excused_mismatches += int((bad & self.excused).sum())

    def resync(self, g_slack, o_slack):
        """Clear excusal where the slack states agree again (both exactly on the same rail or
        within tolerance and neither on a rail)."""
        same = (g_slack == o_slack) | ((np.abs(g_slack - o_slack) <= TOL) & (np.abs(o_slack) < 1) & (np.abs(g_slack) < 1))
        self.excused &= ~same


HOLD_LAYERS = (1 << 5) | (1 << 6)   # DROPOUT | OCCLUSION
SMOOTH, SUBSTEP = 1 << 9, 1 << 10


def compare_records(G: dict, O: list, phys_g=None, strict_state=True, knife=None, mask=0x1FF):
    """Compare exported GPU per-env state G (dict of arrays) with oracle env dicts O.
    With neither DROPOUT nor OCCLUSION enabled the hold state (has_last, last readings) is
    unobservable; the kernel does not move those bytes, so they are not compared."""
    n = len(O)
    get = lambda k: np.array([o[k] for o in O])  # noqa: E731
    for k in ("episode", "delay_bits", "p_index", "t_force", "k_f"):
        assert np.array_equal(G[k].astype(np.int64), get(k).astype(np.int64)), k
    # flags = dropout timers (4 bits per tip) + has_last (bit 20)
    tim = get("timer")
    flags_o = np.zeros(n, dtype=np.int64)
    for i in range(5):
        flags_o |= tim[:, i].astype(np.int64) << (4 * i)
    hold = bool(mask & HOLD_LAYERS)
    if hold:
        flags_o |= get("has_last").astype(np.int64) << 20
    assert np.array_equal(G["flags"].astype(np.int64), flags_o), "flags (dropout timers / has_last)"
    mass = get("mass")
    assert_close("lambda", G["lambda"], get("lambda"), 1e-30)
    assert_close("mass", G["mass"], mass, 1e-30)
    assert_close("dneg", G["dneg"], get("dneg"), 1.0)
    assert_close("dpos", G["dpos"], get("dpos"), 1.0)
    assert_close("c_act", G["c_act"], get("c_act"), 0.03)
    assert_close("off_tip", G["off_tip"], get("off_tip"), 3.3e-3)
    assert_close("c_obj", G["c_obj"], get("c_obj"), 5e-3)
    assert_close("q_c", G["q_c"], get("q_c"), 1.0)
    if mask & SMOOTH:   # prev holds the smoothed (computed) command: fp32 vs fp64
        assert_close("prev", G["prev"], get("prev"), 1.0)
        assert_close("ema", G["ema"], get("ema"), 1.0)
    else:
        assert np.array_equal(G["prev"].astype(np.float64), get("prev")), "prev (copy of the input)"
    slack_o = get("slack")
    if knife is not None:
        knife.resync(G["slack"].astype(np.float64), slack_o)
        assert_close("slack", G["slack"], slack_o, 1.0, tol=1e-5, mask=~knife.excused)
    elif strict_state:
        assert_close("slack", G["slack"], slack_o, 1.0)
    if hold:
        assert_close("last", G["last"], get("last"), 0.1)
    assert_close("f_trig", G["f_trig"], get("f_trig"), np.maximum(mass[:, None], 1e-30))
    if phys_g is not None:
        # floor |base|: ADD_GAUSS can cancel base + sigma z towards 0
        from workload import presets
        ph = get("phys")[:, : phys_g.shape[1]]
        base = np.abs(np.array([d[3] for d in presets.PAPER["phys"]]))[: phys_g.shape[1]]
        assert_close("phys", phys_g, ph, np.maximum(base[None, :], 1e-30))


STAT_INT = list(range(0, 12))
STAT_MOM = list(range(16, 24))


def compare_stats(g, o, n_envs, knife_events=0, t=None):
    """Integer slots exact; fp64 moment slots to 1e-6 of a magnitude bound (they sum fp32 vs fp64
    per-env values).  Backlash-gate counts may differ by the knife-edge count."""
    for s in STAT_INT:
        if s in (7, 8, 9) and knife_events:
            assert abs(g[s] - o[s]) <= 2 * knife_events, (t, s, g[s], o[s])
        else:
            assert g[s] == o[s], (t, s, g[s], o[s])
    scale = {16: 0.09 * n_envs, 17: 0.01 * n_envs, 18: 2.0 * 20 * n_envs, 19: 20 * n_envs,
             20: 20 * n_envs, 21: 20 * n_envs, 22: 15 * n_envs, 23: 10 * n_envs}
    for s in STAT_MOM:
        assert abs(g[s] - o[s]) <= 1e-6 * max(abs(o[s]), scale[s]) * (1 + knife_events), (t, s, g[s], o[s])


# ---- state transfer between the two sides (test infrastructure: marshalling, no method arithmetic) ----
GPU_TO_ORACLE_FIELDS = ("episode", "delay_bits", "p_index", "t_force", "k_f", "lambda", "mass", "dneg", "dpos",
                        "c_act", "off_tip", "c_obj", "q_c", "prev", "slack", "last", "f_trig", "ema")


def oracle_env_from_gpu(G: dict, i: int, orc) -> dict:
    """The oracle env dict of GPU-exported env i (dr_env_state, fp32 -> fp64 exactly): record and
    state fields copied, the flags word split into the dropout timers and has_last, and the episode's
    force probability looked up from its p-index in the oracle's own table."""
    d = {k: np.asarray(G[k][i]).astype(np.float64) if np.asarray(G[k][i]).dtype.kind == "f" else G[k][i]
         for k in GPU_TO_ORACLE_FIELDS}
    flags = int(G["flags"][i])
    d["timer"] = np.array([(flags >> (4 * t)) & 15 for t in range(5)], dtype=np.int64)
    d["has_last"] = (flags >> 20) & 1
    d["p_force"] = orc.force_p(int(G["p_index"][i]))
    return d


def state_array_from_numpy(states, G: dict):
    """Write the dict-of-arrays G (states_to_numpy shape) back into a ctypes dr_env_state array."""
    raw = np.frombuffer(states, dtype=np.uint32).reshape(len(states), -1)
    off = 0
    for name, ty in type(states[0])._fields_:
        key = "lambda" if name == "lambda_" else name
        n = ty._length_ if hasattr(ty, "_length_") else 1
        col = np.asarray(G[key]).reshape(len(states), n)
        raw[:, off:off + n] = col.view(np.uint32) if col.dtype == np.float32 else col.astype(np.uint32)
        off += n
    return states
