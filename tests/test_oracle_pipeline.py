"""Pins for the oracle's reset + step pipeline against what the paper fixes: the std tables
(Table obs-noise, Table action-noise), delay/hold/decay semantics
(PAPER.md:64-66, 77-79, 113-115), timing, closed-form statistics, special
cases (layers off), and the independence of results from how envs are partitioned."""
import json
import math
import os

import numpy as np
import pytest
from scipy import stats
from scipy.spatial.transform import Rotation

from conftest import GOLDEN
from workload import gen, presets
from workload.presets import (ACT_NOISE, BACKLASH, DELAY, DROPOUT, FORCE, FULL, OBS_NOISE,
                              OCCLUSION, PHYS, TIMING)

SEED = presets.SEED_DR


@pytest.fixture(scope="module")
def paper():
    with open(os.path.join(GOLDEN, "paper_values.json")) as f:
        return json.load(f)


def _oracle(mask, n, **kw):
    from oracle.oracle import Oracle
    return Oracle(presets.preset(mask, **kw), n, SEED)


def _se_std(n):
    return 1.0 / math.sqrt(2.0 * n)


def test_presets_are_the_paper_tables(paper):
    P = presets.PAPER
    on, an = paper["obs_noise_std"], paper["action_noise_frac_of_range"]
    rng_ = an["action_range"]
    assert P["act_sigma_uadd"] == pytest.approx(an["uncorrelated_additive"] * rng_)
    assert P["act_sigma_cadd"] == pytest.approx(an["correlated_additive"] * rng_)
    assert P["act_sigma_mult"] == pytest.approx(an["uncorrelated_multiplicative"])
    assert (P["tip_corr"], P["tip_uncorr"]) == (on["fingertip_corr_m"], on["fingertip_uncorr_m"])
    assert (P["obj_corr"], P["obj_uncorr"]) == (on["object_pos_corr_m"], on["object_pos_uncorr_m"])
    assert (P["rot_corr"], P["rot_uncorr"]) == (on["object_rot_corr_rad"], on["object_rot_uncorr_rad"])
    assert (P["tip_marker"], P["base_marker"]) == (on["fingertip_marker_m"], on["hand_base_marker_m"])
    assert P["delay_prob"] == paper["delay"]["prob"]
    tm = paper["timing"]
    assert (P["dt_base"], P["lambda_lo"], P["lambda_hi"]) == (tm["dt_base_s"], tm["lambda_lo"], tm["lambda_hi"])
    assert P["step_nominal"] == tm["step_nominal_s"] == tm["substeps"] * tm["dt_base_s"]
    assert P["delta_jitter_std"] == paper["backlash"]["jitter_std"]
    assert P["backlash_eps"] == paper["backlash"]["eps"]
    assert P["dropout_rate_hz"] == paper["dropout"]["rate_per_s"]
    assert P["dropout_hold_steps"] == math.ceil(paper["dropout"]["duration_s"] / tm["step_nominal_s"])
    f = paper["force"]
    assert (P["force_p_lo"], P["force_p_hi"], P["force_accel_std"], P["force_decay_per_step"]) == \
        (f["p_lo"], f["p_hi"], f["accel_std_m_s2"], f["decay_per_80ms"])


# ----------------------------------------------------------------------------------------------
# episode reset
# ----------------------------------------------------------------------------------------------
@pytest.fixture(scope="module")
def reset_records():
    n = 30000
    orc = _oracle(FULL, n)
    recs = [orc.env(i) for i in range(n)]
    out = {k: np.array([r[k] for r in recs]) for k in recs[0]}
    return out


def test_reset_correlated_obs_offsets(reset_records, paper):
    R = reset_records
    on = paper["obs_noise_std"]
    n = R["c_obj"].size
    # std of correlated object-position offset = 5 mm within 3 %
    assert abs(R["c_obj"].std() / on["object_pos_corr_m"] - 1) < min(0.03, 5 * _se_std(n))
    # [Q14] tip offset = corr 1 mm + marker 3 mm - base marker 1 mm (shared by the 5 tips)
    tip = R["off_tip"].reshape(-1, 5, 3)
    exp_std = math.sqrt(on["fingertip_corr_m"] ** 2 + on["fingertip_marker_m"] ** 2 + on["hand_base_marker_m"] ** 2)
    assert abs(tip.std() / exp_std - 1) < 5 * _se_std(tip.size) + 0.005
    cov01 = np.mean(tip[:, 0, :] * tip[:, 1, :])
    assert abs(cov01 - on["hand_base_marker_m"] ** 2) < 5 * exp_std ** 2 / math.sqrt(tip.shape[0] * 3)
    # orientation offset: angle ~ N(0, 0.1^2) about a random axis [Q15]
    q = R["q_c"]
    ang = 2 * np.arccos(np.clip(np.abs(q[:, 0]), 0, 1))
    assert abs(ang.mean() - on["object_rot_corr_rad"] * math.sqrt(2 / math.pi)) < 0.02 * on["object_rot_corr_rad"]
    assert np.allclose(np.linalg.norm(q, axis=1), 1.0, atol=1e-12)


def test_reset_action_params(reset_records, paper):
    R = reset_records
    n_env = R["delay_bits"].shape[0]
    # delay flags Bernoulli(0.5) per actuator
    bits = ((R["delay_bits"][:, None] >> np.arange(20)[None, :]) & 1).astype(float)
    assert abs(bits.mean() - paper["delay"]["prob"]) < 5 * 0.5 / math.sqrt(bits.size)
    assert R["delay_bits"].max() < (1 << 20)
    # correlated action noise 1.5 % of range 2 (Table action-noise)
    an = paper["action_noise_frac_of_range"]
    assert abs(R["c_act"].std() / (an["correlated_additive"] * an["action_range"]) - 1) < 5 * _se_std(R["c_act"].size)
    # backlash widths: calibrated + N(0, 0.1); calibrations >> 0.1 so no clamping
    cal_n = np.array(presets.PAPER["delta_cal_neg"])
    cal_p = np.array(presets.PAPER["delta_cal_pos"])
    jn, jp = R["dneg"] - cal_n, R["dpos"] - cal_p
    for j in (jn, jp):
        assert abs(j.std() / paper["backlash"]["jitter_std"] - 1) < 5 * _se_std(j.size)
        assert abs(j.mean()) < 5 * 0.1 / math.sqrt(j.size)
    # timing lambda ~ U[1250, 10000]: KS vs scipy uniform
    tm = paper["timing"]
    lam = R["lambda"]
    assert stats.kstest(lam, "uniform", args=(tm["lambda_lo"], tm["lambda_hi"] - tm["lambda_lo"])).pvalue > 1e-3
    # force p loguniform on [0.1 %, 10 %] (KS at 1 %)
    f = paper["force"]
    lp = np.log(R["p_force"])
    assert stats.kstest(lp, "uniform", args=(math.log(f["p_lo"]), math.log(f["p_hi"] / f["p_lo"]))).pvalue > 0.01
    assert ((R["p_force"] >= f["p_lo"]) & (R["p_force"] <= f["p_hi"])).all()
    assert n_env == lam.shape[0]


def test_reset_physics_descriptors(reset_records):
    """[Q20] descriptor schema: per-kind distribution checks."""
    R = reset_records
    ph = R["phys"]
    table = presets.PAPER["phys"]
    n = ph.shape[0]
    for i in range(0, 256, 17):
        k, a, b, base = table[i]
        v = ph[:, i]
        if k == presets.PHYS_UNIFORM_SCALE:
            assert stats.kstest(v / base, "uniform", args=(a, b - a)).pvalue > 1e-3
        elif k == presets.PHYS_LOGUNIFORM_SCALE:
            assert stats.kstest(np.log(v / base), "uniform", args=(math.log(a), math.log(b / a))).pvalue > 1e-3
        elif k == presets.PHYS_ADD_GAUSS:
            assert stats.kstest((v - base) / a, "norm").pvalue > 1e-3
        elif k == presets.PHYS_MUL_LOGNORMAL:
            assert stats.kstest(np.log(v / base) / a, "norm").pvalue > 1e-3
    # the force std uses this episode's mass [Q18]
    assert np.array_equal(R["mass"], ph[:, presets.PAPER["mass_index"]])
    # parameters of different slots are independent draws
    assert abs(np.corrcoef(ph[:, 0], ph[:, 4])[0, 1]) < 5 / math.sqrt(n)
    assert abs(np.corrcoef(ph[:, 2], ph[:, 6])[0, 1]) < 5 / math.sqrt(n)


def test_reset_state_zeroed(reset_records):
    R = reset_records
    for k in ("prev", "slack", "last", "f_trig", "timer"):
        assert (R[k] == 0).all(), k
    assert (R["has_last"] == 0).all() and (R["k_f"] == 0).all() and (R["episode"] == 0).all()


def test_layers_off_reset_is_base():
    """all layers off -> params equal base and all offsets zero."""
    orc = _oracle(0, 50)
    base = np.array([d[3] for d in presets.PAPER["phys"]])
    for i in range(50):
        e = orc.env(i)
        assert np.array_equal(e["phys"], base)
        for k in ("dneg", "dpos", "c_act", "off_tip", "c_obj"):
            assert (e[k] == 0).all(), k
        assert list(e["q_c"]) == [1.0, 0.0, 0.0, 0.0]
        assert e["delay_bits"] == 0 and e["lambda"] == 0 and e["t_force"] == 0


# ----------------------------------------------------------------------------------------------
# step
# ----------------------------------------------------------------------------------------------
def test_layers_off_step_identity():
    """Every layer disabled -> the transform is the identity on the policy view
    (SPEC.md:150, 177, 186, 195, 218); the relative goal is goal (x) conj(q_obj) (scipy)."""
    n, T = 64, 5
    acts, obs = gen.frames(n, T, seed=11)
    orc = _oracle(0, n)
    for t in range(T):
        r = orc.step(acts[t], obs[t])
        assert np.array_equal(r["out_actions"], acts[t].astype(np.float64))
        assert (r["out_dt"] == 0.008).all()
        assert (r["out_force"] == 0).all()
        assert np.array_equal(r["out_obs"][:, 4:22], obs[t][:, 0:18].astype(np.float64))
        qo = obs[t][:, 18:22].astype(np.float64)
        goal = obs[t][:, 22:26].astype(np.float64)
        Rg = Rotation.from_quat(goal[:, [1, 2, 3, 0]])
        Ro = Rotation.from_quat(qo[:, [1, 2, 3, 0]])
        ref = (Rg * Ro.inv()).as_quat()[:, [3, 0, 1, 2]]
        ref *= np.sign(ref[:, :1])
        assert np.allclose(r["out_obs"][:, 0:4], ref, atol=1e-7)
        assert (r["out_obs"][:, 0] >= 0).all()


def test_value_view_isolation():
    """noise is applied to the policy inputs only -- inputs are never written."""
    n = 32
    acts, obs = gen.frames(n, 3, seed=5)
    a0, o0 = acts.copy(), obs.copy()
    orc = _oracle(FULL, n)
    for t in range(3):
        orc.step(acts[t], obs[t])
    assert np.array_equal(acts, a0) and np.array_equal(obs, o0)


def test_timing(paper):
    tm = paper["timing"]
    n, T = 2000, 20
    acts, obs = gen.frames(n, 1)
    # lambda fixed at 1250 -> mean substep 8 ms + 1/1250 s = 8.8 ms within 1 %
    orc = _oracle(TIMING, n, lambda_lo=1250.0, lambda_hi=1250.0)
    dts = np.concatenate([orc.step(acts[0], obs[0])["out_dt"].ravel() for _ in range(T)])
    assert (dts >= tm["dt_base_s"]).all()
    assert abs(dts.mean() / (tm["dt_base_s"] + 1 / 1250.0) - 1) < 0.01
    assert stats.kstest(dts - tm["dt_base_s"], "expon", args=(0, 1 / 1250.0)).pvalue > 1e-3
    # unconditional: E[dt_k] = 8 ms + E[1/lambda] = 8 ms + ln(8)/8750 s = 8.2377 ms
    orc = _oracle(TIMING, n)
    dts = np.concatenate([orc.step(acts[0], obs[0])["out_dt"].ravel() for _ in range(T)])
    e_inv = math.log(tm["lambda_hi"] / tm["lambda_lo"]) / (tm["lambda_hi"] - tm["lambda_lo"])
    assert abs(dts.mean() - (tm["dt_base_s"] + e_inv)) < 0.003 * 0.0082377
    assert (dts >= tm["dt_base_s"]).all()
    # stats slots: sum of dt_env
    r = orc.step(acts[0], obs[0])
    assert math.isclose(r["stats"][16], r["out_dt"].sum(axis=1).sum(), rel_tol=1e-12)


def test_delay_is_a_one_step_shift():
    """flagged actuator, inputs x0, x1, x2 -> outputs 0, x0, x1 (delayed
    by one environment step); flags change only at episode boundaries."""
    n, T = 16, 6
    acts, obs = gen.frames(n, T, seed=3)
    orc = _oracle(DELAY, n, delay_prob=1.0)
    outs = [orc.step(acts[t], obs[t])["out_actions"] for t in range(T)]
    assert (outs[0] == 0).all()
    for t in range(1, T):
        assert np.array_equal(outs[t], acts[t - 1].astype(np.float64))
    orc = _oracle(DELAY, n, delay_prob=0.0)
    for t in range(T):
        assert np.array_equal(orc.step(acts[t], obs[t])["out_actions"], acts[t].astype(np.float64))
    # p = 0.5: per-actuator behaviour is exactly one of {identity, shift}, fixed within an episode
    orc = _oracle(DELAY, n)
    bits = np.array([orc.env(i)["delay_bits"] for i in range(n)])
    outs = [orc.step(acts[t], obs[t])["out_actions"] for t in range(T)]
    for t in range(1, T):
        for i in range(n):
            for j in range(20):
                ref = acts[t - 1][i, j] if (bits[i] >> j) & 1 else acts[t][i, j]
                assert outs[t][i, j] == ref
    assert np.array_equal(bits, [orc.env(i)["delay_bits"] for i in range(n)])
    orc.reset(np.eye(1, n, 0, dtype=np.uint8)[0])
    assert orc.env(0)["episode"] == 1 and orc.env(1)["episode"] == 0
    assert orc.env(1)["delay_bits"] == bits[1]


def test_action_noise_statistics(paper):
    """Table action-noise, range 2 [Q8]: at a = 0 the per-step std is 0.1, the
    episode-mean std 0.03 and the pooled std sqrt(0.1^2 + 0.03^2) = 0.1044 within 2 %
    (SPEC.md:178); the multiplicative term is exactly 0 at a = 0."""
    an = paper["action_noise_frac_of_range"]
    su = an["uncorrelated_additive"] * an["action_range"]
    sc = an["correlated_additive"] * an["action_range"]
    sm = an["uncorrelated_multiplicative"]
    n, T = 1000, 40
    _, obs = gen.frames(n, 1)
    zero = np.zeros((n, 20), dtype=np.float32)
    orc = _oracle(ACT_NOISE, n)
    x = np.stack([orc.step(zero, obs[0])["out_actions"] for _ in range(T)])   # [T][n][20]
    assert abs(x.std() / math.hypot(su, sc) - 1) < 0.02
    within = (x - x.mean(axis=0, keepdims=True)).std() * math.sqrt(T / (T - 1))
    assert abs(within / su - 1) < 0.02
    ep_mean = x.mean(axis=0)
    assert abs(math.sqrt(max(ep_mean.var() - su ** 2 / T, 0)) / sc - 1) < 0.05
    # multiplicative-only
    orc = _oracle(ACT_NOISE, n, act_sigma_uadd=0.0, act_sigma_cadd=0.0)
    assert (orc.step(zero, obs[0])["out_actions"] == 0).all()
    half = np.full((n, 20), 0.5, dtype=np.float32)
    y = np.stack([orc.step(half, obs[0])["out_actions"] for _ in range(10)])
    assert abs(y.std() / (0.5 * sm) - 1) < 5 * _se_std(y.size)
    assert abs(y.mean() - 0.5) < 5 * 0.5 * sm / math.sqrt(y.size)
    # clamp to the action range
    one = np.full((n, 20), 1.0, dtype=np.float32)
    orc = _oracle(ACT_NOISE, n)
    z = orc.step(one, obs[0])["out_actions"]
    assert (z <= 1.0).all() and (z >= -1.0).all() and (z == 1.0).mean() > 0.4


def test_obs_noise_statistics(paper):
    """Table obs-noise with a static true state: per-step (uncorrelated) std of a
    fingertip 2 mm and of the object 1 mm; paired-difference std 2 sqrt(2) mm;
    episode offsets: tips sqrt(1 + 9 + 1) mm [Q14], object 5 mm."""
    on = paper["obs_noise_std"]
    n, T = 1500, 30
    acts, obs = gen.frames(n, 1)
    orc = _oracle(OBS_NOISE, n)
    y = np.stack([orc.step(acts[0], obs[0])["out_obs"] for _ in range(T)])  # [T][n][22]
    tips = y[:, :, 4:19] - obs[0][None, :, 0:15].astype(np.float64)
    objp = y[:, :, 19:22] - obs[0][None, :, 15:18].astype(np.float64)
    w_tip = (tips - tips.mean(axis=0, keepdims=True)).std() * math.sqrt(T / (T - 1))
    w_obj = (objp - objp.mean(axis=0, keepdims=True)).std() * math.sqrt(T / (T - 1))
    assert abs(w_tip / on["fingertip_uncorr_m"] - 1) < 0.01
    assert abs(w_obj / on["object_pos_uncorr_m"] - 1) < 0.02
    d = tips[1] - tips[0]
    assert abs(d.std() / (2 * math.sqrt(2) * 1e-3) - 1) < 0.02
    off_std = math.sqrt(on["fingertip_corr_m"] ** 2 + on["fingertip_marker_m"] ** 2 + on["hand_base_marker_m"] ** 2)
    em = tips.mean(axis=0)
    assert abs(math.sqrt(em.var() - on["fingertip_uncorr_m"] ** 2 / T) / off_std - 1) < 0.03
    eo = objp.mean(axis=0)
    assert abs(math.sqrt(eo.var() - on["object_pos_uncorr_m"] ** 2 / T) / on["object_pos_corr_m"] - 1) < 0.05
    # orientation: goal = q_obj, correlated rotation off -> rel = conj(q_u): angle half-normal, mean 0.1 sqrt(2/pi)
    o2 = obs[0].copy()
    o2[:, 22:26] = o2[:, 18:22]
    orc = _oracle(OBS_NOISE, n, rot_corr=0.0)
    rel = np.concatenate([orc.step(acts[0], o2)["out_obs"][:, 0:4] for _ in range(4)])
    ang = 2 * np.arccos(np.clip(rel[:, 0], 0, 1))
    assert abs(ang.mean() / (on["object_rot_uncorr_rad"] * math.sqrt(2 / math.pi)) - 1) < 0.03


def _held_runs(held):
    """lengths of maximal runs of True in a [T] bool array that start after step 1 and end
    before the last step (complete runs)."""
    runs, cur, start = [], 0, None
    for t, h in enumerate(held):
        if h:
            if cur == 0:
                start = t
            cur += 1
        else:
            if cur and start > 1:
                runs.append(cur)
            cur = 0
    return runs


def test_dropout_rate_and_hold(paper):
    """each fingertip marker is masked with rate 0.2/s for 1 s: per-step initiation
    probability 1 - exp(-0.016) = 0.015873 [Q11]; an isolated mask freezes the reading for exactly
    ceil(1 s / 80 ms) = 13 steps; steady masked fraction 1 - (1 - p)^13 = 0.18782."""
    d = paper["dropout"]
    p = 1 - math.exp(-d["rate_per_s"] * paper["timing"]["step_nominal_s"])
    hold = math.ceil(d["duration_s"] / paper["timing"]["step_nominal_s"])
    n, T = 400, 300
    acts, obs = gen.frames(n, T, seed=9)     # fresh frame every step: a held reading never equals raw
    orc = _oracle(DROPOUT, n)
    inits = masked = 0
    held = np.zeros((T, n, 5), dtype=bool)
    for t in range(T):
        r = orc.step(acts[t], obs[t])
        inits += r["stats"][2]
        masked += r["stats"][3] if t > 0 else 0     # step 0 has no last reading: passes through
        raw = obs[t][:, 0:15].astype(np.float64).reshape(n, 5, 3)
        out = r["out_obs"][:, 4:19].reshape(n, 5, 3)
        held[t] = ~(out == raw).all(axis=2)
    tot = n * 5 * T
    assert abs(inits / tot / p - 1) < 5 / math.sqrt(p * tot)
    # steady state (skip the first 13 steps)
    mfrac = held[hold:].mean()
    assert abs(mfrac - (1 - (1 - p) ** hold)) < 0.01
    assert masked == held.sum()
    runs = []
    for i in range(n):
        for k in range(5):
            runs += _held_runs(held[:, i, k])
    runs = np.array(runs)
    assert runs.min() == hold
    frac13 = (runs == hold).mean()
    assert abs(frac13 - (1 - p) ** (hold - 1)) < 0.03


def test_hold_last_reading_bits():
    """an occluded (or masked) marker returns its last available reading -- the
    output bits equal the previous step's output bits [Q12]; the first step of an episode passes
    through."""
    n, T = 300, 30
    acts, obs = gen.frames(n, 16, seed=21)
    orc = _oracle(OCCLUSION | DROPOUT | OBS_NOISE, n)
    prev = None
    n_held = 0
    for t in range(T):
        r = orc.step(acts[t % 16], obs[t % 16])
        out = r["out_obs"][:, 4:19].reshape(n, 5, 3)
        tips = obs[t % 16][:, 0:15]
        occ = np.array([[orc_occ(tips[i], obs[t % 16][i, 15:18], k) for k in range(5)] for i in range(n)])
        if prev is None:
            first = out
        else:
            same = (out == prev).all(axis=2)
            assert same[occ].all()
            n_held += same.sum()
        prev = out
    assert n_held > 0
    assert first is not None


def orc_occ(tips15, obj3, k):
    from oracle import oracle as O
    return O.occluded(tips15, obj3, presets.PAPER["occl_dist"], k)


def test_random_force(paper):
    """trigger rate E[p] = 0.099 / ln 100 = 0.021498 for loguniform p; per-axis
    std of the triggered force / mass = 1 m/s^2; between triggers the force decays by
    exactly 0.99 per 80 ms step."""
    f = paper["force"]
    n, T = 1500, 120
    acts, obs = gen.frames(n, 1)
    orc = _oracle(FORCE, n)
    mass = np.array([orc.env(i)["mass"] for i in range(n)])
    trig = 0
    fs, prev = [], None
    ratio_ok = 0
    for t in range(T):
        r = orc.step(acts[0], obs[0])
        trig += r["stats"][6]
        F = r["out_force"]
        ks = np.array([orc.env(i)["k_f"] for i in range(n)]) if t % 20 == 0 else None
        if prev is not None:
            newtrig = ~np.isclose(F, prev * f["decay_per_80ms"], rtol=1e-12, atol=0).all(axis=1)
            cont = (~newtrig) & (np.abs(prev).sum(axis=1) > 0)
            ratio_ok += cont.sum()
            fs.append(F[newtrig] / mass[newtrig, None])
        prev = F
        del ks
    rate = trig / (n * T)
    e_p = (f["p_hi"] - f["p_lo"]) / math.log(f["p_hi"] / f["p_lo"])
    assert abs(rate / e_p - 1) < 5 / math.sqrt(e_p * n * T)
    fz = np.concatenate(fs).ravel()
    assert abs(fz.std() / f["accel_std_m_s2"] - 1) < 5 * _se_std(fz.size) + 0.005
    assert ratio_ok > n * T * 0.3
    # fixed p: rate = T/2^32 exactly in expectation
    orc = _oracle(FORCE, n, force_p_lo=0.05, force_p_hi=0.05)
    trig = sum(orc.step(acts[0], obs[0])["stats"][6] for _ in range(40))
    assert abs(trig / (n * 40) / 0.05 - 1) < 5 / math.sqrt(0.05 * n * 40)


def test_backlash_pipeline_invariants():
    n, T = 300, 60
    acts, obs = gen.frames(n, 16, seed=2)
    orc = _oracle(TIMING | ACT_NOISE | BACKLASH, n)
    for t in range(T):
        r = orc.step(acts[t % 16], obs[t % 16])
        s = np.array([orc.env(i)["slack"] for i in range(n)]) if t % 10 == 0 else None
        if s is not None:
            assert (np.abs(s) <= 1).all()
        oa = r["out_actions"]
        assert (np.abs(oa) <= 1).all()
    st = r["stats"]
    assert st[8] + st[9] == n * 20


def test_reproducibility_and_partition_invariance():
    """Same seed -> identical results; results of an env depend only on its global
    id, so any partition of the envs across workers/GPUs gives identical per-env outputs."""
    n, T = 24, 12
    acts, obs = gen.frames(n, T, seed=4)
    from oracle.oracle import Oracle
    P = presets.preset(FULL)
    full = Oracle(P, n, SEED)
    halves = [Oracle(P, n // 2, SEED, gids=np.arange(h * n // 2, (h + 1) * n // 2)) for h in range(2)]
    pick = np.array([3, 17, 22])
    sub = Oracle(P, 3, SEED, gids=pick)
    again = Oracle(P, n, SEED)
    for t in range(T):
        if t == 6:
            m = np.zeros(n, dtype=np.uint8)
            m[pick] = 1
            m[5] = 1
            full.reset(m)
            again.reset(m)
            halves[0].reset(m[: n // 2])
            halves[1].reset(m[n // 2:])
            sub.reset(m[pick])
        a = full.step(acts[t], obs[t])
        b = [halves[h].step(acts[t][h * n // 2:(h + 1) * n // 2], obs[t][h * n // 2:(h + 1) * n // 2]) for h in range(2)]
        c = sub.step(acts[t][pick], obs[t][pick])
        d = again.step(acts[t], obs[t])
        for k in ("out_actions", "out_obs", "out_dt", "out_force"):
            assert np.array_equal(a[k], np.concatenate([b[0][k], b[1][k]])), k
            assert np.array_equal(a[k][pick], c[k]), k
            assert np.array_equal(a[k], d[k]), k
        assert np.array_equal(a["stats"], d["stats"])
    # a different seed changes the draws
    other = Oracle(P, n, SEED + 1)
    assert not np.array_equal(other.step(acts[0], obs[0])["out_obs"], Oracle(P, n, SEED).step(acts[0], obs[0])["out_obs"])


def test_openmp_build_is_bit_identical():
    """The all-core oracle (-fopenmp build of the same source, the bench's all-core CPU baseline) gives
    the single-thread oracle's results bit for bit: envs are independent and the step's stats are
    summed in env order after the parallel loop."""
    from oracle.oracle import Oracle
    n, T = 257, 6
    acts, obs = gen.frames(n, T, seed=9)
    P = presets.preset(FULL | presets.SMOOTH)
    one, omp = Oracle(P, n, SEED), Oracle(P, n, SEED, omp=True)
    for t in range(T):
        if t == 3:
            m = (np.arange(n) % 3 == 1).astype(np.uint8)
            one.reset(m)
            omp.reset(m)
        a = one.step(acts[t], obs[t], want_margin=True)
        b = omp.step(acts[t], obs[t], want_margin=True)
        for k in a:
            assert np.array_equal(a[k], b[k]), (t, k)
    for i in (0, 100, 256):
        ea, eb = one.env(i), omp.env(i)
        for k in ea:
            assert np.array_equal(ea[k], eb[k]), (i, k)


def test_state_import_resume_equals_uninterrupted():
    """State import (orc_set_env) pinned by the reproducibility principle (seeded
    deterministic randomization; SPEC.md:499 bit-exact resume): a second oracle that imports every env's
    state and the step index after 7 steps (one reset in between) continues exactly like the
    uninterrupted run, resets included -- so the env state holds everything the future depends on."""
    from oracle.oracle import Oracle
    n, T = 9, 14
    acts, obs = gen.frames(n, T, seed=5)
    P = presets.preset(FULL | presets.SMOOTH)
    a = Oracle(P, n, SEED)
    b = Oracle(P, n, SEED)
    for t in range(T):
        if t in (3, 10):
            m = (np.arange(n) % 2 == t % 2).astype(np.uint8)
            a.reset(m)
            if t > 7:
                b.reset(m)
        if t == 7:
            for i in range(n):
                b.set_env(i, a.env(i))
            b.step_index = a.step_index
        ra = a.step(acts[t], obs[t])
        if t >= 7:
            rb = b.step(acts[t], obs[t])
            for k in ra:
                assert np.array_equal(ra[k], rb[k]), (t, k)
    for i in range(n):
        ea, eb = a.env(i), b.env(i)
        for k in ea:
            assert np.array_equal(ea[k], eb[k]), (i, k)


def test_state_import_backlash_golden_rows_through_step():
    """The golden backlash rows (PAPER.md:102-109 hand evaluations, tests/golden/backlash_hand.txt)
    through the whole step from an imported state: with BACKLASH the only layer the action reaches
    the gate unchanged and dt_env = 10 dt_base, so the step's out_actions and slack are the row's
    values (to the fp32 rounding of the inputs and the fp64 sum of the ten substeps)."""
    from oracle.oracle import Oracle
    rows = []
    with open(os.path.join(GOLDEN, "backlash_hand.txt")) as f:
        for line in f:
            if line.strip() and not line.startswith("#"):
                lhs, rhs, tol, note = [x.strip() for x in line.split("|", 3)]
                rows.append(([float(x) for x in lhs.split()], [float(x) for x in rhs.split()], float(tol), note))
    for dt in sorted({r[0][4] for r in rows}):
        sel = [r for r in rows if r[0][4] == dt]
        n = len(sel)
        orc = Oracle(presets.preset(BACKLASH, dt_base=dt / 10), n, SEED)
        acts = np.zeros((n, 20), np.float32)
        for i, ((s, a, dn, dp, _), _, _, _) in enumerate(sel):
            e = orc.env(i)
            e["slack"][0], e["dneg"][0], e["dpos"][0] = s, dn, dp
            orc.set_env(i, e)
            acts[i, 0] = a
        obs = np.zeros((n, 26), np.float32)
        obs[:, 18] = obs[:, 22] = 1.0
        r = orc.step(acts, obs)
        for i, ((s, a, dn, dp, _), (s_new, alpha, out), tol, note) in enumerate(sel):
            got_out, got_s = r["out_actions"][i, 0], orc.env(i)["slack"][0]
            a32 = float(np.float32(a))
            assert abs(got_s - s_new) <= 1e-9 + 1e-7 * abs(s_new), (note, got_s, s_new)
            assert abs(got_out - out) <= max(tol, 1e-7 * abs(out)) + 1e-7 * abs(a32 - a), (note, got_out, out)
            if out == 0.0 and tol == 0.0:   # exact zero rows: the sign of zero is alpha * a's [Q3]
                assert got_out == 0.0 and math.copysign(1.0, got_out) == math.copysign(1.0, out), note


def test_reset_mask_semantics():
    n = 10
    acts, obs = gen.frames(n, 3, seed=8)
    orc = _oracle(FULL, n)
    for t in range(3):
        orc.step(acts[t], obs[t])
    before = [orc.env(i) for i in range(n)]
    m = np.zeros(n, dtype=np.uint8)
    m[[2, 7]] = 1
    orc.reset(m)
    r = orc.step(acts[0], obs[0])
    assert r["stats"][10] == 2
    for i in range(n):
        e = orc.env(i)
        if m[i]:
            assert e["episode"] == 1
            assert not np.array_equal(e["c_act"], before[i]["c_act"])
        else:
            assert e["episode"] == 0
            assert np.array_equal(e["c_act"], before[i]["c_act"])
    assert orc.step(acts[1], obs[1])["stats"][10] == 0


# ---- on-the-fly parameter updates ----------------------
def test_update_params_identity_and_step_vs_episode_split():
    """An update with the same parameters changes nothing (bitwise); a step-draw parameter takes
    effect at the next step (a0 with the uncorrelated/multiplicative action noise zeroed is the
    closed form clamp(a + c_act)); an episode-draw parameter only at the next
    reset (lambda range collapsed to one point: reset envs get exactly that lambda, the others
    keep theirs)."""
    n, T = 16, 6
    acts, obs = gen.frames(n, T)
    a = _oracle(FULL, n)
    b = _oracle(FULL, n)
    for t in range(T):
        if t == 3:
            b.update_params(presets.preset(FULL))
        ra, rb = a.step(acts[t], obs[t]), b.step(acts[t], obs[t])
        for k in ("out_actions", "out_obs", "out_dt", "out_force", "stats"):
            assert np.array_equal(ra[k], rb[k]), (t, k)
    a.close(), b.close()

    o = _oracle(ACT_NOISE, n)
    o.step(acts[0], obs[0])
    o.update_params(presets.preset(ACT_NOISE, act_sigma_uadd=0.0, act_sigma_mult=0.0))
    r = o.step(acts[1], obs[1])
    cact = np.array([o.env(i)["c_act"] for i in range(n)])
    assert np.array_equal(r["out_actions"], np.clip(acts[1].astype(np.float64) + cact, -1.0, 1.0))
    o.close()

    o = _oracle(TIMING, n)
    lam0 = np.array([o.env(i)["lambda"] for i in range(n)])
    o.update_params(presets.preset(TIMING, lambda_lo=5000.0, lambda_hi=5000.0))
    m = (np.arange(n) % 2).astype(np.uint8)
    o.reset(m)
    lam1 = np.array([o.env(i)["lambda"] for i in range(n)])
    assert np.array_equal(lam1[m == 0], lam0[m == 0])
    assert (lam1[m == 1] == 5000.0).all()
    o.close()


def test_update_params_force_and_dropout_thresholds():
    """Force p range collapsed to p0 after an update: reset envs carry T = floor(p0 2^32) (the
    table's midpoints all equal p0); a dropout rate of 0 after the update stops new
    initiations from the next step while running timers count down."""
    from oracle import oracle as O
    n = 64
    acts, obs = gen.frames(n, 30)
    o = _oracle(FULL, n)
    o.update_params(presets.preset(FULL, force_p_lo=0.25, force_p_hi=0.25, dropout_rate_hz=0.0))
    assert o.force_threshold(0) == o.force_threshold(65535) == O.bernoulli_threshold(0.25)
    before = [o.env(i)["t_force"] for i in range(n)]
    o.reset((np.arange(n) < 32).astype(np.uint8))
    after = [o.env(i)["t_force"] for i in range(n)]
    assert all(after[i] == O.bernoulli_threshold(0.25) for i in range(32))
    assert after[32:] == before[32:]
    inits = 0
    for t in range(30):
        inits += o.step(acts[t], obs[t])["stats"][2]
    assert inits == 0
    o.close()


# ---- §8(f) rank 2: EMA action smoothing and the per-substep backlash variant -------------------
def test_smoothing_geometric_step_response():
    """EMA with coefficient 0.3 per 80 ms step: a constant command a from a
    zero state gives a (1 - 0.7^(t+1)) at step t -- the geometric closed form; a reset returns the
    state to 0 [Q25]."""
    from workload.presets import SMOOTH
    n, T = 8, 12
    o = _oracle(SMOOTH, n)
    a = np.full((n, 20), 0.6, np.float32)
    obs = gen.frames(n, 1)[1][0]
    a64 = float(np.float32(0.6))
    for t in range(T):
        r = o.step(a, obs)
        assert np.abs(r["out_actions"] - a64 * (1.0 - 0.7 ** (t + 1))).max() < 1e-12
    o.reset((np.arange(n) < 4).astype(np.uint8))
    r = o.step(a, obs)
    assert np.abs(r["out_actions"][:4] - 0.3 * a64).max() < 1e-15
    assert np.abs(r["out_actions"][4:] - a64 * (1.0 - 0.7 ** (T + 1))).max() < 1e-12
    o.close()


def test_substep_backlash_hand_computed_and_consistent():
    """Per-substep backlash [Q26] with TIMING off (every dt_k = 8 ms), delta+1 = 4, a = 0.5 from
    s = 0: the slack climbs 0.016 per substep (0.5 * 4 * 0.008), the gate stays closed (alpha = 0,
    output 0) until the start-of-substep slack sits on the rail +1, then passes a exactly
    (PAPER.md:102-109).  Without rail contact the 10 substep updates end where the one per-step
    update with dt_env = sum dt_k ends (linearity), and out_actions = the last substep."""
    from workload.presets import SUBSTEP_BACKLASH
    n = 4
    kw = dict(delta_cal_pos=[4.0] * 20, delta_cal_neg=[4.0] * 20, delta_jitter_std=0.0)
    o = _oracle(BACKLASH | SUBSTEP_BACKLASH, n, **kw)
    a = np.full((n, 20), 0.5, np.float32)
    obs = gen.frames(n, 1)[1][0]
    outs = []
    for t in range(8):
        r = o.step(a, obs, want_sub=True)
        assert np.array_equal(r["out_actions"], r["out_actions_sub"][:, -1])
        outs.append(r["out_actions_sub"][0, :, 0])
    sub = np.concatenate(outs)     # 80 substeps of actuator 0
    k_rail = int(np.ceil(1.0 / 0.016 - 1e-9))   # the update that reaches +1 (63rd)
    assert (np.abs(sub[:k_rail]) < 1e-9).all()       # closed (alpha 0, or eps-sized on the rail hit)
    assert (sub[k_rail:] == 0.5).all()               # open: s == sgn(a)
    s_final = o.env(0)["slack"][0]
    assert s_final == 1.0
    # linearity: away from the rails, substep and per-step slack agree
    p = _oracle(BACKLASH | SUBSTEP_BACKLASH | TIMING, n, **kw)
    q = _oracle(BACKLASH | TIMING, n, **kw)
    a2 = np.full((n, 20), 0.2, np.float32)
    for t in range(3):
        p.step(a2, obs)
        q.step(a2, obs)
        sp = np.array([p.env(i)["slack"] for i in range(n)])
        sq = np.array([q.env(i)["slack"] for i in range(n)])
        assert np.abs(sp - sq).max() < 1e-12 and np.abs(sq).max() < 1.0
    o.close(), p.close(), q.close()


def test_substep_backlash_invariants():
    """Every substep keeps the slack in [-1, 1] and |out| <= |a_n| with out a_n >= 0, on the FULL
    layer set with resets (PAPER.md:102-109 invariants)."""
    from workload.presets import SMOOTH, SUBSTEP_BACKLASH
    n, T = 64, 20
    acts, obs = gen.frames(n, T)
    o = _oracle(FULL | SMOOTH | SUBSTEP_BACKLASH, n)
    for t in range(T):
        r = o.step(acts[t], obs[t], want_sub=True)
        s = np.array([o.env(i)["slack"] for i in range(n)])
        assert np.abs(s).max() <= 1.0
        sub = r["out_actions_sub"]
        assert np.abs(sub).max() <= 1.0
        assert np.array_equal(sub[:, -1], r["out_actions"])
        if t == 10:
            o.reset((np.arange(n) % 2).astype(np.uint8))
    o.close()
