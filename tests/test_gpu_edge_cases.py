"""GPU parity at the boundaries the paper's formulas have, driven through the C-ABI from crafted
states (dr_state_import on the GPU, Oracle.set_env on the oracle):

* the backlash model on every row of tests/golden/backlash_hand.txt -- sgn(+-0),
  a = -0.0, tiny actions against a rail, rail hits whose alpha is eps-sized (kept in fp32) or below
  fp32 resolution (exactly 0 in fp32, Q5), SPEC.md:204-206's worked examples;
* the occlusion distance rule (strict "closer than r") at the exact
  dyadic boundary D = r^2 and one fp32 ulp inside it, which forces the kernels' exact-fp64 fallback;
* windowed re-sync (SURVEY.md §8(c).4 mode M2) on BASELINE config 2: every W steps the oracle imports
  the GPU's exported state, so fp32 slack drift is bounded and the knife-edge band can be tight.

Every test runs on both step kernels (DR_STEP_MODE, read at dr_init)."""
import math
import os

import numpy as np
import pytest

from parity import (KnifeTracker, assert_close, compare_obs, compare_records, compare_stats, oracle_env_from_gpu,
                    state_array_from_numpy)
from workload import gen, presets
from workload.presets import BACKLASH, CFG2, OCCLUSION

pytestmark = pytest.mark.gpu
SEED = presets.SEED_DR
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.fixture(params=["throughput", "latency"], autouse=True)
def step_mode(request, monkeypatch):
    monkeypatch.setenv("DR_STEP_MODE", request.param)
    return request.param


@pytest.fixture(autouse=True)
def _finalize_leaked_context():
    yield
    from paper_1906_11633_b200 import dr
    dr.load().dr_finalize()


def _backlash_rows():
    rows = []
    with open(os.path.join(GOLDEN, "backlash_hand.txt")) as f:
        for line in f:
            if not line.strip() or line.startswith("#"):
                continue
            lhs, rhs, tol, note = [x.strip() for x in line.split("|", 3)]
            rows.append(([float(x) for x in lhs.split()], [float(x) for x in rhs.split()], float(tol), note))
    return rows


def _neutral_obs(n):
    o = np.zeros((n, 26), np.float32)
    o[:, 18] = 1.0   # object quaternion (w, x, y, z) = identity
    o[:, 22] = 1.0   # goal quaternion
    return o


@pytest.mark.parametrize("dt", [0.08, 0.1])
def test_backlash_golden_rows_through_kernel(torch_cuda, dt):
    """Each golden row (s, a, delta-1, delta+1, dt) is one actuator of a crafted state: BACKLASH is the
    only layer, so a reaches the gate unchanged and dt_env = 10 x dt_base.  GPU vs oracle on the same
    imported state: outputs and slack within 1e-6, the sign of a zero output, alpha = 1 decisions and
    the rail-hit / gate counters exact.  GPU vs the golden hand values: outputs within the fp32
    quantisation of the row's inputs; rail hits with |sgn - s| < 2^-15 keep their eps-sized alpha
    (relative 1e-5); wider ones give alpha = 0 exactly in fp32 (Q5)."""
    torch = torch_cuda
    from oracle.oracle import Oracle
    from paper_1906_11633_b200 import DRContext, dr
    rows = [r for r in _backlash_rows() if r[0][4] == dt]
    assert rows
    n = 3   # 60 actuator slots: the rows first, then neutral fillers (s = 0, a = 0)
    P = presets.preset(BACKLASH, dt_base=dt / 10)
    ctx = DRContext(P, n, SEED)
    orc = Oracle(P, n, SEED)
    try:
        st = dr.dr_state_export()
        G = dr.states_to_numpy(st)
        acts = np.zeros((n, 20), np.float32)
        G["flags"][:] = 0
        G["prev"][:] = 0.0
        G["slack"][:] = 0.0
        G["dneg"][:] = 1.0
        G["dpos"][:] = 1.0
        for k, ((s, a, dn, dp, _), _, _, _) in enumerate(rows):
            e, j = divmod(k, 20)
            G["slack"][e, j], G["dneg"][e, j], G["dpos"][e, j] = s, dn, dp
            acts[e, j] = a
        state_array_from_numpy(st, G)
        dr.dr_state_import(st)
        G = dr.states_to_numpy(dr.dr_state_export())   # what the GPU holds (fp32)
        for i in range(n):
            orc.set_env(i, oracle_env_from_gpu(G, i, orc))
        obs = _neutral_obs(n)
        ctx.step(torch.from_numpy(acts).cuda(), torch.from_numpy(obs).cuda())
        r = orc.step(acts, obs, want_margin=True)
        torch.cuda.synchronize()
        out_g = ctx.out_actions.cpu().numpy().astype(np.float64)
        out_o = r["out_actions"]
        G1 = dr.states_to_numpy(dr.dr_state_export())
        s_g = G1["slack"].astype(np.float64)
        s_o = np.array([orc.env(i)["slack"] for i in range(n)])
        # GPU vs oracle, element by element (no knife-edge excusal: every margin is far from tau)
        assert_close("out_actions", out_g, out_o, 1.0)
        assert_close("slack", s_g, s_o, 1.0)
        assert np.array_equal(np.signbit(out_g[out_o == 0.0]), np.signbit(out_o[out_o == 0.0])), "sign of zero"
        assert np.array_equal(out_g == acts, out_o == acts.astype(np.float64)), "alpha = 1 decisions"
        compare_stats(ctx.last_stats(), r["stats"], n)
        # GPU vs the golden hand values
        for k, ((s, a, dn, dp, _), (s_new, alpha, out), tol, note) in enumerate(rows):
            e, j = divmod(k, 20)
            assert abs(s_g[e, j] - s_new) <= 1e-6, (note, s_g[e, j], s_new)
            assert abs(out_g[e, j] - out) <= 1e-6, (note, out_g[e, j], out)
            if out == 0.0 and tol == 0.0:   # exact zero rows: the sign of zero is alpha * a's [Q3]
                assert out_g[e, j] == 0.0 and math.copysign(1.0, out_g[e, j]) == math.copysign(1.0, out), note
            if alpha == 1.0:
                assert out_g[e, j] == np.float32(a), note
            elif 0.0 < alpha < 1.0:
                num = abs(math.copysign(1.0, a) - np.float32(s))
                if num < 2.0 ** -15:   # eps is above half an ulp of num: fp32 keeps the eps-sized alpha
                    assert abs(out_g[e, j] / np.float32(a) - alpha) <= 1e-5 * alpha, (note, out_g[e, j], alpha)
                else:                  # eps below fp32 resolution at |sgn - s|: alpha = 0 exactly [Q5]
                    assert out_g[e, j] == 0.0, (note, out_g[e, j])
                assert abs(s_g[e, j]) == 1.0, note
        # the filler actuators: a = 0 at s = 0 -> out 0, slack 0
        k0 = len(rows)
        assert (out_g.ravel()[k0:] == 0.0).all() and (s_g.ravel()[k0:] == 0.0).all()
    finally:
        ctx.close()
        orc.close()


def _occlusion_cases():
    """(name, tips [5][3], obj [3], expected occluded-tip bits) with r = 5 * 2^-8 m: tip pairs at a
    (3, 4, 5) triangle scaled by 2^-8 are exactly r apart (D = r^2: not occluded, strict <)."""
    far = [[0.1, 0.0, 0.0], [0.2, 0.0, 0.0], [0.3, 0.0, 0.0]]
    u = 2.0 ** -8
    down = lambda x: float(np.nextafter(np.float32(x), np.float32(0)))  # noqa: E731  one fp32 ulp towards 0
    cases = [
        ("tip pair at D = r^2", [[0, 0, 0], [3 * u, 4 * u, 0]] + far, [0.5, 0.5, 0.5], 0b00000),
        ("tip pair one ulp inside", [[0, 0, 0], [3 * u, down(4 * u), 0]] + far, [0.5, 0.5, 0.5], 0b00011),
        ("tip-object at D = r^2", [[0, 0, 0], [0.05, 0, 0]] + far, [0, 0, 5 * u], 0b00000),
        ("tip-object one ulp inside", [[0, 0, 0], [0.05, 0, 0]] + far, [0, 0, down(5 * u)], 0b00001),
        ("tip pair one ulp outside", [[0, 0, 0], [3 * u, float(np.nextafter(np.float32(4 * u), np.float32(1))), 0]]
         + far, [0.5, 0.5, 0.5], 0b00000),
        ("offset pair at D = r^2", [[0.75, 0.5, 0.25], [0.75 + 3 * u, 0.5 + 4 * u, 0.25]] + far, [0.5, 0.5, 0.5], 0b00000),
        ("offset pair one ulp inside", [[0.75, 0.5, 0.25], [0.75 + 3 * u, down(0.5 + 4 * u), 0.25]] + far,
         [0.5, 0.5, 0.5], 0b00011),
        ("three tips, one inside pair", [[0, 0, 0], [3 * u, 4 * u, 0], [0, -down(5 * u), 0], [0.3, 0, 0], [0.4, 0, 0]],
         [0.5, 0.5, 0.5], 0b00101),
    ]
    return cases


def test_occlusion_exact_dyadic_boundary_through_kernel(torch_cuda):
    """OCCLUSION alone (the distance rule, r = 5 x 2^-8 m exactly): step 0 places the tips far apart
    (a reading now exists), step 1 the boundary configurations.  A tip is occluded iff another tip or
    the object is strictly closer than r in the exactly rounded fp64 distance:
    D = r^2 is not occluded, one fp32 ulp closer is.  Occluded tips repeat their step-0 reading bit for
    bit; the decisions, the held readings and the occluded / held counters equal the oracle's and the
    hand-derived bits."""
    torch = torch_cuda
    from oracle.oracle import Oracle
    from paper_1906_11633_b200 import DRContext
    cases = _occlusion_cases()
    n = len(cases)
    r = 5.0 * 2.0 ** -8
    P = presets.preset(OCCLUSION, occl_dist=r)
    ctx = DRContext(P, n, SEED)
    orc = Oracle(P, n, SEED)
    try:
        obs0 = _neutral_obs(n)
        for e in range(n):
            obs0[e, 0:15] = np.arange(15, dtype=np.float32) * 0.1 + e   # far apart, no occlusion
            obs0[e, 15:18] = [9.0, 9.0, 9.0]
        obs1 = _neutral_obs(n)
        for e, (_, tips, obj, _) in enumerate(cases):
            obs1[e, 0:15] = np.asarray(tips, np.float32).ravel()
            obs1[e, 15:18] = np.asarray(obj, np.float32)
        acts = np.zeros((n, 20), np.float32)
        outs = []
        for t, obs in enumerate((obs0, obs1)):
            ctx.step(torch.from_numpy(acts).cuda(), torch.from_numpy(obs).cuda())
            ro = orc.step(acts, obs)
            torch.cuda.synchronize()
            og = ctx.out_obs.cpu().numpy()
            assert np.array_equal(og[:, 4:22].astype(np.float64), ro["out_obs"][:, 4:22]), f"tips/object t={t}"
            compare_stats(ctx.last_stats(), ro["stats"], n, t=t)
            outs.append(og)
        held_g = np.all(outs[1][:, 4:19].reshape(n, 5, 3) == outs[0][:, 4:19].reshape(n, 5, 3), axis=2)
        raw1 = obs1[:, 0:15].reshape(n, 5, 3)
        for e, (name, _, _, bits) in enumerate(cases):
            for i in range(5):
                occ = bool((bits >> i) & 1)
                if occ:
                    assert held_g[e, i], (name, i)
                else:
                    assert np.array_equal(outs[1][e, 4 + 3 * i:7 + 3 * i], raw1[e, i]), (name, i)
        expected_total = sum(bin(c[3]).count("1") for c in cases)
        s = ctx.last_stats()
        assert s[4] == expected_total and s[5] == expected_total   # occluded, held
    finally:
        ctx.close()
        orc.close()


W_RESYNC = 50
KNIFE_TAU_M2 = 1e-6


def test_config2_windowed_resync_m2(torch_cuda):
    """SURVEY.md §8(c).4 mode M2 on BASELINE config 2 (4,096 envs, backlash + action/obs noise):
    1,000 steps on all envs; every W = 50 steps the oracle imports the GPU's exported state of 1,024
    sampled envs, so fp32 slack drift stays bounded and the checker holds slack to 1e-6 with a
    knife-edge band of tau = 1e-6.  Bounds asserted: knife-edge events <= 1e-4 per
    actuator-step, excused output mismatches <= the events."""
    torch = torch_cuda
    from oracle.oracle import Oracle
    from paper_1906_11633_b200 import DRContext, dr
    n, T = 4096, 1000
    rng = np.random.default_rng(22)
    sample = np.sort(rng.choice(n, 1024, replace=False))
    P = presets.preset(CFG2)
    acts, obs = gen.frames(n, 16)
    A = [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in acts]
    O = [torch.from_numpy(np.ascontiguousarray(o)).cuda() for o in obs]
    ctx = DRContext(P, n, SEED)
    orc = Oracle(P, len(sample), SEED, gids=sample)
    knife = KnifeTracker(len(sample), tau=KNIFE_TAU_M2)
    max_slack_err = 0.0
    try:
        for t in range(T):
            if t % W_RESYNC == 0:
                G = dr.states_to_numpy(dr.dr_state_export())
                for i, g in enumerate(sample):
                    orc.set_env(i, oracle_env_from_gpu(G, g, orc))
                knife.excused[:] = False
            f = t % 16
            ctx.step(A[f], O[f])
            r = orc.step(acts[f][sample], obs[f][sample], want_margin=True)
            torch.cuda.synchronize()
            knife.update_before_compare(r["margin"])
            knife.compare_actions(ctx.out_actions.cpu().numpy()[sample], r["out_actions"], t)
            compare_obs(ctx.out_obs.cpu().numpy()[sample], r["out_obs"], t)
            assert_close(f"out_dt t={t}", ctx.out_dt.cpu().numpy()[sample], r["out_dt"], 0.008)
            if t % 10 == 9:
                G = dr.states_to_numpy(dr.dr_state_export())
                Gs = {k: v[sample] for k, v in G.items()}
                Os = [orc.env(i) for i in range(len(sample))]
                knife.resync(Gs["slack"].astype(np.float64), np.array([o["slack"] for o in Os]))
                err = np.abs(Gs["slack"].astype(np.float64) - np.array([o["slack"] for o in Os]))
                max_slack_err = max(max_slack_err, float(np.where(knife.excused, 0.0, err).max()))
                compare_records(Gs, Os, knife=None, strict_state=False, mask=CFG2)
                assert_close(f"slack t={t}", Gs["slack"], np.array([o["slack"] for o in Os]), 1.0,
                             mask=~knife.excused)
        steps = T * len(sample) * 20
        print(f"M2 config 2: knife events {knife.events} ({knife.events / steps:.2e} per actuator-step), "
              f"excused mismatches {knife.excused_mismatches}, max slack |err| {max_slack_err:.3g}")
        assert knife.events <= 1e-4 * steps
        assert knife.excused_mismatches <= knife.events
    finally:
        ctx.close()
        orc.close()
