"""GPU parity: the CUDA path (through the C-ABI, libdr.so) against the fp64 oracle on the same
seeded inputs, element by element (tests/parity.py states the contract)."""
import math

import numpy as np
import pytest

from parity import (KnifeTracker, assert_close, compare_obs, compare_records, compare_stats)
from workload import gen, presets
from workload.presets import (ACT_NOISE, BACKLASH, CFG2, DELAY, DROPOUT, FORCE, FULL, OBS_NOISE,
                              OCCLUSION, PHYS, SMOOTH, SUBSTEP_BACKLASH, TIMING)

pytestmark = pytest.mark.gpu
SEED = presets.SEED_DR


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.fixture(params=["throughput", "latency"], autouse=True)
def step_mode(request, monkeypatch):
    """Every parity test runs on both step kernels (DR_STEP_MODE, read at dr_init): the throughput
    kernel (persistent tiles, one thread per env) and the latency kernel (8 warps per 32 envs)."""
    monkeypatch.setenv("DR_STEP_MODE", request.param)
    return request.param


@pytest.fixture(autouse=True)
def _finalize_leaked_context():
    """A failing test must not leave its context behind (dr_init would return DR_EALREADY)."""
    yield
    from paper_1906_11633_b200 import dr
    dr.load().dr_finalize()   # DR_ENOTINIT when nothing leaked


def _ctx(preset, n, seed=SEED, **kw):
    from paper_1906_11633_b200 import DRContext
    return DRContext(preset, n, seed, **kw)


def _frames_cuda(torch, arr):
    """One separately allocated (256-B aligned) device tensor per frame: dr_step requires
    16-byte aligned rows."""
    return [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in arr]


def _oracle(preset, gids, seed=SEED):
    from oracle.oracle import Oracle
    return Oracle(preset, len(gids), seed, gids=np.asarray(gids, dtype=np.int64))


def run_pair(torch, mask, n_env, T, n_frames=8, resets=None, sample=None, state_every=1,
             stats=True, seed=SEED, frame_seed=presets.SEED_WORKLOAD, updates=None, occl_masks=None, **kw):
    """Run the GPU on all n_env envs and the oracle on `sample` (default: all); compare every
    step.  `resets`: {t: uint8 mask [n_env]} applied before step t; `updates`: {t: parameter
    overrides} swapped in with dr_update_params / orc_update_params before step t."""
    P = presets.preset(mask, **kw)
    acts, obs = gen.frames(n_env, n_frames, seed=frame_seed)
    A = _frames_cuda(torch, acts)
    O = _frames_cuda(torch, obs)
    gids = np.arange(n_env) if sample is None else np.asarray(sample)
    full = sample is None
    ctx = _ctx(P, n_env, seed)
    orc = _oracle(P, gids, seed)
    knife = KnifeTracker(len(gids))
    try:
        G = ctx.export()
        compare_records({k: v[gids] for k, v in G.items()}, [orc.env(i) for i in range(len(gids))],
                        phys_g=ctx.phys()[gids], mask=mask)
        occ_dev = occ_orc = None
        if occl_masks is not None:   # simulator occlusion bits (dr_set_occlusion_input)
            from paper_1906_11633_b200 import dr as _dr
            occ_dev = torch.zeros(n_env, dtype=torch.uint8, device="cuda")
            _dr.dr_set_occlusion_input(occ_dev, n_env)
            occ_orc = orc.set_occlusion_mask(np.zeros(len(gids), np.uint8))
        for t in range(T):
            if occl_masks is not None:
                occ_dev.copy_(torch.from_numpy(occl_masks[t]))
                occ_orc[:] = occl_masks[t][gids]
            if updates and t in updates:
                P = presets.preset(mask, **{**kw, **updates[t]})
                ctx.update_params(P)
                orc.update_params(P)
            if resets and t in resets:
                m = resets[t]
                ctx.reset(torch.from_numpy(m).cuda())
                orc.reset(m[gids])
            f = t % n_frames
            ctx.step(A[f], O[f])
            sub = bool(mask & SUBSTEP_BACKLASH)
            r = orc.step(acts[f][gids], obs[f][gids], want_margin=True, want_sub=sub)
            torch.cuda.synchronize()
            oa = ctx.out_actions.cpu().numpy()[gids]
            oo = ctx.out_obs.cpu().numpy()[gids]
            od = ctx.out_dt.cpu().numpy()[gids]
            of = ctx.out_force.cpu().numpy()[gids]
            knife.update_before_compare(r["margin"])
            knife.compare_actions(oa, r["out_actions"], t)
            if sub:
                gs = ctx.out_actions_sub.cpu().numpy()[gids]
                assert np.array_equal(gs[:, -1], oa), "out_actions == last substep"
                assert_close(f"out_actions_sub t={t}", gs, r["out_actions_sub"], 1.0,
                             mask=~np.broadcast_to(knife.excused[:, None, :], gs.shape))
            compare_obs(oo, r["out_obs"], t)
            assert_close(f"out_dt t={t}", od, r["out_dt"], 0.008)
            mass = np.array([orc.env(i)["mass"] for i in range(len(gids))]) if (mask & FORCE) else np.ones(len(gids))
            assert_close(f"out_force t={t}", of, r["out_force"], mass[:, None] * P["force_accel_std"])
            if full and stats:
                compare_stats(ctx.last_stats(), r["stats"], n_env, knife.events, t)
            if state_every and (t % state_every == 0 or t == T - 1):
                G = ctx.export()
                compare_records({k: v[gids] for k, v in G.items()}, [orc.env(i) for i in range(len(gids))],
                                knife=knife, mask=mask)
        # the knife-edge accounting is bounded, not only counted: events are rare
        # (measured ~2e-5 per actuator-step at tau = 1e-5 on config 2) and an excused actuator
        # mismatches at most until its slack re-syncs
        act_steps = T * len(gids) * 20
        assert knife.events <= max(4, 1e-4 * act_steps), ("knife events", knife.events, act_steps)
        assert knife.excused_mismatches <= 16 * max(knife.events, 1), ("excused mismatches", knife.excused_mismatches)
        return knife
    finally:
        ctx.close()
        orc.close()


def test_debug_philox_words_bit_exact(torch_cuda):
    """RNG integer streams are bit-exact: the device Philox words the kernels draw equal the
    oracle's from-spec Philox for every env, in both the step and the reset domain."""
    torch = torch_cuda
    from oracle import oracle as O
    from paper_1906_11633_b200 import dr
    n = 257
    seed = 0x0123456789ABCDEF
    ctx = _ctx(presets.preset(FULL), n, seed=seed, env_offset=1000, n_env_global=5000)
    try:
        out = torch.empty(n, 4, dtype=torch.int32, device="cuda")
        for dom, ch, blk in [(0, 0x01, 0), (7, 0x02, 3), (123456, 0x08, 1), (2, 0x101, 63), (0xFFFFFFFF, 0x10C, 5)]:
            dr.dr_debug_philox(dom, ch, blk, out)
            torch.cuda.synchronize()
            g = out.cpu().numpy().view(np.uint32)
            for e in range(0, n, 16):
                ref = O.philox((1000 + e, dom, ch, blk), (seed & 0xFFFFFFFF, seed >> 32))
                assert tuple(int(x) for x in g[e]) == ref, (dom, ch, blk, e)
    finally:
        ctx.close()


def test_reset_records_and_phys(torch_cuda):
    """Episode-0 records + physical parameters for 2000 envs (all layers, PHYS on)."""
    torch = torch_cuda
    P = presets.preset(FULL)
    n = 2000
    ctx = _ctx(P, n)
    orc = _oracle(P, np.arange(n))
    try:
        compare_records(ctx.export(), [orc.env(i) for i in range(n)], phys_g=ctx.phys())
        # masked reset: episode counters + resampled records only where masked
        m = (np.arange(n) % 7 == 3).astype(np.uint8)
        ctx.reset(torch.from_numpy(m).cuda())
        orc.reset(m)
        torch.cuda.synchronize()
        G = ctx.export()
        compare_records(G, [orc.env(i) for i in range(n)], phys_g=ctx.phys())
        assert (G["episode"] == m).all()
    finally:
        ctx.close()


@pytest.mark.parametrize("n", [1, 200, 2049])
def test_reset_kernel_densities(torch_cuda, n):
    """The reset kernel (thread-per-env record in whole sectors + warp-per-env physics rows) gives
    the oracle's episode records and physics rows -- full init, then masked resets at two densities
    (a lone env, every 3rd env) -- and the steps after them agree."""
    torch = torch_cuda
    P = presets.preset(FULL)
    ctx = _ctx(P, n)
    orc = _oracle(P, np.arange(n))
    try:
        compare_records(ctx.export(), [orc.env(i) for i in range(n)], phys_g=ctx.phys())
        for m in [(np.arange(n) == n - 1).astype(np.uint8), (np.arange(n) % 3 == 0).astype(np.uint8)]:
            ctx.reset(torch.from_numpy(m).cuda())
            orc.reset(m)
            torch.cuda.synchronize()
            compare_records(ctx.export(), [orc.env(i) for i in range(n)], phys_g=ctx.phys())
    finally:
        ctx.close()
    run_pair(torch_cuda, FULL, n, 6, n_frames=6, resets={3: (np.arange(n) % 4 == 1).astype(np.uint8)})


@pytest.mark.parametrize("mask", [CFG2, PHYS, 0, FULL & ~PHYS])
def test_reset_kernel_layer_sets(torch_cuda, mask):
    """The reset kernel with PHYS off (physics rows = the descriptor bases, no draws) or alone:
    records and physics rows equal the oracle's after init and after a masked reset."""
    torch = torch_cuda
    n = 300
    P = presets.preset(mask)
    ctx = _ctx(P, n)
    orc = _oracle(P, np.arange(n))
    try:
        compare_records(ctx.export(), [orc.env(i) for i in range(n)], phys_g=ctx.phys())
        m = (np.arange(n) % 7 == 2).astype(np.uint8)
        ctx.reset(torch.from_numpy(m).cuda())
        orc.reset(m)
        torch.cuda.synchronize()
        compare_records(ctx.export(), [orc.env(i) for i in range(n)], phys_g=ctx.phys())
    finally:
        ctx.close()


def test_reset_mask_patterns(torch_cuda):
    """The reset's scan schedule (CTA c owns the interleaved 32-env mask chunks c, c + G, ...): at
    20,011 envs (626 chunks over the 592-CTA grid: some CTAs own two chunks, the last one a ragged
    tail) a contiguous block, the first env alone, every other env and an explicit all-ones mask
    each give the oracle's records and physics rows for every env, as does dr_reset(NULL) (every
    env), and the next step's stats slot 10 counts exactly the resets."""
    torch = torch_cuda
    P = presets.preset(FULL)
    n = 20011
    ctx = _ctx(P, n)
    orc = _oracle(P, np.arange(n))
    acts, obs = gen.frames(n, 1)
    A, O = torch.from_numpy(acts[0]).cuda(), torch.from_numpy(obs[0]).cuda()
    e = np.arange(n)
    masks = [((e >= 9000) & (e < 17011)), e == 0, e % 2 == 1, np.ones(n, dtype=bool), None]
    try:
        for m in masks:
            dev = None if m is None else torch.from_numpy(m.astype(np.uint8)).cuda()   # None: dr_reset(NULL) = all
            m = np.ones(n, np.uint8) if m is None else m.astype(np.uint8)
            ctx.reset(dev)
            orc.reset(m)
            torch.cuda.synchronize()
            compare_records(ctx.export(), [orc.env(i) for i in range(n)], phys_g=ctx.phys(), strict_state=False)
            ctx.step(A, O)
            orc.step(acts[0], obs[0])
            assert ctx.last_stats()[10] == int(m.sum())
        # two resets back to back (the second reads the episode counters the first just wrote, so it
        # must not scan early), then a step: counts and records as the oracle's
        m1, m2 = (e % 3 == 0).astype(np.uint8), (e % 5 == 0).astype(np.uint8)
        ctx.reset(torch.from_numpy(m1).cuda())
        ctx.reset(torch.from_numpy(m2).cuda())
        orc.reset(m1)
        orc.reset(m2)
        torch.cuda.synchronize()
        compare_records(ctx.export(), [orc.env(i) for i in range(n)], phys_g=ctx.phys(), strict_state=False)
        ctx.step(A, O)
        assert ctx.last_stats()[10] == int(m1.sum() + m2.sum())
    finally:
        ctx.close()
        orc.close()


def test_config1_free_running(torch_cuda):
    """BASELINE config 1: 4 envs x 50 steps, all layers, fixed seed; every output, state and
    stats slot each step (M1 free-running), with resets mid-run."""
    r = {20: np.array([0, 1, 0, 0], np.uint8), 35: np.ones(4, np.uint8)}
    k = run_pair(torch_cuda, FULL, 4, 50, n_frames=50, resets=r)
    assert k.events == 0


@pytest.mark.parametrize("mask", [0, TIMING, ACT_NOISE, DELAY, BACKLASH | TIMING, OBS_NOISE, DROPOUT,
                                  OCCLUSION, FORCE, PHYS, DROPOUT | OCCLUSION | OBS_NOISE, CFG2,
                                  FULL & ~TIMING, FULL & ~PHYS])
def test_layer_subsets(torch_cuda, mask):
    run_pair(torch_cuda, mask, 200, 25, n_frames=25, resets={12: (np.arange(200) % 5 == 0).astype(np.uint8)})


@pytest.mark.parametrize("n", [1, 3, 127, 129, 1000])
def test_ragged_sizes(torch_cuda, n):
    """Tile tails (TILE = 128), single env, odd counts: scalar staging paths."""
    run_pair(torch_cuda, FULL, n, 12, n_frames=12, resets={6: (np.arange(n) % 2 == 0).astype(np.uint8)})


@pytest.mark.parametrize("mask,n", [(FULL | SMOOTH, 200), (FULL | SMOOTH | SUBSTEP_BACKLASH, 200),
                                    (CFG2 | SUBSTEP_BACKLASH, 131), (BACKLASH | SUBSTEP_BACKLASH, 70),
                                    (SMOOTH | DELAY, 33)])
def test_smoothing_and_substep_backlash(torch_cuda, mask, n):
    """EMA action smoothing and the per-substep backlash
    variant -- every output incl. the [n][10][20] substep actions, state incl.
    the EMA, and stats, with resets mid-run."""
    run_pair(torch_cuda, mask, n, 20, n_frames=20, resets={9: (np.arange(n) % 3 == 1).astype(np.uint8)})


@pytest.mark.parametrize("mask", [FULL, FULL & ~DROPOUT, CFG2 | OCCLUSION, OCCLUSION])
def test_simulator_occlusion_input(torch_cuda, mask):
    """the simulator's per-marker occlusion bits replace the distance rule
    (PAPER.md:66 collision sites) -- random bits every step, hold decisions bit-exact."""
    n, T = 300, 16
    rng = np.random.default_rng(7)
    masks = [(rng.random((n, 5)) < 0.2).astype(np.uint8) @ (1 << np.arange(5, dtype=np.uint8)) for _ in range(T)]
    masks = [m.astype(np.uint8) for m in masks]
    run_pair(torch_cuda, mask, n, T, n_frames=T, occl_masks=masks,
             resets={8: (np.arange(n) % 4 == 0).astype(np.uint8)})


@pytest.mark.parametrize("over", [
    # saturated probabilities, maximal hold, every marker occluded, exact-threshold force
    dict(delay_prob=1.0, dropout_rate_hz=1e4, dropout_hold_steps=15, occl_dist=0.2, force_p_lo=1.0, force_p_hi=1.0),
    # nothing fires: zero probabilities / radii, zero hold
    dict(delay_prob=0.0, dropout_rate_hz=0.0, dropout_hold_steps=0, occl_dist=0.0, force_p_lo=1e-9, force_p_hi=1e-9),
    # backlash widths near 0 (the jitter clamps ~31 % of them at 0, Q7), heavy action noise (clamps),
    # a point lambda, zero obs noise
    dict(delta_cal_neg=[0.05] * 20, delta_cal_pos=[0.05] * 20, act_sigma_uadd=2.0, act_sigma_mult=1.0,
         act_sigma_cadd=0.5, lambda_lo=3000.0, lambda_hi=3000.0, tip_uncorr=0.0, obj_uncorr=0.0, rot_uncorr=0.0,
         tip_corr=0.0, obj_corr=0.0, rot_corr=0.0, tip_marker=0.0, base_marker=0.0),
    # huge backlash widths (every step hits a rail), decay 1 (force never decays), mass-free physics off
    dict(delta_cal_neg=[50.0] * 20, delta_cal_pos=[80.0] * 20, force_decay_per_step=1.0, force_accel_std=3.0),
])
def test_extreme_parameters(torch_cuda, over):
    """Degenerate and saturated parameter settings of every randomizer (SPEC.md:127 ranges' ends):
    same parity contract, with resets mid-run."""
    n = 160
    run_pair(torch_cuda, FULL, n, 18, n_frames=18, resets={9: (np.arange(n) % 3 == 0).astype(np.uint8)}, **over)


def test_update_params_mid_run(torch_cuda):
    """On-the-fly parameter updates: step-draw parameters change from the next
    step, episode-draw parameters at each env's next reset -- identically on both sides."""
    n = 300
    upd = {
        5: dict(act_sigma_uadd=0.2, act_sigma_mult=0.05, tip_uncorr=4e-3, obj_uncorr=3e-3, rot_uncorr=0.2,
                dropout_rate_hz=2.0, dropout_hold_steps=5, occl_dist=0.03, force_accel_std=2.0,
                force_decay_per_step=0.9, force_p_lo=0.05, force_p_hi=0.5, lambda_lo=2000.0, lambda_hi=3000.0,
                delay_prob=0.9, act_sigma_cadd=0.01, delta_jitter_std=0.3, dt_base=0.01),
        14: dict(act_sigma_uadd=0.0, act_sigma_mult=0.0, force_p_lo=1e-3, force_p_hi=1e-3),
    }
    resets = {9: (np.arange(n) % 3 == 0).astype(np.uint8), 16: (np.arange(n) % 2 == 1).astype(np.uint8)}
    run_pair(torch_cuda, FULL, n, 22, n_frames=22, resets=resets, updates=upd)


def test_update_params_rejects_shape_changes(torch_cuda):
    from paper_1906_11633_b200 import dr
    ctx = _ctx(presets.preset(CFG2), 64)
    try:
        with pytest.raises(dr.DRError, match="layer_mask"):
            ctx.update_params(presets.preset(FULL))
        with pytest.raises(dr.DRError, match="n_phys"):
            ctx.update_params(presets.preset(CFG2, n_phys=8))
        with pytest.raises(dr.DRError, match="delay_prob"):
            ctx.update_params(presets.preset(CFG2, delay_prob=1.5))
    finally:
        ctx.close()


def test_config2_cfg2_4096(torch_cuda):
    """BASELINE config 2 shape (4,096 envs, backlash + action/obs noise): 100 steps on all envs,
    then 1,000 steps on a 64-env sample (the full run length), knife-edge aware."""
    k = run_pair(torch_cuda, CFG2, 4096, 100, n_frames=16, state_every=10)
    print("config2 knife-edges (100 steps x 4096 envs):", k.events, "excused mismatches:", k.excused_mismatches)
    assert k.events <= 1e-4 * 100 * 4096 * 20 and k.excused_mismatches <= k.events
    rng = np.random.default_rng(2)
    sample = np.sort(rng.choice(4096, 64, replace=False))
    k = run_pair(torch_cuda, CFG2, 4096, 1000, n_frames=16, sample=sample, state_every=50)
    print("config2 knife-edges (1000 steps x 64 envs):", k.events)


def test_config3_full_65536_sampled(torch_cuda):
    """BASELINE config 3 (65,536 envs, full pipeline incl. dropout/occlusion hold and forces) in
    the launch configuration bench.py times, compared on 256 sampled envs, with 10 % Bernoulli
    resets every 10 steps."""
    n = 65536
    rng = np.random.default_rng(3)
    sample = np.sort(np.concatenate([[0, 1, 127, 128, n - 1], rng.choice(n, 251, replace=False)]))
    resets = {t: gen.reset_mask_bernoulli(rng, n, 0.1) for t in (10, 20)}
    run_pair(torch_cuda, FULL, n, 30, n_frames=8, sample=sample, resets=resets, state_every=10)


def test_config5_reset_stress_sampled(torch_cuda):
    """BASELINE config 5 pattern (env e resets when (e + t) mod 10 == 0) at 262,144 envs,
    sampled comparison of records and outputs."""
    n = 1 << 18
    rng = np.random.default_rng(5)
    sample = np.sort(rng.choice(n, 128, replace=False))
    resets = {t: gen.reset_mask_ring(n, t) for t in range(1, 6)}
    run_pair(torch_cuda, FULL, n, 6, n_frames=4, sample=sample, resets=resets, state_every=1)


def test_config4_config5_full_size_sampled_1M(torch_cuda):
    """BASELINE configs 4 and 5 at their full size (1,048,576 envs, all layers) in bench.py's launch
    configuration (persistent grid of 592 CTAs, chained steps, a 4-frame input ring): 10 steps with
    config 5's resets before every step ((e + t) mod 10 == 0, so every env resets once), then 2
    more without; 96 sampled envs (incl. the first and last tiles) compared with the oracle every
    step, records and state every 4 steps."""
    n = 1 << 20
    rng = np.random.default_rng(45)
    sample = np.sort(np.unique(np.concatenate([[0, 1, 127, 128, n - 129, n - 2, n - 1],
                                                rng.choice(n, 89, replace=False)])))
    resets = {t: gen.reset_mask_ring(n, t) for t in range(10)}
    run_pair(torch_cuda, FULL, n, 12, n_frames=4, sample=sample, resets=resets, state_every=4, stats=False)


def _run_outputs(torch, P, n, T, seed=SEED, env_offset=0, n_env_global=0, rows=None, resets=None, graph=False):
    acts, obs = gen.frames(n_env_global or n, 6)
    lo = env_offset
    A = _frames_cuda(torch, acts[:, lo:lo + n])
    O = _frames_cuda(torch, obs[:, lo:lo + n])
    ctx = _ctx(P, n, seed, env_offset=env_offset, n_env_global=n_env_global)
    outs = []
    try:
        for t in range(T):
            if resets and t in resets:
                ctx.reset(torch.from_numpy(resets[t][lo:lo + n].copy()).cuda())
            ctx.step(A[t % 6], O[t % 6])
            outs.append([x.clone() for x in (ctx.out_actions, ctx.out_obs, ctx.out_dt, ctx.out_force)])
        torch.cuda.synchronize()
        st = ctx.last_stats()
        return [[x.cpu().numpy() for x in o] for o in outs], st
    finally:
        ctx.close()


def test_determinism_and_shard_invariance(torch_cuda):
    """Same seed -> bitwise-identical outputs and stats; an env's outputs depend only
    on its global id, so a 2-way shard (env_offset) reproduces the single-GPU run bit for bit."""
    torch = torch_cuda
    P = presets.preset(FULL)
    n = 1024
    res = {4: (np.arange(n) % 3 == 0).astype(np.uint8)}
    a, sa = _run_outputs(torch, P, n, 8, resets=res)
    b, sb = _run_outputs(torch, P, n, 8, resets=res)
    for x, y in zip(a, b):
        for u, v in zip(x, y):
            assert np.array_equal(u, v)
    assert np.array_equal(sa, sb)
    h0, _ = _run_outputs(torch, P, n // 2, 8, env_offset=0, n_env_global=n, resets=res)
    h1, _ = _run_outputs(torch, P, n // 2, 8, env_offset=n // 2, n_env_global=n, resets=res)
    for x, y0, y1 in zip(a, h0, h1):
        for u, v0, v1 in zip(x, y0, y1):
            assert np.array_equal(u, np.concatenate([v0, v1]))


def test_export_import_resume(torch_cuda):
    """Checkpoint/resume (the paper's seeded deterministic randomization):
    resets at steps 3 and 7, export at step 10, import into a fresh context, continue with another
    reset at step 14 -> outputs identical to the uninterrupted run.  The imported envs' physics rows
    are re-derived from (seed, global id, episode): identical to the exporting context's rows."""
    torch = torch_cuda
    from paper_1906_11633_b200 import dr
    P = presets.preset(FULL)
    n = 300
    acts, obs = gen.frames(n, 20)
    A, O = _frames_cuda(torch, acts), _frames_cuda(torch, obs)
    resets = {3: (np.arange(n) % 3 == 0), 7: (np.arange(n) % 5 == 1), 14: (np.arange(n) % 4 == 2)}
    resets = {t: torch.from_numpy(m.astype(np.uint8)).cuda() for t, m in resets.items()}
    ctx = _ctx(P, n)
    ref = []
    for t in range(20):
        if t == 10:
            snap = dr.dr_state_export()
            tsnap = dr.dr_step_index()
            phys_snap = ctx.phys()
        if t in resets:
            ctx.reset(resets[t])
        ctx.step(A[t], O[t])
        if t >= 10:
            ref.append([x.cpu().numpy() for x in (ctx.out_actions, ctx.out_obs, ctx.out_dt, ctx.out_force)])
    phys_end = ctx.phys()
    ctx.close()
    ctx = _ctx(P, n)
    dr.dr_state_import(snap)
    dr.dr_set_step_index(tsnap)
    assert np.array_equal(ctx.phys(), phys_snap), "physics rows after import"
    for t in range(10, 20):
        if t in resets:
            ctx.reset(resets[t])
        ctx.step(A[t], O[t])
        got = [x.cpu().numpy() for x in (ctx.out_actions, ctx.out_obs, ctx.out_dt, ctx.out_force)]
        for u, v in zip(got, ref[t - 10]):
            assert np.array_equal(u, v)
    assert np.array_equal(ctx.phys(), phys_end)
    ctx.close()


def test_cuda_graph_replay_advances_step(torch_cuda):
    """A CUDA graph of dr_step calls replays with a device-resident step counter: two replays of
    a 4-step graph equal 8 eager steps."""
    torch = torch_cuda
    from paper_1906_11633_b200 import dr
    P = presets.preset(FULL)
    n = 512
    acts, obs = gen.frames(n, 4)
    A, O = _frames_cuda(torch, acts), _frames_cuda(torch, obs)
    eager = []
    ctx = _ctx(P, n)
    for t in range(8):
        ctx.step(A[t % 4], O[t % 4])
        eager.append(ctx.out_obs.cpu().numpy())
    ctx.close()
    ctx = _ctx(P, n)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    outs = [torch.empty_like(ctx.out_obs) for _ in range(4)]
    with torch.cuda.stream(s):
        dr.dr_set_stream(s.cuda_stream)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for t in range(4):
                dr.dr_step(A[t], O[t], ctx.out_actions, outs[t], ctx.out_dt, ctx.out_force)
    for rep in range(2):
        g.replay()
        torch.cuda.synchronize()
        for t in range(4):
            assert np.array_equal(outs[t].cpu().numpy(), eager[4 * rep + t]), (rep, t)
    ctx.close()


def test_workspace_adoption_and_host_path(torch_cuda):
    """A caller-owned (torch) workspace and the host-buffer dr_step_host path give the same
    bits as the default device path."""
    torch = torch_cuda
    from paper_1906_11633_b200 import dr
    P = presets.preset(FULL)
    n = 777
    acts, obs = gen.frames(n, 3)
    A, O = _frames_cuda(torch, acts), _frames_cuda(torch, obs)
    ref = []
    ctx = _ctx(P, n)
    for t in range(3):
        ctx.step(A[t], O[t])
        ref.append([x.cpu().numpy() for x in (ctx.out_actions, ctx.out_obs, ctx.out_dt, ctx.out_force)])
    ctx.close()
    ctx = _ctx(P, n, workspace=True)
    for t in range(3):
        ctx.step(A[t], O[t])
        got = [x.cpu().numpy() for x in (ctx.out_actions, ctx.out_obs, ctx.out_dt, ctx.out_force)]
        for u, v in zip(got, ref[t]):
            assert np.array_equal(u, v)
    ctx.close()
    ctx = _ctx(P, n)
    ha = [torch.from_numpy(a).pin_memory() for a in acts]
    ho = [torch.from_numpy(o).pin_memory() for o in obs]
    outs = [torch.empty(n, c).pin_memory() for c in (20, 22, 10, 3)]
    for t in range(3):
        dr.dr_step_host(ha[t], ho[t], *outs)
        dr.dr_synchronize()
        for u, v in zip(outs, ref[t]):
            assert np.array_equal(u.numpy(), v)
    ctx.close()
    # pipelined: three back-to-back calls (copy streams overlapping), one sync at the end
    ctx = _ctx(P, n)
    outs3 = [[torch.empty(n, c).pin_memory() for c in (20, 22, 10, 3)] for _ in range(3)]
    for t in range(3):
        dr.dr_step_host(ha[t], ho[t], *outs3[t])
    dr.dr_synchronize()
    for t in range(3):
        for u, v in zip(outs3[t], ref[t]):
            assert np.array_equal(u.numpy(), v), t
    ctx.close()


@pytest.mark.parametrize("n", [777, 778])
def test_host_path_contiguous_buffers(torch_cuda, n):
    """dr_step_host with the inputs and the outputs each in one host allocation (the one-copy
    paths: inputs always merge; outputs merge for even n, where the device set has no padding)
    gives the device path's bits, pipelined over three calls."""
    torch = torch_cuda
    from paper_1906_11633_b200 import dr
    P = presets.preset(FULL)
    acts, obs = gen.frames(n, 3)
    A, O = _frames_cuda(torch, acts), _frames_cuda(torch, obs)
    ctx = _ctx(P, n)
    ref = []
    for t in range(3):
        ctx.step(A[t], O[t])
        ref.append([x.cpu().numpy() for x in (ctx.out_actions, ctx.out_obs, ctx.out_dt, ctx.out_force)])
    ctx.close()
    ctx = _ctx(P, n)
    hins, houts = [], []
    for t in range(3):
        hin = torch.empty(n * 46).pin_memory()
        hin[:n * 20].copy_(torch.from_numpy(acts[t]).reshape(-1))
        hin[n * 20:].copy_(torch.from_numpy(obs[t]).reshape(-1))
        hout = torch.full((n * 55,), float("nan")).pin_memory()
        views, o = [], 0
        for c in (20, 22, 10, 3):
            views.append(hout[o:o + n * c].view(n, c))
            o += n * c
        hins.append((hin[:n * 20].view(n, 20), hin[n * 20:].view(n, 26)))
        houts.append(views)
        dr.dr_step_host(*hins[t], *houts[t])
    dr.dr_synchronize()
    for t in range(3):
        for u, v in zip(houts[t], ref[t]):
            assert np.array_equal(u.numpy(), v), t
    ctx.close()


def test_value_view_isolation_and_invariants_1M(torch_cuda):
    """Inputs are never written; GPU-only invariants over every env of a 1M-env
    full-pipeline run: |a_out| <= 1, dt_k >= 8 ms, relative-goal w >= 0 and unit norm, slack in
    [-1, 1], dropout timers <= 12."""
    torch = torch_cuda
    P = presets.preset(FULL)
    n = 1 << 20
    g = torch.Generator(device="cuda").manual_seed(1)
    k = torch.randint(0, 11, (n, 20), device="cuda", generator=g)
    A = (-1.0 + (2.0 * k + 1.0) / 11.0).float()
    O = torch.randn(n, 26, device="cuda", generator=g) * 0.01
    O[:, 18:22] /= O[:, 18:22].norm(dim=1, keepdim=True)
    O[:, 22:26] /= O[:, 22:26].norm(dim=1, keepdim=True)
    A0, O0 = A.clone(), O.clone()
    ctx = _ctx(P, n)
    try:
        for t in range(4):
            ctx.step(A, O)
            torch.cuda.synchronize()
            assert ctx.out_actions.abs().max().item() <= 1.0
            assert ctx.out_dt.min().item() >= np.float32(0.008)
            rel = ctx.out_obs[:, :4]
            assert rel[:, 0].min().item() >= 0.0
            assert (rel.norm(dim=1) - 1).abs().max().item() < 1e-5
            assert torch.isfinite(ctx.out_obs).all() and torch.isfinite(ctx.out_force).all()
        assert torch.equal(A, A0) and torch.equal(O, O0)
        st = ctx.export(0, 4096)
        assert np.abs(st["slack"]).max() <= 1.0
        tim = np.stack([(st["flags"] >> (4 * i)) & 15 for i in range(5)])
        assert tim.max() <= 12
        s = ctx.last_stats()
        assert s[0] == n
    finally:
        ctx.close()


def test_large_8M_envs_sampled(torch_cuda):
    """Size edge: 8,388,608 envs (8x config 4, ~20 GB of state + I/O, grid-stride over 65,536 tiles)
    -- inputs generated on the device, 48 sampled envs (incl. the first and last tiles) compared
    with the oracle every step, a masked reset of every 7th env in between."""
    torch = torch_cuda
    from oracle.oracle import Oracle
    from paper_1906_11633_b200 import dr
    P = presets.preset(FULL)
    n = 1 << 23
    rng = np.random.default_rng(8)
    sample = np.sort(np.concatenate([[0, 1, 127, 128, n - 129, n - 2, n - 1], rng.choice(n, 41, replace=False)]))
    gen_t = torch.Generator(device="cuda").manual_seed(presets.SEED_WORKLOAD)
    ctx = _ctx(P, n)
    orc = Oracle(P, len(sample), SEED, gids=sample)
    idx = torch.from_numpy(sample).cuda()
    try:
        for t in range(4):
            if t == 2:
                m = (torch.arange(n, device="cuda") % 7 == 3).to(torch.uint8)
                ctx.reset(m)
                orc.reset(m[idx].cpu().numpy())
            k = torch.randint(0, 11, (n, 20), device="cuda", generator=gen_t)
            A = (-1.0 + (2.0 * k + 1.0) / 11.0).float().contiguous()
            del k
            O = torch.empty(n, 26, device="cuda")
            O[:, 0:15] = torch.tensor(gen.TIP_NOMINAL.reshape(-1), device="cuda", dtype=torch.float32) + \
                gen.TIP_JITTER * torch.randn(n, 15, device="cuda", generator=gen_t)
            O[:, 15:18] = torch.tensor(gen.OBJ_NOMINAL, device="cuda", dtype=torch.float32) + \
                gen.OBJ_JITTER * torch.randn(n, 3, device="cuda", generator=gen_t)
            q = torch.randn(n, 8, device="cuda", generator=gen_t)
            O[:, 18:22] = q[:, 0:4] / q[:, 0:4].norm(dim=-1, keepdim=True)
            O[:, 22:26] = q[:, 4:8] / q[:, 4:8].norm(dim=-1, keepdim=True)
            del q
            ctx.step(A, O)
            r = orc.step(A[idx].cpu().numpy(), O[idx].cpu().numpy(), want_margin=True)
            torch.cuda.synchronize()
            knife = KnifeTracker(len(sample))
            knife.update_before_compare(r["margin"])
            knife.compare_actions(ctx.out_actions[idx].cpu().numpy(), r["out_actions"], t)
            compare_obs(ctx.out_obs[idx].cpu().numpy(), r["out_obs"], t)
            assert_close(f"out_dt t={t}", ctx.out_dt[idx].cpu().numpy(), r["out_dt"], 0.008)
            mass = np.array([orc.env(i)["mass"] for i in range(len(sample))])
            assert_close(f"out_force t={t}", ctx.out_force[idx].cpu().numpy(), r["out_force"], mass[:, None])
            assert ctx.last_stats()[0] == n
            del A, O
        for i, gid in enumerate(sample[:: 6]):
            st = dr.states_to_numpy(dr.dr_state_export(int(gid), int(gid) + 1))
            assert st["episode"][0] == orc.env(6 * i)["episode"] and st["t_force"][0] == orc.env(6 * i)["t_force"]
    finally:
        ctx.close()
        orc.close()


def test_full_size_statistics_1M(torch_cuda):
    """Full-size parity via properties that hold at any size (1M envs, full pipeline, 24 steps),
    against closed forms fixed by the paper's tables: E[dt_env] = 10 (8 ms + ln 8 / 8750 s)
    (PAPER.md:84-88); the force trigger rate E[p] = 0.099 / ln 100 (loguniform 0.1 %-10 %,
    PAPER.md:113); the dropout initiation rate 1 - exp(-0.2 * 0.08) per tip-step and the
    steady-state masked fraction 1 - (1 - p)^13; half of all actuators delayed
    (PAPER.md:77-78); unit-variance uncorrelated action and fingertip normals."""
    torch = torch_cuda
    P = presets.preset(FULL)
    n = 1 << 20
    g = torch.Generator(device="cuda").manual_seed(5)
    k = torch.randint(0, 11, (n, 20), device="cuda", generator=g)
    A = (-1.0 + (2.0 * k + 1.0) / 11.0).float().contiguous()
    O = torch.empty(n, 26, device="cuda")
    O[:, 0:15] = torch.tensor(gen.TIP_NOMINAL.reshape(-1), device="cuda", dtype=torch.float32) + \
        gen.TIP_JITTER * torch.randn(n, 15, device="cuda", generator=g)
    O[:, 15:18] = torch.tensor(gen.OBJ_NOMINAL, device="cuda", dtype=torch.float32) + \
        gen.OBJ_JITTER * torch.randn(n, 3, device="cuda", generator=g)
    q = torch.randn(n, 8, device="cuda", generator=g)
    O[:, 18:22] = q[:, :4] / q[:, :4].norm(dim=1, keepdim=True)
    O[:, 22:26] = q[:, 4:] / q[:, 4:].norm(dim=1, keepdim=True)
    ctx = _ctx(P, n)
    T = 24
    acc = np.zeros(32)
    try:
        for t in range(T):
            ctx.step(A, O)
            s = ctx.last_stats()
            assert s[0] == n
            acc += s
            if t == T - 1:
                masked_last = s[3] / (5.0 * n)
    finally:
        ctx.close()
    steps = T * n
    # substep timing: E[dt_env] over lambda ~ U[1250, 10000]
    e_dt = 10 * (0.008 + math.log(8.0) / 8750.0)
    assert abs(acc[16] / steps - e_dt) < 5e-6
    # force trigger rate (2.4e7 env-steps; binomial sd ~3e-5)
    assert abs(acc[6] / steps - 0.099 / math.log(100.0)) < 2e-4
    # dropout: initiation rate per tip-step and the steady-state masked fraction (after 13+ steps)
    p_d = 1.0 - math.exp(-0.2 * 0.08)
    assert abs(acc[2] / (5 * steps) - p_d) < 2e-4
    assert abs(masked_last - (1.0 - (1.0 - p_d) ** 13)) < 2e-3
    # delay flags: half of all actuators (each env's 20 flags drawn once per episode)
    assert abs(acc[1] / (20 * steps) - 0.5) < 2e-3
    # unit-variance normals: sum z_u^2 over actions, sum z^2 over fingertip coordinates
    assert abs(acc[21] / (20 * steps) - 1.0) < 2e-3
    assert abs(acc[22] / (15 * steps) - 1.0) < 2e-3
