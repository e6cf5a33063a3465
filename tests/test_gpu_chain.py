"""Chained steps (dr_step.cuh): back-to-back dr_step calls overlap at their boundary -- a step reads
each 128-env tile only after the previous step published it, and finishes only after its
predecessor did.  The results must be those of fully serialised steps (DR_CHAIN=0) bit for bit:
every step's outputs, the exported state, the physics rows and every stats slot -- with resets in
between (a reset always waits), ragged tail tiles, more tiles than CTAs, and CUDA-graph replays."""
import numpy as np
import pytest

from workload import gen, presets

pytestmark = pytest.mark.gpu
SEED = presets.SEED_DR


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.fixture(autouse=True)
def _finalize_leaked_context():
    yield
    from paper_1906_11633_b200 import dr
    dr.load().dr_finalize()


def _run(torch, monkeypatch, chain, mask, n, T, resets, graph_at=None, G=4, mode="throughput"):
    from paper_1906_11633_b200 import DRContext, dr
    monkeypatch.setenv("DR_STEP_MODE", mode)
    monkeypatch.setenv("DR_CHAIN", "1" if chain else "0")
    acts, obs = gen.frames(n, 4, seed=123)
    A = [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in acts]
    O = [torch.from_numpy(np.ascontiguousarray(o)).cuda() for o in obs]
    M = {t: torch.from_numpy(m).cuda() for t, m in resets.items()}
    s = torch.cuda.Stream()
    outs = []
    with torch.cuda.stream(s):
        ctx = DRContext(presets.preset(mask), n, SEED, stream=s)
        bufs = [[torch.empty_like(x) for x in (ctx.out_actions, ctx.out_obs, ctx.out_dt, ctx.out_force)] for _ in range(T)]
        t = 0
        while t < T:
            if graph_at is not None and t == graph_at:
                g = torch.cuda.CUDAGraph()   # G back-to-back steps captured (PDL edges in the graph)
                with torch.cuda.graph(g, stream=s):
                    for i in range(G):
                        ctx.step(A[(t + i) % 4], O[(t + i) % 4], outs=bufs[t + i])
                g.replay()
                t += G
                continue
            if t in M:
                ctx.reset(M[t])
            ctx.step(A[t % 4], O[t % 4], outs=bufs[t])   # no host synchronisation between steps
            t += 1
        torch.cuda.synchronize()
        outs = [[x.cpu().numpy() for x in b] for b in bufs]
        st = ctx.export()
        ph = ctx.phys()
        stats = ctx.stats.cpu().numpy()
        t_dev = dr.dr_step_index_sync()
        ctx.close()
    return outs, st, ph, stats, t_dev


@pytest.mark.parametrize("mask,n,mode", [(presets.FULL, 300, "throughput"), (presets.FULL, 70001, "throughput"),
                                         (presets.CFG2, 131077, "throughput"),
                                         (presets.FULL | presets.SMOOTH, 5000, "throughput"),
                                         (presets.FULL, 4099, "latency"), (presets.CFG2, 200, "latency")])
def test_chained_steps_equal_serialised(torch_cuda, monkeypatch, mask, n, mode):
    T = 14
    resets = {5: (np.arange(n) % 7 == 3).astype(np.uint8), 6: (np.arange(n) % 5 == 0).astype(np.uint8)}
    a = _run(torch_cuda, monkeypatch, True, mask, n, T, resets, graph_at=9, mode=mode)
    b = _run(torch_cuda, monkeypatch, False, mask, n, T, resets, graph_at=9, mode=mode)
    for t, (x, y) in enumerate(zip(a[0], b[0])):
        for u, v in zip(x, y):
            assert np.array_equal(u, v), f"step {t}"
    for k in a[1]:
        assert np.array_equal(a[1][k], b[1][k]), k
    assert np.array_equal(a[2], b[2])
    assert np.array_equal(a[3], b[3])          # the whole stats ring (the last 4 steps)
    assert a[4] == b[4] == T
