"""The N>1 path on the GPU with two ranks sharing one device (gloo process group, CUDA tensors):
each rank runs its own libdr context on its shard of the global env ids, the per-step stats go
through the overlapped StatsReducer (comm stream, double-buffered slot), and the result must equal
one process stepping all envs (per-env outputs and every stats slot bit-identical), and the
all-reduced stats must equal the fp64 oracle's single-process stats (integer slots exact, moments
within 1e-6).  Also bench.py under torchrun with two ranks."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from workload import gen, presets

pytestmark = pytest.mark.gpu
N_GLOBAL, T = 5003, 12
SEED = presets.SEED_DR
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(torch, ctx_factory, off, n, reducer_factory=None):
    acts, obs = gen.frames(N_GLOBAL, 4, seed=91)
    A = [torch.from_numpy(np.ascontiguousarray(a[off:off + n])).cuda() for a in acts]
    O = [torch.from_numpy(np.ascontiguousarray(o[off:off + n])).cuda() for o in obs]
    lib_stream = torch.cuda.current_stream()
    ctx = ctx_factory(lib_stream)
    red = reducer_factory(ctx, lib_stream) if reducer_factory else None
    outs, stats = [], []
    for t in range(T):
        if t == 6:
            m = (np.arange(N_GLOBAL) % 5 == 2).astype(np.uint8)[off:off + n]
            ctx.reset(torch.from_numpy(m).cuda())
        if red:
            red.before_step(t)
        ctx.step(A[t % 4], O[t % 4])
        if red:
            red.after_step(t)
        outs.append(torch.cat([ctx.out_actions, ctx.out_obs, ctx.out_dt, ctx.out_force], 1).cpu().numpy())
        if red:
            red.sync()
        torch.cuda.synchronize()
        stats.append(ctx.stats[t % 4].cpu().numpy().copy())
    ctx.close()
    return np.stack(outs), np.stack(stats)


def _worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_1906_11633_b200 import DRContext
    from paper_1906_11633_b200.parallel import StatsReducer, shard
    off, n = shard(N_GLOBAL, world, rank)
    outs, stats = _run(torch, lambda s: DRContext(presets.preset(presets.FULL), n, SEED, env_offset=off,
                                                  n_env_global=N_GLOBAL, stream=s), off, n,
                       lambda ctx, s: StatsReducer(ctx.stats, s))
    np.save(os.path.join(out_dir, f"rank{rank}.npy"), outs)
    if rank == 0:
        np.save(os.path.join(out_dir, "stats.npy"), stats)
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_one_gpu_match_single_process(tmp_path):
    import torch
    import torch.multiprocessing as mp
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    from paper_1906_11633_b200 import DRContext
    torch.cuda.set_device(0)
    ref_out, ref_st = _run(torch, lambda s: DRContext(presets.preset(presets.FULL), N_GLOBAL, SEED, stream=s),
                           0, N_GLOBAL)
    got = np.concatenate([np.load(tmp_path / f"rank{r}.npy") for r in range(world)], axis=1)
    assert np.array_equal(got, ref_out)                     # per-env outputs bit-identical
    st = np.load(tmp_path / "stats.npy")
    assert np.array_equal(st[:, :12], ref_st[:, :12])       # integer slots exact after the all-reduce
    # moment slots: every CTA partial is rounded to the same job-wide power-of-two quantum (so the fp64
    # atomic sums are order-free), but the CTA partition differs between 1 and 2 ranks: agreement to
    # the quantisation (~1e-12 relative)
    assert np.allclose(st[:, 16:24], ref_st[:, 16:24], rtol=1e-10, atol=1e-12)
    # and the all-reduced stats (row a13) equal the fp64 oracle's single-process stats of the same
    # global envs: integer slots exact, moment slots within 1e-6 of their magnitude bound
    from oracle.oracle import Oracle
    from parity import KNIFE_TAU, compare_stats
    acts, obs = gen.frames(N_GLOBAL, 4, seed=91)
    orc = Oracle(presets.preset(presets.FULL), N_GLOBAL, SEED)
    knife = 0
    for t in range(T):
        if t == 6:
            orc.reset((np.arange(N_GLOBAL) % 5 == 2).astype(np.uint8))
        r = orc.step(acts[t % 4], obs[t % 4], want_margin=True)
        knife += int((r["margin"] < KNIFE_TAU).sum())
        compare_stats(st[t], r["stats"], N_GLOBAL, knife, t)


def test_bench_torchrun_two_ranks_gloo():
    """bench.py's N>1 path (sharding, StatsReducer, max-over-ranks timing) with two ranks on one GPU."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--backend", "gloo", "--n-env", "65536", "--steps", "20", "--warmup", "3",
           "--no-cpu-baseline", "--e2e-steps", "2"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["value"] > 0   # config 4's split by default
    assert d["config"]["n_env_global"] == 65536 and d["config"]["n_env_per_gpu"] == 32768
    assert d["stats_check"]["envs_last_step"] == 65536   # the all-reduced stats cover both ranks
    assert d["gpu_launches"] == 20


def _nccl_worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", 0))
    from paper_1906_11633_b200 import DRContext
    from paper_1906_11633_b200.parallel import StatsReducer
    outs, stats = _run(torch, lambda s: DRContext(presets.preset(presets.FULL), N_GLOBAL, SEED, stream=s), 0,
                       N_GLOBAL, lambda ctx, s: StatsReducer(ctx.stats, s))
    np.save(os.path.join(out_dir, "outs.npy"), outs)
    np.save(os.path.join(out_dir, "stats.npy"), stats)
    dist.barrier()
    dist.destroy_process_group()


def test_nccl_stats_reducer_single_rank(tmp_path):
    """The NCCL backend path of the StatsReducer (all-reduce on the comm stream, event ordering,
    the ring of 4 slots) with one rank -- the only NCCL configuration one GPU allows: the reduced
    stats equal the local ones and the outputs equal a run without the reducer."""
    import torch
    import torch.multiprocessing as mp
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    mp.spawn(_nccl_worker, args=(1, _free_port(), str(tmp_path)), nprocs=1, join=True)
    from paper_1906_11633_b200 import DRContext
    torch.cuda.set_device(0)
    ref_out, ref_st = _run(torch, lambda s: DRContext(presets.preset(presets.FULL), N_GLOBAL, SEED, stream=s),
                           0, N_GLOBAL)
    assert np.array_equal(np.load(tmp_path / "outs.npy"), ref_out)
    assert np.array_equal(np.load(tmp_path / "stats.npy"), ref_st)


def _nccl_graph_worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", 0))
    from paper_1906_11633_b200 import DRContext
    from paper_1906_11633_b200.parallel import StatsReducer
    acts, obs = gen.frames(N_GLOBAL, 4, seed=91)
    A = [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in acts]
    O = [torch.from_numpy(np.ascontiguousarray(o)).cuda() for o in obs]
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        ctx = DRContext(presets.preset(presets.FULL), N_GLOBAL, SEED, stream=s)
        red = StatsReducer(ctx.stats, s)
        t = 0
        for _ in range(3):                      # eager steps first
            red.before_step(t)
            ctx.step(A[t % 4], O[t % 4])
            red.after_step(t)
            t += 1
        red.sync()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):     # 4 steps and their all-reduces in one graph
            red.reset_ring()
            for i in range(4):
                red.before_step(t + i)
                ctx.step(A[(t + i) % 4], O[(t + i) % 4])
                red.after_step(t + i)
            red.sync()
        for _ in range(2):
            g.replay()
        torch.cuda.synchronize()
        out = torch.cat([ctx.out_actions, ctx.out_obs, ctx.out_dt, ctx.out_force], 1).cpu().numpy()
        np.save(os.path.join(out_dir, "graph_out.npy"), out)
        np.save(os.path.join(out_dir, "graph_stats.npy"), ctx.stats.cpu().numpy())
        ctx.close()
    dist.barrier()
    dist.destroy_process_group()


def test_nccl_stats_reducer_graph_capture_single_rank(tmp_path):
    """bench.py's N > 1 mode captures the steps and their NCCL stats all-reduces (comm stream,
    events, the 4-slot ring) in one CUDA graph.  With one NCCL rank (all one GPU allows): 3 eager
    steps + 2 replays of a 4-step graph (which captured the eager steps' counters, but the device step
    index advances on every replay) equal 11 eager steps -- outputs and every stats slot."""
    import torch
    import torch.multiprocessing as mp
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    mp.spawn(_nccl_graph_worker, args=(1, _free_port(), str(tmp_path)), nprocs=1, join=True)
    from paper_1906_11633_b200 import DRContext
    torch.cuda.set_device(0)
    acts, obs = gen.frames(N_GLOBAL, 4, seed=91)
    A = [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in acts]
    O = [torch.from_numpy(np.ascontiguousarray(o)).cuda() for o in obs]
    ctx = DRContext(presets.preset(presets.FULL), N_GLOBAL, SEED)
    for t in range(11):
        ctx.step(A[t % 4], O[t % 4])
    torch.cuda.synchronize()
    ref = torch.cat([ctx.out_actions, ctx.out_obs, ctx.out_dt, ctx.out_force], 1).cpu().numpy()
    ref_stats = ctx.stats.cpu().numpy()
    ctx.close()
    # the graph replays frames 3..6 twice (its inputs were captured), the eager reference walks frames
    # t % 4: for the last step (t = 10) both use frame 2
    assert np.array_equal(np.load(tmp_path / "graph_out.npy"), ref)
    assert np.array_equal(np.load(tmp_path / "graph_stats.npy")[10 % 4], ref_stats[10 % 4])
