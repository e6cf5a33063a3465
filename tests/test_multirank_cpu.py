"""The N>1 path on CPU: world_size-2 gloo process group, envs sharded by global id, per-step
stats all-reduced.  The fp64 oracle stands in for each rank's device context (it keys every draw
by the global env id, exactly like the kernels); the check is that sharding + the stats
all-reduce reproduce the single-process run: per-env outputs bit-identical, integer stats
exact, fp64 moment stats to rounding."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from workload import gen, presets

N_GLOBAL, T = 37, 6          # odd size: uneven shards
SEED = presets.SEED_DR


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.oracle import Oracle
    from paper_1906_11633_b200.parallel import shard, stats_all_reduce
    off, n = shard(N_GLOBAL, world, rank)
    acts, obs = gen.frames(N_GLOBAL, T, seed=77)
    orc = Oracle(presets.preset(presets.FULL), n, SEED, gids=np.arange(off, off + n))
    outs, stats = [], []
    for t in range(T):
        if t == 3:
            m = (np.arange(N_GLOBAL) % 4 == 1).astype(np.uint8)
            orc.reset(m[off:off + n])
        r = orc.step(acts[t][off:off + n], obs[t][off:off + n])
        st = torch.from_numpy(r["stats"].copy())
        stats_all_reduce(st)
        stats.append(st.numpy())
        outs.append(np.concatenate([r["out_actions"], r["out_obs"], r["out_dt"], r["out_force"]], axis=1))
    np.save(os.path.join(out_dir, f"rank{rank}.npy"), np.stack(outs))
    if rank == 0:
        np.save(os.path.join(out_dir, "stats.npy"), np.stack(stats))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_ranges():
    from paper_1906_11633_b200.parallel import shard
    for n, w in [(37, 2), (1 << 20, 8), (10, 3), (8, 8)]:
        ranges = [shard(n, w, r) for r in range(w)]
        assert ranges[0][0] == 0
        for (o0, n0), (o1, _) in zip(ranges, ranges[1:]):
            assert o0 + n0 == o1
        assert sum(x[1] for x in ranges) == n
        assert max(x[1] for x in ranges) - min(x[1] for x in ranges) <= 1
    with pytest.raises(ValueError):
        shard(3, 4, 0)


def test_two_rank_gloo_sharding_matches_single_process(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    from oracle.oracle import Oracle
    acts, obs = gen.frames(N_GLOBAL, T, seed=77)
    orc = Oracle(presets.preset(presets.FULL), N_GLOBAL, SEED)
    ref_out, ref_st = [], []
    for t in range(T):
        if t == 3:
            orc.reset((np.arange(N_GLOBAL) % 4 == 1).astype(np.uint8))
        r = orc.step(acts[t], obs[t])
        ref_out.append(np.concatenate([r["out_actions"], r["out_obs"], r["out_dt"], r["out_force"]], axis=1))
        ref_st.append(r["stats"])
    got = np.concatenate([np.load(tmp_path / f"rank{r}.npy") for r in range(world)], axis=1)
    assert np.array_equal(got, np.stack(ref_out))          # bit-identical per-env outputs
    st = np.load(tmp_path / "stats.npy")
    ref_st = np.stack(ref_st)
    assert np.array_equal(st[:, :12], ref_st[:, :12])       # integer slots exact
    assert np.allclose(st[:, 16:24], ref_st[:, 16:24], rtol=1e-12, atol=1e-12)
