"""Environment-sharded data parallelism.

Envs are independent, so the path shards by environment: rank r of W owns the contiguous
global ids [offset_r, offset_r + n_r) and runs its own libdr context with env_offset =
offset_r and n_env_global = N (same seed).  Philox counters use global ids, so every env's
outputs are bit-identical for any W.  The only exchange is the per-step statistics vector
(32 x fp64 = 256 B), summed over ranks with one all-reduce on a dedicated comm stream so it
overlaps the next steps (a ring of 4 stats slots).  Plumbing only: no arithmetic of the
method lives here.
"""
from __future__ import annotations


def shard(n_global: int, world: int, rank: int):
    """(offset, n_local) of `rank`: contiguous blocks, the first n_global % world ranks one larger."""
    if not (0 <= rank < world) or n_global < world:
        raise ValueError(f"cannot shard {n_global} envs over {world} ranks (rank {rank})")
    base, extra = divmod(n_global, world)
    n = base + (1 if rank < extra else 0)
    off = rank * base + min(rank, extra)
    return off, n


def stats_all_reduce(stats_slot, group=None, async_op: bool = False):
    """Sum one [32] fp64 stats slot over the ranks (NCCL on GPU tensors, gloo on CPU tensors)."""
    import torch.distributed as dist
    return dist.all_reduce(stats_slot, op=dist.ReduceOp.SUM, group=group, async_op=async_op)


class StatsReducer:
    """The overlapped per-step stats all-reduce on a dedicated comm stream.

    Step t's kernel accumulates into stats slot t % 4 and clears slot (t + 1) % 4 (include/dr.h).
    The all-reduce of slot t % 4 runs on the comm stream after an event recorded behind step t,
    so it overlaps the following steps; before step t is enqueued, the library stream waits for
    the all-reduce of step t - 3 (whose slot step t clears), so the ring is never raced."""

    SLOTS = 4

    def __init__(self, stats, lib_stream, group=None):
        import torch
        self.stats = stats
        self.lib_stream = lib_stream
        self.comm_stream = torch.cuda.Stream()
        self.group = group
        self.done = [None] * self.SLOTS

    def reset_ring(self):
        """Forget the pending all-reduce events (e.g. at the start of a CUDA-graph capture whose
        predecessor work was joined by sync())."""
        self.done = [None] * self.SLOTS

    def before_step(self, t: int):
        ev = self.done[(t + 1) % self.SLOTS]   # the all-reduce of step t - 3
        if ev is not None:
            self.lib_stream.wait_event(ev)

    def after_step(self, t: int):
        import torch
        ev = torch.cuda.Event()
        ev.record(self.lib_stream)
        self.comm_stream.wait_event(ev)
        with torch.cuda.stream(self.comm_stream):
            stats_all_reduce(self.stats[t % self.SLOTS], group=self.group)
        done = torch.cuda.Event()
        done.record(self.comm_stream)
        self.done[t % self.SLOTS] = done

    def sync(self):
        self.lib_stream.wait_stream(self.comm_stream)


class ShardedDR:
    """One rank's context plus the overlapped stats all-reduce (needs CUDA + an initialised
    process group)."""

    def __init__(self, preset: dict, n_global: int, seed: int, lib_stream=None):
        import torch
        import torch.distributed as dist
        from . import DRContext
        self.world = dist.get_world_size() if dist.is_initialized() else 1
        self.rank = dist.get_rank() if dist.is_initialized() else 0
        self.offset, self.n = shard(n_global, self.world, self.rank)
        self.lib_stream = lib_stream or torch.cuda.current_stream()
        self.ctx = DRContext(preset, self.n, seed, env_offset=self.offset, n_env_global=n_global,
                             stream=self.lib_stream)
        self.reducer = StatsReducer(self.ctx.stats, self.lib_stream) if self.world > 1 else None
        self.t = 0

    def step(self, actions, raw_obs):
        if self.reducer is not None:
            self.reducer.before_step(self.t)
        out = self.ctx.step(actions, raw_obs)
        if self.reducer is not None:
            self.reducer.after_step(self.t)
        self.t += 1
        return out

    def sync_comm(self):
        if self.reducer is not None:
            self.reducer.sync()

    def close(self):
        self.ctx.close()
