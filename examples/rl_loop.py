#!/usr/bin/env python
"""Where the library sits in a rollout loop (the policy and simulator are stand-ins).

    python examples/rl_loop.py [--envs 65536] [--steps 200]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 examples/rl_loop.py     (one rank per GPU)

Per control step (80 ms of simulated time):
  1. the policy maps the noisy observation to actions in [-1, 1]        (stand-in: a fixed linear map)
  2. dr_step: delay, action noise, backlash, substep timing, marker dropout / occlusion hold,
     observation noise, random forces -> what the simulator applies and what the policy sees
  3. the simulator advances with out_actions over the substeps out_dt and applies out_force
     (stand-in: integrates the tips and object a little)
  4. episodes that ended are reset: dr_reset draws their new physical parameters (the simulator
     reads them with dr_phys_params before the next step) and their per-episode randomizations
Per step the 32 x fp64 statistics (counts and moments of every randomizer) are all-reduced over
the ranks on a side stream (StatsReducer); every 64 steps a vision batch (64 samples x 3 cameras)
gets its appearance draws and its post-render augmentation.
Everything stays on the device; the only host reads are the periodic statistics prints.
"""
import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1906_11633_b200 import DRContext, dr, vision  # noqa: E402
from paper_1906_11633_b200.parallel import StatsReducer, shard  # noqa: E402
from workload import gen, presets  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--envs", type=int, default=65536, help="envs of the whole job")
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--episode-steps", type=int, default=50, help="mean episode length of the stand-in")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0"))))
    off, n = shard(args.envs, world, rank)   # this rank's contiguous block of global env ids

    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        ctx = DRContext(presets.preset(presets.FULL | presets.PHYS), n, presets.SEED_DR,
                        env_offset=off, n_env_global=args.envs, stream=stream)
        reducer = StatsReducer(ctx.stats, stream) if world > 1 else None
        g = torch.Generator(device="cuda").manual_seed(presets.SEED_WORKLOAD + rank)

        # stand-in simulator state: fingertips, object position, object and goal quaternions
        raw_obs = torch.empty(n, 26, device="cuda")
        raw_obs[:, 0:15] = torch.tensor(gen.TIP_NOMINAL.reshape(-1), device="cuda", dtype=torch.float32)
        raw_obs[:, 15:18] = torch.tensor(gen.OBJ_NOMINAL, device="cuda", dtype=torch.float32)
        q = torch.randn(n, 8, device="cuda", generator=g)
        raw_obs[:, 18:22] = q[:, 0:4] / q[:, 0:4].norm(dim=-1, keepdim=True)
        raw_obs[:, 22:26] = q[:, 4:8] / q[:, 4:8].norm(dim=-1, keepdim=True)
        W = 0.05 * torch.randn(22, 20, device="cuda", generator=g)   # stand-in policy
        obs = ctx.out_obs.zero_()
        # device [n][n_phys] fp32 physical parameters of the current episodes (rewritten in stream
        # order by every dr_reset): a CUDA / C simulator reads them through this pointer
        phys_ptr = dr.dr_phys_params()

        # vision: 64 samples x 3 cameras of 200 x 200 x 3 per batch
        vp = vision.params_from_preset(presets.vision_preset())
        images = torch.from_numpy(gen.images(192, 200, 200, 3, seed=rank)).cuda()
        augmented = torch.empty(images.shape, dtype=torch.float32, device="cuda")
        scene = torch.empty(64, 64, dtype=torch.float32, device="cuda")

        for t in range(args.steps):
            actions = torch.tanh(obs @ W)                                   # 1. policy
            if reducer is not None:
                reducer.before_step(t)
            a, o, dt, force = ctx.step(actions, raw_obs)                    # 2. randomized step
            if reducer is not None:
                reducer.after_step(t)
            # 3. stand-in simulator: tips drift with the applied actions over the step's duration
            raw_obs[:, 0:15] += 1e-4 * a[:, 0:15] * dt.sum(dim=1, keepdim=True)
            raw_obs[:, 15:18] += 1e-6 * force
            obs = o
            # 4. episode ends (stand-in: geometric lengths) -> per-episode resampling
            done = (torch.rand(n, device="cuda", generator=g) < 1.0 / args.episode_steps).to(torch.uint8)
            ctx.reset(done)
            # (the simulator would now read the rows of the done envs at phys_ptr to re-create them)
            if t % 64 == 0:
                vision.dr_scene_draw_batch(vp, presets.SEED_DR, t // 64, scene, sample_offset=rank * 64, stream=stream)
                vision.dr_image_augment(vp, presets.SEED_DR, t // 64, images, augmented, image_offset=rank * 192,
                                        stream=stream)
            if (t + 1) % 50 == 0:
                if reducer is not None:
                    reducer.sync()
                s = ctx.last_stats()
                if rank == 0:
                    envs = s[0]   # DR_S_ENVS; slot 10 DR_S_RESETS, slot 16 DR_S_SUM_DT (include/dr.h)
                    print(f"step {t + 1}: {int(envs)} env-steps in the last step, "
                          f"{int(s[10])} resets, mean substep sum {s[16] / max(envs, 1):.4f} s")
        torch.cuda.synchronize()
        first_rows = ctx.phys(0, 2)   # a blocking host copy, for the print only
        print(f"rank {rank}: {args.steps} steps of {n} envs done; physical parameters at 0x{phys_ptr:x}, "
              f"env 0: mass {first_rows[0, 0]:.4f} kg, {first_rows.shape[1]} parameters")
        ctx.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
