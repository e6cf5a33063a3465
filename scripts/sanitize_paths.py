"""Every libdr kernel path once at small, ragged sizes, for compute-sanitizer (memcheck, racecheck,
synccheck, initcheck): both step kernels (throughput with a ragged tail tile, latency), every
reset kernel version, the substep/smoothing layer set, the host-buffer step, the vision kernels
(cluster and two-pass augmentation, unaligned bytes), scene draws and pose augmentation.
Run: compute-sanitizer --tool <tool> python scripts/sanitize_paths.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1906_11633_b200 import DRContext, dr, vision  # noqa: E402
from workload import gen, presets  # noqa: E402


def run_dr(mask, n, steps, env=None):
    for k, v in (env or {}).items():
        os.environ[k] = v
    try:
        P = presets.preset(mask)
        acts, obs = gen.frames(n, 4)
        A = [torch.from_numpy(acts[i]).cuda() for i in range(4)]   # separate (16-byte aligned) frames
        O = [torch.from_numpy(obs[i]).cuda() for i in range(4)]
        with DRContext(P, n, presets.SEED_DR) as ctx:
            for t in range(steps):
                if t == 2:
                    ctx.reset(torch.from_numpy((np.arange(n) % 3 == 1).astype(np.uint8)).cuda())
                ctx.step(A[t % 4], O[t % 4])
            ctx.export()
            ctx.phys()
            torch.cuda.synchronize()
    finally:
        for k in (env or {}):
            del os.environ[k]


run_dr(presets.FULL, 300, 4)                                     # throughput kernel, ragged tail tile
run_dr(presets.FULL, 300, 4, {"DR_STEP_MODE": "latency"})
run_dr(presets.CFG2, 70, 3, {"DR_STEP_MODE": "latency"})
run_dr(presets.FULL, 257, 3)                                     # reset + step at a ragged size
run_dr(presets.FULL | presets.SMOOTH | presets.SUBSTEP_BACKLASH, 130, 3)
run_dr(presets.FULL, 300, 3, {"DR_PDL": "0"})
# host-buffer step
P = presets.preset(presets.FULL)
acts, obs = gen.frames(200, 2)
with DRContext(P, 200, presets.SEED_DR) as ctx:
    outs = [torch.empty(200, c).pin_memory() for c in (20, 22, 10, 3)]
    for t in range(3):
        dr.dr_step_host(torch.from_numpy(acts[t % 2]).pin_memory(), torch.from_numpy(obs[t % 2]).pin_memory(), *outs)
    dr.dr_synchronize()
# vision
VP = presets.vision_preset()
vp = vision.params_from_preset(VP)
for shape in ((3, 17, 13, 3), (2, 64, 48, 4), (2, 200, 200, 3)):
    x = torch.from_numpy(gen.images(*shape, seed=1)).cuda()
    out = torch.empty(x.shape, dtype=torch.float32, device="cuda")
    st = torch.empty(x.shape[0], 4, device="cuda")
    vision.dr_image_augment(vp, presets.SEED_DR, 0, x, out, st)
torch.cuda.synchronize()
scene = torch.empty(37, 64, dtype=torch.float32, device="cuda")
vision.dr_scene_draw_batch(vp, presets.SEED_DR, 1, scene)
# inputs come from host copies (tracked by initcheck; writes by torch kernels are outside the
# --kernel-name filter and would read as uninitialised)
pose_in = torch.from_numpy(np.random.default_rng(7).standard_normal((101, 7)).astype(np.float32)).cuda()
pose_out = torch.empty_like(pose_in)
vision.dr_pose_augment(vision.pose_params_from_preset(presets.pose_preset()), presets.SEED_DR, 0, pose_in, pose_out)
torch.cuda.synchronize()
print("sanitize paths OK")
