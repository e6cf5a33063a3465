#!/usr/bin/env python
"""Vision timing probe: where the bench step's time goes beyond the augment kernel.  Back-to-back
dr_image_augment launches of the paper's 192-image batch over bench.py's 4-batch ring, then the
same with one piece of the bench step added at a time (img_stats output, a timing event per step,
the 64 scene draws on a side stream with a per-step fork/join, the scene draws on the same stream)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1906_11633_b200 import vision  # noqa: E402
from workload import gen, presets  # noqa: E402

NI, H, W, C, S = 192, 200, 200, 3, 64
P = vision.params_from_preset(presets.vision_preset())
X = [torch.from_numpy(gen.images(NI, H, W, C, seed=k)).cuda() for k in range(4)]
Y = [torch.empty(NI, H, W, C, dtype=torch.float32, device="cuda") for _ in range(4)]
ST = torch.empty(NI, 4, dtype=torch.float32, device="cuda")
SC = torch.empty(S, 64, dtype=torch.float32, device="cuda")
s, side = torch.cuda.Stream(), torch.cuda.Stream()


def run(stats, events, scene):
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(1001)] if events else None

    def step(t):
        if scene == "side":
            f = torch.cuda.Event()
            f.record(s)
            side.wait_event(f)
            vision.dr_scene_draw_batch(P, 1, t, SC, stream=side)
        elif scene == "same":
            vision.dr_scene_draw_batch(P, 1, t, SC, stream=s)
        vision.dr_image_augment(P, 1, t, X[t % 4], Y[t % 4], ST if stats else None, stream=s)
        if scene == "side":
            j = torch.cuda.Event()
            j.record(side)
            s.wait_event(j)

    with torch.cuda.stream(s):
        for t in range(50):
            step(t)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        K = 1000
        e0.record(s)
        for t in range(K):
            step(t)
            if events:
                evs[t].record(s)
        e1.record(s)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / K * 1e3


for args in [(False, False, None), (True, False, None), (True, True, None), (True, False, "side"),
             (True, True, "side"), (True, False, "same")]:
    print(f"stats={args[0]} events={args[1]} scene={args[2]}: {run(*args):.2f} us per step")
