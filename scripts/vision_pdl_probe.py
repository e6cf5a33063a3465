#!/usr/bin/env python
"""A/B probe: back-to-back dr_image_augment calls (192 images of 200x200x3, a 4-batch ring, no
scene draws, no events between launches), us per batch (DR_LIB selects the build)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_1906_11633_b200 import vision
    from workload import gen, presets
    NI, H, W, C = 192, presets.VISION_H, presets.VISION_W, presets.VISION_C
    P = vision.params_from_preset(presets.vision_preset())
    s = torch.cuda.Stream()
    X = [torch.from_numpy(gen.images(NI, H, W, C, seed=11 + k)).cuda() for k in range(4)]
    Y = [torch.empty(NI, H, W, C, dtype=torch.float32, device="cuda") for _ in range(4)]
    ST = [torch.empty(NI, 4, dtype=torch.float32, device="cuda") for _ in range(4)]
    torch.cuda.synchronize()
    res = []
    for rep in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for t in range(50):
            vision.dr_image_augment(P, presets.SEED_DR, t, X[t % 4], Y[t % 4], ST[t % 4], stream=s)
        a.record(s)
        for t in range(500):
            vision.dr_image_augment(P, presets.SEED_DR, t, X[t % 4], Y[t % 4], ST[t % 4], stream=s)
        b.record(s)
        torch.cuda.synchronize()
        res.append(a.elapsed_time(b) / 500 * 1000)
    print("us per batch:", " ".join(f"{x:.2f}" for x in res))


if __name__ == "__main__":
    main()
