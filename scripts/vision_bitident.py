#!/usr/bin/env python
"""Bit identity of two builds' image augmentation (DR_LIB selects the build): the paper's batch
(192 images of 200x200x3) and a ragged batch (5 images of 17x13x3), outputs and image stats.
python scripts/vision_bitident.py out.npz | --compare a.npz b.npz"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def dump(path):
    import torch
    from paper_1906_11633_b200 import vision
    from workload import gen, presets
    P = vision.params_from_preset(presets.vision_preset())
    out = {}
    for name, shape, batch in (("paper", (192, 200, 200, 3), 3), ("ragged", (5, 17, 13, 3), 4)):
        x = torch.from_numpy(gen.images(*shape, seed=7)).cuda()
        y = torch.empty(x.shape, dtype=torch.float32, device="cuda")
        st = torch.empty(shape[0], 4, dtype=torch.float32, device="cuda")
        vision.dr_image_augment(P, presets.SEED_DR, batch, x, y, st)
        torch.cuda.synchronize()
        out[name] = y.cpu().numpy()
        out[name + "_stats"] = st.cpu().numpy()
    np.savez(path, **out)


if __name__ == "__main__":
    if sys.argv[1] == "--compare":
        A, B = np.load(sys.argv[2]), np.load(sys.argv[3])
        bad = [k for k in A.files if A[k].tobytes() != B[k].tobytes()]
        print(f"{len(A.files)} arrays, {len(bad)} differ" + (f": {bad}" if bad else " (bit-identical)"))
        sys.exit(1 if bad else 0)
    dump(sys.argv[1])
