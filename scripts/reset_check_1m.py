#!/usr/bin/env python
"""Bit-identity of two libdr builds on BASELINE config 5's reset pattern at full size (1M envs,
every 10th env resetting per step, the bench's masks): python scripts/reset_check_1m.py out.npz
(DR_LIB selects the build) dumps the reset counts of 6 steps, the exported state / records and
physics rows of envs [0, 65536) and of the last 65,536 envs; --compare a.npz b.npz checks them."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def dump(path):
    import torch
    from paper_1906_11633_b200 import DRContext, dr
    from workload import presets
    P = presets.preset(presets.FULL | presets.PHYS)
    n = 1 << 20
    A = torch.zeros(n, 20, device="cuda")
    O = torch.zeros(n, 26, device="cuda")
    O[:, 18] = 1.0
    O[:, 22] = 1.0
    e = torch.arange(n, device="cuda")
    masks = [((e + t) % 10 == 0).to(torch.uint8) for t in range(10)]
    out = {}
    ctx = DRContext(P, n, presets.SEED_DR)
    try:
        for t in range(6):
            ctx.reset(masks[t])
            ctx.step(A, O)
            out[f"stats_{t}"] = np.asarray(ctx.last_stats())
        torch.cuda.synchronize()
        for lo, hi in ((0, 65536), (n - 65536, n)):
            for k, v in ctx.export(lo, hi).items():
                out[f"state_{lo}_{k}"] = np.asarray(v)
            out[f"phys_{lo}"] = np.asarray(ctx.phys(lo, hi))
    finally:
        ctx.close()
    np.savez(path, **out)
    print("resets per step:", [int(out[f"stats_{t}"][10]) for t in range(6)])


if __name__ == "__main__":
    if sys.argv[1] == "--compare":
        A, B = np.load(sys.argv[2]), np.load(sys.argv[3])
        bad = [k for k in A.files if A[k].tobytes() != B[k].tobytes()]
        print(f"{len(A.files)} arrays, {len(bad)} differ" + (f": {bad[:8]}" if bad else " (bit-identical)"))
        sys.exit(1 if bad else 0)
    dump(sys.argv[1])
