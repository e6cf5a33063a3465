#!/usr/bin/env python
"""Bit-identity check between two libdr builds (A/B refactors that must not change a single bit):
python scripts/bitident.py <dump.npz>  runs 12 steps of 4,096 envs (all layers + PHYS, resets every
3rd step, both step kernels via DR_STEP_MODE) with the library DR_LIB selects and saves every output,
the exported state and the physics rows; --compare a.npz b.npz checks them bit for bit."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def dump(path):
    import torch
    from paper_1906_11633_b200 import DRContext
    from workload import gen, presets
    P = presets.preset(presets.FULL | presets.PHYS)
    n = 4096
    acts, obs = gen.frames(n, 4)
    A = [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in acts]
    O = [torch.from_numpy(np.ascontiguousarray(o)).cuda() for o in obs]
    out = {}
    ctx = DRContext(P, n, presets.SEED_DR)
    try:
        for t in range(12):
            if t % 3 == 2:
                ctx.reset(torch.from_numpy(gen.reset_mask_ring(n, t, 4)).cuda())
            ctx.step(A[t % 4], O[t % 4])
            for k in ("out_actions", "out_obs", "out_dt", "out_force"):
                out[f"{k}_{t}"] = getattr(ctx, k).cpu().numpy().copy()
        torch.cuda.synchronize()
        for k, v in ctx.export().items():
            out[f"state_{k}"] = np.asarray(v)
        out["phys"] = ctx.phys()
        out["stats"] = np.asarray(ctx.last_stats())
    finally:
        ctx.close()
    np.savez(path, **out)


def compare(a, b):
    A, B = np.load(a), np.load(b)
    bad = [k for k in A.files if A[k].tobytes() != B[k].tobytes()]
    print(f"{len(A.files)} arrays, {len(bad)} differ" + (f": {bad[:8]}" if bad else " (bit-identical)"))
    return not bad


if __name__ == "__main__":
    if sys.argv[1] == "--compare":
        sys.exit(0 if compare(sys.argv[2], sys.argv[3]) else 1)
    dump(sys.argv[1])
