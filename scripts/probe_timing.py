#!/usr/bin/env python
"""A/B probe only (DR_LIB=variants/probe.so, built with -DDR_PROBE_TIMING): per-CTA globaltimer
stamps of the step kernel at config 2 (4,096 envs, cfg-2 layers, CUDA graph of 100 steps) --
entry, ticket, readiness wait, work done, fence, readiness published, end -- read back from the
physics-row buffer the probe build writes them over."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_1906_11633_b200 import DRContext, dr
    from workload import gen, presets
    n = int(os.environ.get("N_ENV", 4096))
    mask = presets.CFG2 if n <= 16384 else presets.FULL
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        ctx = DRContext(presets.preset(mask), n, presets.SEED_DR, stream=s)
        acts, obs = gen.frames(n, 2)
        A, O = torch.from_numpy(acts[0]).cuda(), torch.from_numpy(obs[0]).cuda()
        for _ in range(20):
            ctx.step(A, O)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(100):
                ctx.step(A, O)
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
    t_end = dr.dr_step_index_sync()
    ph = np.ascontiguousarray(ctx.phys()).view(np.uint64).reshape(-1)
    ctx.close()
    G = int(os.environ.get("GRID", (n + 31) // 32 if n <= 16384 else min((n + 127) // 128, 592)))
    a = ph[: 8 * G * 16].reshape(8, G, 16).astype(np.int64)
    print(f"n_env {n} grid {G} last step {t_end - 1}")
    names = ["ticket", "ready-wait", "work", "reduce", "fence+release", "stats+done"]
    steps = [(t_end - 8 + i) for i in range(8)]
    for k in range(6):
        d = np.concatenate([a[t % 8, :, k + 1] - a[t % 8, :, k] for t in steps[1:]])
        print(f"  {names[k]:14s} median {np.median(d):8.0f} ns  p90 {np.percentile(d, 90):8.0f}  max {d.max():8.0f}")
    # step period and per-CTA hand-over: CTA c's start of step t+1 vs its readiness of step t
    per = [(a[(t + 1) % 8, :, 0].min() - a[t % 8, :, 0].min()) for t in steps[1:-1]]
    hand = np.concatenate([a[(t + 1) % 8, :, 2] - a[t % 8, :, 5] for t in steps[1:-1]])
    start = np.concatenate([a[(t + 1) % 8, :, 0] - a[t % 8, :, 5] for t in steps[1:-1]])
    print(f"  step period (first CTA starts) median {np.median(per):.0f} ns")
    print(f"  CTA c: next step's start - this step's ready: median {np.median(start):.0f} ns (negative = started before)")
    print(f"  CTA c: next step's wait done - this step's ready: median {np.median(hand):.0f} ns")
    if n <= 16384:   # latency kernel: each warp role's finish, relative to the readiness wait
        w = np.concatenate([a[t % 8, :, 8:16] - a[t % 8, :, 2:3] for t in steps[1:]])
        print("  per-warp role done after the wait (median ns, warps 0-7):", [int(x) for x in np.median(w, axis=0)])
    span = [a[t % 8, :, 6].max() - a[t % 8, :, 0].min() for t in steps[1:]]
    print(f"  one step's span (first start -> last end) median {np.median(span):.0f} ns")


if __name__ == "__main__":
    main()
