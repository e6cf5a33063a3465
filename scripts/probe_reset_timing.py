#!/usr/bin/env python
"""A/B probe only (DR_LIB=variants/probe.so built with -DDR_PROBE_TIMING): per-CTA globaltimer
stamps of one config-5 reset (1M envs, every 10th env): start, after the grid dependency wait,
after the scan, first / last warp done with its work, end -- distributions over the grid."""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_1906_11633_b200 import DRContext, dr
    from workload import gen, presets
    n = 1 << 20
    ctx = DRContext(presets.preset(presets.FULL | presets.PHYS), n, presets.SEED_DR)
    lib = dr.load()
    lib.dr_debug_probe_read.argtypes = [C.c_void_p, C.c_size_t, C.c_int]
    e = torch.arange(n, device="cuda")
    masks = [((e + t) % 10 == 0).to(torch.uint8) for t in range(10)]
    acts, obs = gen.frames(n, 1)
    A, O = torch.from_numpy(acts[0]).cuda(), torch.from_numpy(obs[0]).cuda()
    for t in range(6):
        ctx.reset(masks[t])
        ctx.step(A, O)
    torch.cuda.synchronize()
    lib.dr_debug_probe_read(None, 0, 1)
    ctx.reset(masks[6])
    torch.cuda.synchronize()
    buf = np.zeros((4096, 8), np.uint64)
    lib.dr_debug_probe_read(buf.ctypes.data, buf.nbytes, 0)
    ctx.close()
    G = int((buf[:, 0] > 0).sum())
    b = buf[:G].astype(np.int64)
    t0 = b[:, 0].min()
    rel = lambda k: (b[:, k] - t0) / 1000.0   # noqa: E731
    print(f"grid {G}, kernel span {(b[:, 3].max() - t0) / 1000:.1f} us")
    for k, name in [(0, "start"), (1, "after wait"), (2, "after scan"), (5, "first warp done"), (4, "last warp done"), (3, "end")]:
        r = rel(k)
        print(f"  {name:16s} min {r.min():7.2f}  median {np.median(r):7.2f}  p90 {np.percentile(r, 90):7.2f}  max {r.max():7.2f} us")
    work = (b[:, 4] - b[:, 2]) / 1000.0
    spread = (b[:, 4] - b[:, 5]) / 1000.0
    print(f"  per-CTA work (scan done -> last warp) median {np.median(work):.2f} us, min {work.min():.2f}, max {work.max():.2f}")
    sm = b[:, 6]
    cnt = np.bincount(sm, minlength=int(sm.max()) + 1)
    print(f"  CTAs per SM: {np.bincount(cnt)} (histogram of counts 0, 1, 2, ...)")
    end_sm = np.array([rel(3)[sm == k].max() if (sm == k).any() else np.nan for k in range(len(cnt))])
    print(f"  per-SM last end: min {np.nanmin(end_sm):.1f} median {np.nanmedian(end_sm):.1f} max {np.nanmax(end_sm):.1f} us")
    for c in sorted(set(cnt[cnt > 0])):
        m = np.isin(sm, np.where(cnt == c)[0])
        print(f"    SMs with {c} CTAs: CTA work median {np.median(work[m]):.1f} us, end median {np.median(rel(3)[m]):.1f}")
    # by SM index halves (the two dies)
    half = len(cnt) // 2
    for lo, hi in ((0, half), (half, len(cnt))):
        m = (sm >= lo) & (sm < hi)
        print(f"    SMs {lo}-{hi - 1}: CTA work median {np.median(work[m]):.1f} us, end median {np.median(rel(3)[m]):.1f}")
    print(f"  per-CTA warp spread (first -> last warp done) median {np.median(spread):.2f} us, max {spread.max():.2f}")


if __name__ == "__main__":
    main()
