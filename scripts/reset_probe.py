#!/usr/bin/env python
"""dr_reset alone at 1M envs (BASELINE config 5's mask pattern): ms per dr_reset with 10 % of envs
resetting and with an empty mask (the fixed cost: launches, list pass, queue drain), CUDA events
around 50 back-to-back resets (DR_LIB selects the build)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_1906_11633_b200 import DRContext
    from workload import presets
    n = 1 << 20
    ctx = DRContext(presets.preset(presets.FULL | presets.PHYS), n, presets.SEED_DR)
    e = torch.arange(n, device="cuda")
    masks = {"10pct": [((e + t) % 10 == 0).to(torch.uint8) for t in range(10)],
             "empty": [torch.zeros(n, dtype=torch.uint8, device="cuda")] * 10}
    s = torch.cuda.current_stream()
    res = {}
    for name, ms in masks.items():
        for t in range(10):
            ctx.reset(ms[t])
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for t in range(50):
            ctx.reset(ms[t % 10])
        b.record(s)
        torch.cuda.synchronize()
        res[name] = a.elapsed_time(b) / 50
    ctx.close()
    print(" ".join(f"{k} {v * 1000:.2f} us" for k, v in res.items()))


if __name__ == "__main__":
    main()
