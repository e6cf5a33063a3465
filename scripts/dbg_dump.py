"""Debug: run a run_pair-like scenario on the GPU and dump outputs + exported states per step."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1906_11633_b200 import DRContext, dr  # noqa: E402
from workload import gen, presets  # noqa: E402

tag, mask, n, T = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
RESET_T = int(os.environ.get("RESET_T", "9"))
P = presets.preset(mask)
acts, obs = gen.frames(n, 20, seed=presets.SEED_WORKLOAD)
A = [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in acts]
O = [torch.from_numpy(np.ascontiguousarray(o)).cuda() for o in obs]
out = {}
with DRContext(P, n, presets.SEED_DR) as ctx:
    for t in range(T):
        if t == RESET_T:
            ctx.reset(torch.from_numpy((np.arange(n) % 3 == 1).astype(np.uint8)).cuda())
        ctx.step(A[t % 20], O[t % 20])
        torch.cuda.synchronize()
        out[f"a{t}"] = ctx.out_actions.cpu().numpy()
        out[f"o{t}"] = ctx.out_obs.cpu().numpy()
        G = ctx.export()
        for k, v in G.items():
            out[f"s{t}_{k}"] = np.array(v)
np.savez(f"gpurun_out/dump_{tag}.npz", **out)
print("dumped", tag)
