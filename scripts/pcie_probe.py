"""PCIe ceiling for bench.py's e2e leg: pinned H2D of one step's inputs (193 MB at 1M envs), D2H of
its outputs (231 MB), alone and concurrently on two streams (the dr_step_host overlap)."""
import json
import torch

n = 1 << 20
hb, db = n * 46 * 4, n * 55 * 4
h_in = torch.empty(hb // 4).pin_memory()
h_out = torch.empty(db // 4).pin_memory()
d_in = torch.empty(hb // 4, device="cuda")
d_out = torch.empty(db // 4, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    s1.wait_stream(torch.cuda.current_stream())
    s2.wait_stream(torch.cuda.current_stream())
    for _ in range(reps):
        fn()
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def h2d():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)


def both():
    h2d()
    d2h()


t_h = timed(h2d)
t_d = timed(d2h)
t_b = timed(both)
print(json.dumps({"h2d_GBps": hb / t_h / 1e6, "d2h_GBps": db / t_d / 1e6, "h2d_ms": t_h, "d2h_ms": t_d,
                  "both_ms": t_b, "e2e_bound_env_steps_per_s": n / (t_b / 1e3)}))
