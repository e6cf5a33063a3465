#!/usr/bin/env python
"""bench.py -- randomized env-steps/s of the fused DR step on B200 (BASELINE.json metric).

Default workload (N=1): BASELINE config 4's single-GPU reference -- 1,048,576 envs, full
pipeline (all 9 layers), Shadow-hand shapes.  Under torchrun the envs are sharded by global id
(env_offset = offset of the rank's shard, same seed): by default the 1M envs of config 4 are split
over the N ranks ("strong", config 4's "1M envs sharded 2/4/8"); --scaling weak gives every rank
1M envs.  The per-step NCCL all-reduce of the 32 x fp64 stats vector runs on a comm stream -- the
path's one collective -- and for N > 1 the steps and their all-reduces are
captured in CUDA graphs of 100 steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config full1m|cfg2|cfg3|reset]
  python bench.py --impl reference ...   # the fp64 CPU oracle on the box's host cores

One JSON line on rank 0.  `value` = env-steps/s over all ranks with inputs resident in HBM
(CUDA events on the library stream, max over ranks); `e2e` = the same metric through
dr_step_host with pinned host buffers (H2D of inputs + D2H of all outputs inside the timed
region); `roofline` for the step kernel; `cpu_baseline` = the oracle on a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_GLOBAL_1M = 1 << 20
# algorithmic bytes per env-step: inputs + outputs + episode record read
# + state read/write, for the layer sets the configs use
BYTES_FULL = 184 + 220 + 344 + 480
ST_BYTES_PER_ENV = 80 * 4   # state planes per env (dr_internal.h ST_PLANES)
BYTES_CFG2 = 184 + 220 + 332 + 160 + 4   # + the flags word (FRESH marker) read per step


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="full1m", choices=["full1m", "cfg2", "cfg3", "reset", "vision"])
    ap.add_argument("--n-env", type=int, default=0, help="override the env count (per GPU if weak, global if strong)")
    ap.add_argument("--scaling", default="strong", choices=["weak", "strong"],
                    help="strong (default): the config's env count is split over the ranks (BASELINE config 4: "
                         "1M envs sharded over 2 / 4 / 8 GPUs); weak: every rank owns the config's env count")
    ap.add_argument("--e2e-steps", type=int, default=30)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-envs", type=int, default=65536)
    ap.add_argument("--cpu-sample-steps", type=int, default=24)
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no e2e/cpu legs)")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend for N > 1 (gloo: tests that run several ranks on one GPU)")
    ap.add_argument("--graph", type=int, default=-1,
                    help="steps per CUDA graph in the timed region (0 = eager launches; default: 100 for the "
                         "launch-bound small configs at N=1 and for every N > 1 run over NCCL, else 0)")
    return ap.parse_args()


# per resetting env: phys row, the 89 record words (written as 12 whole 32-byte groups = 384 B), the
# FRESH flag and the episode-counter read
RESET_BYTES = 1024 + 356 + 4 + 4


def config_of(name, n_override):
    from workload import presets
    if name == "full1m":
        return dict(workload="cfg4-1M-envs-full-pipeline", mask=presets.FULL, n=n_override or N_GLOBAL_1M,
                    bytes=BYTES_FULL, scaling="strong", resets=False)
    if name == "cfg2":
        return dict(workload="cfg2-4096-envs-backlash+act/obs-noise", mask=presets.CFG2, n=n_override or 4096,
                    bytes=BYTES_CFG2, scaling="strong", resets=False)
    if name == "cfg3":
        return dict(workload="cfg3-65536-envs-full-pipeline", mask=presets.FULL, n=n_override or 65536,
                    bytes=BYTES_FULL, scaling="strong", resets=False)
    return dict(workload="cfg5-1M-envs-10pct-resets-per-step", mask=presets.FULL, n=n_override or N_GLOBAL_1M,
                bytes=BYTES_FULL, scaling="strong", resets=True)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons every 20 ms, each sample stamped with the host clock.
    The bench runs a >= 1 s pre-roll at the timed load with the sampler on (short timed regions,
    e.g. --steps 20 at 0.2 ms, are shorter than any sampling interval) and keeps it on through the
    timed region; the report says how many samples fell inside the timed window itself."""

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []
        self.window = None

    def start(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.monotonic(), line.strip()))

    def mark_timed(self, t0, t1):
        self.window = (t0, t1)

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.05)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        time.sleep(0.05)
        sm, mx, reasons, in_timed = [], None, set(), 0
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ts, ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            if self.window and self.window[0] <= ts <= self.window[1] + 0.025:
                in_timed += 1
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        sm.sort()
        med = sm[len(sm) // 2] if sm else None
        return {"sm_mhz": med, "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm),
                "samples_in_timed_window": in_timed, "interval_ms": 20,
                "coverage": ">= 1 s pre-roll at the timed load + the timed region"}


def host_cpu():
    """(logical cores, CPU model) of this host."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return os.cpu_count(), model


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def mix_ceiling(mix, achieved):
    """The HBM ceiling of a kernel's own read/write mix (profiles/bw_ceiling.json, measured by
    scripts/bw_ceiling.cu on a B200): a second denominator beside the copy peak, or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "bw_ceiling.json")) as f:
            d = json.load(f)[mix]
        return {"gbs": d["gbs"], "frac": achieved / d["gbs"], "mix": d["mix"],
                "source": "profiles/bw_ceiling.json (scripts/bw_ceiling.cu, PDL, back to back)"}
    except Exception:
        return None


def ncu_traffic(workload):
    """Per-launch dram bytes of a kernel from the committed ncu summary (profiles/ncu_step_summary.json:
    the step kernel per workload, the reset kernel under "cfg5-reset-kernel"), if any."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_step_summary.json")) as f:
            d = json.load(f)
        return d.get(workload, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


def ncu_entry(workload):
    """The committed ncu summary entry of a workload (profiles/ncu_step_summary.json), or {}."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_step_summary.json")) as f:
            return json.load(f).get(workload, {})
    except Exception:
        return {}


def run_reference(args):
    """--impl reference: the fp64 CPU oracle, as it stands, on this box's host cores (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import numpy as np
    from oracle.oracle import Oracle
    from workload import gen, presets
    if args.config == "vision":
        from oracle import oracle as O
        k = max(1, min(args.steps, 8))
        imgs = gen.images(k, presets.VISION_H, presets.VISION_W, presets.VISION_C)
        t0 = time.perf_counter()
        O.image_augment(presets.vision_preset(), presets.SEED_DR, 0, imgs)
        dt = time.perf_counter() - t0
        v = k / dt
        print(json.dumps({"impl": "reference", "metric": "augmented images/sec", "value": v, "unit": "images/s",
                          "n_gpus": args.gpus, "steps": k, "warmup": 0, "ms_per_step": dt / k * 1e3,
                          "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                          "data": "synthetic", "config": {"workload": "vision-200x200x3 images (oracle sample)"},
                          "cpu_baseline": {"value": v, "unit": "images/s", "cores": 1, "kind": "oracle",
                                           "sample": f"{k} images of 200x200x3 (fp64 oracle, single thread)"},
                          "e2e": {"value": v, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}),
              flush=True)
        return
    cfg = config_of(args.config, args.n_env)
    cfg["scaling"] = args.scaling
    cores, model = host_cpu()
    # the oracle as it stands, all host cores (the -fopenmp build: OpenMP over envs), a bounded
    # sample of the workload per step so the whole --steps K --warmup W run takes a few minutes
    n = min(cfg["n"], args.cpu_sample_envs)
    P = presets.preset(cfg["mask"])
    acts, obs = gen.frames(n, 4)
    orc = Oracle(P, n, presets.SEED_DR, omp=True)
    for t in range(args.warmup):
        orc.step(acts[t % 4], obs[t % 4])
    steps = max(1, min(args.steps, args.cpu_sample_steps))
    t0 = time.perf_counter()
    for t in range(steps):
        if cfg["resets"]:
            orc.reset(gen.reset_mask_ring(n, t))
        orc.step(acts[t % 4], obs[t % 4])
    dt = time.perf_counter() - t0
    v = n * steps / dt
    line = {"impl": "reference", "metric": "randomized env-steps/sec", "value": v, "unit": "env-steps/s",
            "n_gpus": args.gpus, "steps": steps, "warmup": args.warmup, "ms_per_step": dt / steps * 1e3,
            "higher_is_better": True, "scaling": cfg["scaling"], "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": cfg["workload"], "n_env_sample": n, "layers": hex(cfg["mask"])},
            "cpu_baseline": {"value": v, "unit": "env-steps/s", "cores": cores, "kind": "oracle", "cpu_model": model,
                             "sample": f"{n} envs x {steps} steps of {cfg['workload']} (fp64 oracle, OpenMP over envs)"},
            "e2e": {"value": v, "unit": "env-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _oracle_rate(cfg, n, steps, omp):
    """env-steps/s of the fp64 oracle (single-thread or -fopenmp build) on n envs x steps."""
    from oracle.oracle import Oracle
    from workload import gen, presets
    P = presets.preset(cfg["mask"])
    acts, obs = gen.frames(n, 4)
    orc = Oracle(P, n, presets.SEED_DR, omp=omp)
    orc.step(acts[0], obs[0])   # first touch
    t0 = time.perf_counter()
    for t in range(steps):
        if cfg["resets"]:
            orc.reset(gen.reset_mask_ring(n, t))
        orc.step(acts[t % 4], obs[t % 4])
    dt = time.perf_counter() - t0
    orc.close()
    return n * steps / dt, dt


def cpu_baseline(cfg, args):
    """The oracle as it stands on this host: single thread (liboracle.so) and all cores (the same
    source built with -fopenmp, parallel over envs; bit-identical results).  Bounded samples:
    ~10 s single-thread, ~10 s all-core.  `value` is the all-core rate (the paper's DR ran on CPU
    workers, so all cores is the honest CPU comparison)."""
    cores, model = host_cpu()
    n = min(cfg["n"], args.cpu_sample_envs)
    v1, _ = _oracle_rate(cfg, n, args.cpu_sample_steps, omp=False)
    na = n
    probe, dtp = _oracle_rate(cfg, na, 2, omp=True)
    steps_all = max(2, min(200, int(10.0 / max(dtp / 2, 1e-6))))
    va, _ = _oracle_rate(cfg, na, steps_all, omp=True)
    return {"value": va, "unit": "env-steps/s", "cores": cores, "kind": "oracle", "cpu_model": model,
            "sample": f"all cores: {na} envs x {steps_all} steps of {cfg['workload']} (fp64 oracle, OpenMP over envs); "
                      f"single thread: {n} envs x {args.cpu_sample_steps} steps",
            "single_thread": {"value": v1, "unit": "env-steps/s", "cores": 1}}


def run_vision(args):
    """--config vision: one step = the appearance draws of the paper's
    batch of 64 samples + the post-render augmentation of its 192 camera images (200 x 200 x 3
    u8), per rank.  A ring of 4 distinct input/output batches (92 MB in, 368 MB out)
    keeps the working set above L2.  Metric: augmented images/s."""
    import torch
    import torch.distributed as dist
    from paper_1906_11633_b200 import vision
    from workload import gen, presets

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    S, NI, H, W, Cc = presets.VISION_BATCH_SAMPLES, presets.VISION_BATCH_SAMPLES * presets.VISION_CAMERAS, \
        presets.VISION_H, presets.VISION_W, presets.VISION_C
    E = H * W * Cc
    R = 4
    P = vision.params_from_preset(presets.vision_preset())
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        host = [gen.images(NI, H, W, Cc, seed=presets.SEED_WORKLOAD + 101 * rank + k) for k in range(R)]
        X = [torch.from_numpy(h).cuda() for h in host]
        Y = [torch.empty(NI, H, W, Cc, dtype=torch.float32, device="cuda") for _ in range(R)]
        ST = [torch.empty(NI, 4, dtype=torch.float32, device="cuda") for _ in range(R)]   # per-batch image stats
        SC = torch.empty(S, 64, dtype=torch.float32, device="cuda")
        torch.cuda.synchronize()

        side = torch.cuda.Stream()

        def one_step(t):
            # batch index b = t: fresh draws every step; images of rank r have global ids r * NI + i.
            # The 64 scene draws (latency-bound, independent of the images) run on a side stream,
            # forked from the step stream and joined back into it once per run of steps (fork() /
            # join()), so consecutive augmentations stay adjacent on their stream: a batch's
            # clusters read their images while the previous batch is still writing (programmatic
            # dependent launch; an event between two launches breaks that overlap).
            b = t
            vision.dr_scene_draw_batch(P, presets.SEED_DR, b, SC, sample_offset=rank * S, stream=side)
            vision.dr_image_augment(P, presets.SEED_DR, b, X[t % R], Y[t % R], ST[t % R], image_offset=rank * NI,
                                    stream=stream)

        def fork():
            ev = torch.cuda.Event()
            ev.record(stream)
            side.wait_event(ev)

        def join():
            ev = torch.cuda.Event()
            ev.record(side)
            stream.wait_event(ev)

        fork()
        for t in range(args.warmup):
            one_step(t)
        join()
        torch.cuda.synchronize()
        sampler = ClockSampler(local)
        sampler.start()
        w0 = time.perf_counter()   # >= 1 s pre-roll at the timed load (clock coverage, see ClockSampler)
        t_base = args.warmup
        while True:
            fork()
            for _ in range(20):
                one_step(t_base)
                t_base += 1
            join()
            torch.cuda.synchronize()
            if time.perf_counter() - w0 >= 1.0:
                break
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        l0 = vision.dr_total_kernel_launches()
        # events at the two ends only (an event between two launches costs ~2 us per step:
        # scripts/vision_probe.py)
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        h0 = time.monotonic()
        evs[0].record(stream)
        fork()
        for i in range(args.steps):
            one_step(t_base + i)
        join()
        evs[1].record(stream)
        torch.cuda.synchronize()
        sampler.mark_timed(h0, time.monotonic())
        if world > 1:
            dist.barrier()
        launches = vision.dr_total_kernel_launches() - l0
        clocks = sampler.stop()
        elapsed_ms = evs[0].elapsed_time(evs[-1])
        per = [elapsed_ms / args.steps]
        t_ms = torch.tensor([elapsed_ms], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t_ms, op=dist.ReduceOp.MAX)
        elapsed_ms = float(t_ms.item())
        # e2e: pinned host u8 batch -> device -> augment -> fp32 result back to pinned host memory
        e2e = None
        if not args.profile and args.e2e_steps > 0:
            # pipelined like dr_step_host: step i's upload (copy stream 1) overlaps step i-1's download
            # (copy stream 2) and compute; two device buffer sets, ordered by events
            hx = torch.from_numpy(host[0]).pin_memory()
            hy = [torch.empty(NI, H, W, Cc, dtype=torch.float32).pin_memory() for _ in range(2)]
            s_up, s_down = torch.cuda.Stream(), torch.cuda.Stream()
            ev_up = [torch.cuda.Event() for _ in range(2)]
            ev_aug = [torch.cuda.Event() for _ in range(2)]
            ev_down = [torch.cuda.Event() for _ in range(2)]
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for i in range(args.e2e_steps):
                b = i & 1
                if i >= 2:
                    s_up.wait_event(ev_aug[b])      # step i-2's augment has read X[b]
                with torch.cuda.stream(s_up):
                    X[b].copy_(hx, non_blocking=True)
                ev_up[b].record(s_up)
                stream.wait_event(ev_up[b])
                if i >= 2:
                    stream.wait_event(ev_down[b])   # step i-2's download has read Y[b]
                vision.dr_scene_draw_batch(P, presets.SEED_DR, i, SC, sample_offset=rank * S, stream=stream)
                vision.dr_image_augment(P, presets.SEED_DR, i, X[b], Y[b], ST[b], image_offset=rank * NI, stream=stream)
                ev_aug[b].record(stream)
                s_down.wait_event(ev_aug[b])
                with torch.cuda.stream(s_down):
                    hy[b].copy_(Y[b], non_blocking=True)
                ev_down[b].record(s_down)
            torch.cuda.synchronize()
            e2e_s = time.perf_counter() - t0
            te = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
            if world > 1:
                dist.all_reduce(te, op=dist.ReduceOp.MAX)
            e2e = {"value": world * NI * args.e2e_steps / float(te.item()), "unit": "images/s",
                   "h2d_bytes_per_step": world * NI * E, "d2h_bytes_per_step": world * NI * E * 4,
                   "api": "dr_image_augment (pinned host u8 in, fp32 out; uploads / downloads on two copy streams)",
                   "steps": args.e2e_steps}
    value = world * NI * args.steps / (elapsed_ms / 1e3)
    kern_ms = sum(per) / len(per)
    peak, peak_kind = measured_peak()
    bytes_step = NI * E * 5 + S * 256
    achieved = bytes_step / (kern_ms / 1e3) / 1e9
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline and not args.profile:
            from oracle import oracle as O
            k = 8
            t0 = time.perf_counter()
            O.image_augment(presets.vision_preset(), presets.SEED_DR, 0, host[0][:k])
            O.scene_draw(presets.vision_preset(), presets.SEED_DR, 0, S)
            dt = time.perf_counter() - t0
            cpu = {"value": k / dt, "unit": "images/s", "cores": 1, "kind": "oracle",
                   "sample": f"{k} images of 200x200x3 + {S} scene draws (fp64 oracle, single thread)"}
        line = {"metric": "augmented images/sec", "value": value, "unit": "images/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8->f32",
                "data": "synthetic",
                "config": {"workload": "vision-192x200x200x3-per-rank (64 samples x 3 cameras, PAPER.md:290)",
                           "images_per_step_per_gpu": NI, "scene_draws_per_step_per_gpu": S,
                           "l2": "4-batch ring, 460 MB working set > L2"},
                "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                             "frac": achieved / peak, "traffic": None, "peak_kind": peak_kind,
                             "bytes_per_step": bytes_step, "kernel": "dr::image_augment_kernel (+ scene_draw_kernel)",
                             "kernel_ms_avg": kern_ms, "kernel_ms_median": per[len(per) // 2],
                             "mix_ceiling": mix_ceiling("vision_1r_4w", achieved)},
                "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches), "clocks": clocks}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.config == "vision" and args.impl != "reference":
        return run_vision(args)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    from paper_1906_11633_b200 import DRContext, dr
    from workload import presets

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    local = local % torch.cuda.device_count()   # several ranks may share a GPU in tests (gloo)
    torch.cuda.set_device(local)
    if world > 1:
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    cfg = config_of(args.config, args.n_env)
    cfg["scaling"] = args.scaling
    n_glob = cfg["n"] * world if args.scaling == "weak" else cfg["n"]
    from paper_1906_11633_b200.parallel import StatsReducer, shard
    off, n = shard(n_glob, world, rank)
    P = presets.preset(cfg["mask"])

    lib_stream = torch.cuda.Stream()
    with torch.cuda.stream(lib_stream):
        ctx = DRContext(P, n, presets.SEED_DR, env_offset=off, n_env_global=n_glob, stream=lib_stream)
        # synthetic device-resident frame ring (4 frames), Shadow-hand shapes (workload.gen recipe)
        F = 4
        g = torch.Generator(device="cuda").manual_seed(presets.SEED_WORKLOAD + rank)
        k = torch.randint(0, 11, (F, n, 20), device="cuda", generator=g)
        A = (-1.0 + (2.0 * k + 1.0) / 11.0).float().contiguous()
        del k
        O = torch.empty(F, n, 26, device="cuda")
        from workload.gen import TIP_NOMINAL, OBJ_NOMINAL, TIP_JITTER, OBJ_JITTER
        O[:, :, 0:15] = torch.tensor(TIP_NOMINAL.reshape(-1), device="cuda", dtype=torch.float32) + \
            TIP_JITTER * torch.randn(F, n, 15, device="cuda", generator=g)
        O[:, :, 15:18] = torch.tensor(OBJ_NOMINAL, device="cuda", dtype=torch.float32) + \
            OBJ_JITTER * torch.randn(F, n, 3, device="cuda", generator=g)
        q = torch.randn(F, n, 8, device="cuda", generator=g)
        O[:, :, 18:22] = q[..., 0:4] / q[..., 0:4].norm(dim=-1, keepdim=True)
        O[:, :, 22:26] = q[..., 4:8] / q[..., 4:8].norm(dim=-1, keepdim=True)
        del q
        reducer = StatsReducer(ctx.stats, lib_stream) if world > 1 else None
        masks = None
        if cfg["resets"]:
            e = torch.arange(off, off + n, device="cuda")
            masks = [((e + t) % 10 == 0).to(torch.uint8) for t in range(10)]
        torch.cuda.synchronize()

    def one_step(t, mid=None):
        if reducer is not None:
            reducer.before_step(t)   # the all-reduce of step t-3 is done before step t clears its slot
        if masks is not None:
            ctx.reset(masks[t % 10])
            if mid is not None:
                mid.record(lib_stream)   # between dr_reset and dr_step: the two kernels' shares
        ctx.step(A[t % F], O[t % F])
        if reducer is not None:
            # the path's one collective: sum of the 32 x fp64 stats of step t over ranks,
            # on its own stream so it overlaps the next steps (stats slots form a ring of 4)
            reducer.after_step(t)

    with torch.cuda.stream(lib_stream):
        for t in range(args.warmup):
            one_step(t)
        torch.cuda.synchronize()
        # pre-roll at the timed load for >= 1 s with the clock sampler on (the timed region of a
        # short --steps run is shorter than nvidia-smi's sampling interval)
        sampler = ClockSampler(local)
        sampler.start()
        w0 = time.perf_counter()
        t_next = args.warmup
        while True:
            for _ in range(10):
                one_step(t_next)
                t_next += 1
            torch.cuda.synchronize()
            if time.perf_counter() - w0 >= 1.0:
                break
        t_base = t_next
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        launches0 = dr.dr_kernel_launches()
        # CUDA graphs of G steps: the launch-bound small configs at N = 1, and every N > 1 run over NCCL
        # (the step kernels and the per-step stats all-reduce of the comm stream captured together, so
        # no rank's host issues a launch or a collective per step)
        graphable = world == 1 or args.backend == "nccl"
        G = args.graph if args.graph >= 0 else (100 if (graphable and (world > 1 or n * cfg["bytes"] < 2e8)) else 0)
        if G > 0 and (not graphable or args.steps % G or (cfg["resets"] and G % 10)):
            G = 0   # graphs need K % G == 0 (and whole 10-step reset-mask cycles); gloo cannot be captured
        if G > 0:
            # launch-bound configs: one CUDA graph of G steps (the step index is device-resident, so
            # every replay advances it); events around each replay, per-step time = replay / G.
            # Inside the capture the reducer only waits for all-reduces of the same graph: the graph
            # ends by joining the comm stream, so the previous replay's all-reduces are complete.
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=lib_stream):
                if reducer is not None:
                    reducer.reset_ring()
                for i in range(G):
                    one_step(t_base + i)
                if reducer is not None:
                    reducer.sync()
            per_graph_launches = dr.dr_kernel_launches() - launches0
            graph.replay()   # warm replay
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            reps = args.steps // G
            evs = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
            h0 = time.monotonic()
            evs[0].record(lib_stream)
            for i in range(reps):
                graph.replay()
                evs[i + 1].record(lib_stream)
        else:
            # events only at the two ends: an event recorded between two launches makes the second
            # wait for the first to drain and costs ~2 us per step (it also stops chained steps from
            # overlapping); the reset / step split comes from a separate pass below
            evs = [torch.cuda.Event(enable_timing=True)]
            h0 = time.monotonic()
            evs[0].record(lib_stream)
            for i in range(args.steps):
                one_step(t_base + i)
        if reducer is not None:
            reducer.sync()
        end = torch.cuda.Event(enable_timing=True)
        end.record(lib_stream)
        torch.cuda.synchronize()
        sampler.mark_timed(h0, time.monotonic())
        if world > 1:
            dist.barrier()
        launches = per_graph_launches * reps if G > 0 else dr.dr_kernel_launches() - launches0
        clocks = sampler.stop()
        elapsed_ms = evs[0].elapsed_time(end)
        if G > 0:
            per = [evs[i].elapsed_time(evs[i + 1]) / G for i in range(len(evs) - 1)]
        else:
            per = [elapsed_ms / args.steps]
        t_ms = torch.tensor([elapsed_ms], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t_ms, op=dist.ReduceOp.MAX)
        elapsed_ms = float(t_ms.item())
        stats = ctx.last_stats()
        r_ms = s_ms = None
        if cfg["resets"] and G == 0:
            # diagnostic pass after the timed region (not part of value): events around each dr_reset
            # and dr_step give the two kernels' shares of a step
            D = min(args.steps, 50)
            ev_a = [torch.cuda.Event(enable_timing=True) for _ in range(D + 1)]
            ev_m = [torch.cuda.Event(enable_timing=True) for _ in range(D)]
            ev_a[0].record(lib_stream)
            for i in range(D):
                one_step(t_base + args.steps + i, ev_m[i])
                ev_a[i + 1].record(lib_stream)
            torch.cuda.synchronize()
            r_ms = [ev_a[i].elapsed_time(ev_m[i]) for i in range(D)]
            s_ms = [ev_m[i].elapsed_time(ev_a[i + 1]) for i in range(D)]
        cold = None
        l2_bytes = int(getattr(torch.cuda.get_device_properties(torch.cuda.current_device()), "L2_cache_size", 0) or 0)
        if not cfg["resets"] and l2_bytes and n * (384 + ST_BYTES_PER_ENV + 4 * 184 + 220) <= 1.25 * l2_bytes:
            # cold-L2 diagnostic (not part of value; SURVEY §8(d) "report warm and cold" for the
            # L2-borderline configs): each step preceded by a write of 2x the L2 size, events around
            # the step alone
            with torch.cuda.stream(lib_stream):
                flush = torch.empty(2 * l2_bytes // 4, dtype=torch.float32, device="cuda")
                D = 30
                ev_c = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(D)]
                for i in range(D):
                    flush.fill_(float(i))
                    ev_c[i][0].record(lib_stream)
                    one_step(t_base + args.steps + i)
                    ev_c[i][1].record(lib_stream)
                torch.cuda.synchronize()
                c_ms = sorted(a.elapsed_time(b) for a, b in ev_c)
                del flush
            cold = {"ms_per_step_median": c_ms[D // 2], "value": n_glob / (c_ms[D // 2] / 1e3),
                    "method": "each step after a 2x-L2 write, CUDA events around the step, median of 30"}

    value = n_glob * args.steps / (elapsed_ms / 1e3)
    split = None
    if r_ms:
        # dr_reset and dr_step launch times from the diagnostic pass (events around each)
        r_avg = sum(r_ms) / len(r_ms)
        # the reset kernel on its own: algorithmic bytes (1,392 B per resetting env + the 1-byte mask of
        # every env) over its own launch time, and ncu's DRAM bytes per launch against them
        r_bytes = (n // 10) * RESET_BYTES + n
        r_traffic = ncu_traffic("cfg5-reset-kernel")
        r_gbs = r_bytes / (r_avg / 1e3) / 1e9
        split = {"reset_ms_avg": r_avg, "step_ms_avg": sum(s_ms) / len(s_ms),
                 "resets_per_step": n // 10, "resets_per_s": (n // 10) / (r_avg / 1e3), "reset_bytes_per_env": RESET_BYTES,
                 "reset": {"bound": "issue", "achieved": r_gbs, "unit": "GB/s", "frac_of_hbm": r_gbs / measured_peak()[0],
                           "algorithmic_bytes": r_bytes, "traffic": r_traffic,
                           "traffic_over_algorithmic": (r_traffic / r_bytes) if r_traffic else None}}
        # the reset's own roofline is instruction issue: one warp-instruction per cycle per SM
        # sub-partition (4 per SM, B300_MICROARCH.md), at the SM clock sampled under load; the
        # warp-instructions per launch come from the committed ncu capture of the same kernel
        w_inst = ncu_entry("cfg5-reset-kernel").get("warp_instructions")
        if w_inst:
            n_sm = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
            mhz = clocks.get("sm_mhz") or clocks.get("sm_max_mhz") if isinstance(clocks, dict) else None
            if mhz:
                peak_ips = 4 * n_sm * mhz * 1e6
                ach = w_inst / (r_avg / 1e3)
                split["reset"]["issue"] = {"warp_instructions_per_launch": w_inst, "achieved": ach, "peak": peak_ips,
                                           "unit": "warp-instructions/s", "frac": ach / peak_ips, "sm_mhz": mhz,
                                           "peak_basis": "1 warp-instruction / cycle / SM sub-partition x 4 x SMs x sampled SM clock"}
    per.sort()
    kern_ms = sum(per) / len(per)
    peak, peak_kind = measured_peak()
    # algorithmic bytes per step: the step's 1228 B per env, plus (reset config) 1,384 B per
    # resetting env (phys row 1024 + record 356 + FRESH flag 4) and the 1-byte mask per env
    bytes_step = cfg["bytes"] * n + ((n // 10) * RESET_BYTES + n if cfg["resets"] else 0)
    achieved = bytes_step / (kern_ms / 1e3) / 1e9
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": None if cfg["resets"] else ncu_traffic(cfg["workload"]), "peak_kind": peak_kind,
                "bytes_per_env_step": bytes_step / n, "kernel": "dr::step_kernel_warp" + (" + dr::reset_kernel (one step = dr_reset + dr_step)" if cfg["resets"] else ""),
                "kernel_ms_avg": kern_ms, "kernel_ms_median": per[len(per) // 2]}
    if split:
        roofline["split"] = split
    if not cfg["resets"] and cfg["bytes"] == 1228:   # the full pipeline's 768 : 460 mix
        roofline["mix_ceiling"] = mix_ceiling("step_5r_3w", achieved)
    # the working set every step touches (records 384 B + state planes 320 B + the 4-frame input ring
    # + one output set per env): at config 3's 65,536 envs (109 MB) it largely fits the 126 MB L2, so
    # part of the algorithmic bytes come from L2 and frac can exceed 1; at 1M (1.7 GB) it cannot
    l2 = int(getattr(torch.cuda.get_device_properties(torch.cuda.current_device()), "L2_cache_size", 0) or 0)
    ws = n * (384 + ST_BYTES_PER_ENV + 4 * 184 + 220)
    roofline["working_set_bytes"] = ws
    roofline["l2_bytes"] = l2   # cudaDevAttrL2CacheSize
    roofline["l2_resident"] = bool(l2 and ws <= 1.25 * l2)
    if cold:
        cold["achieved"] = bytes_step / (cold["ms_per_step_median"] / 1e3) / 1e9
        cold["frac"] = cold["achieved"] / peak
        roofline["cold_l2"] = cold
    if roofline["l2_resident"]:
        roofline["note"] = "working set ~ L2 size: part of the bytes are L2 hits; frac against HBM overstates"

    # ---- e2e: through dr_step_host with pinned host buffers (copies inside the timed region) ----
    e2e = None
    if not args.profile and args.e2e_steps > 0:
        with torch.cuda.stream(lib_stream):
            # one pinned allocation each way (inputs [n*20 | n*26], outputs [n*20 | n*22 | n*10 | n*3]),
            # so dr_step_host moves each direction in one copy (include/dr.h)
            hin = torch.empty(n * (20 + 26)).pin_memory()
            ha, ho = hin[:n * 20].view(n, 20), hin[n * 20:].view(n, 26)
            ha.copy_(A[0].cpu())
            ho.copy_(O[0].cpu())
            hout = torch.empty(n * (20 + 22 + 10 + 3)).pin_memory()
            outs, o = [], 0
            for c in (20, 22, 10, 3):
                outs.append(hout[o:o + n * c].view(n, c))
                o += n * c
            dr.dr_step_host(ha, ho, *outs)
            dr.dr_synchronize()
            if world > 1:
                dist.barrier()
            # small configs: at least ~500 calls, so the host-clock region is tens of ms, not host jitter
            e2e_steps = args.e2e_steps if n >= 262144 else max(args.e2e_steps, 500)
            t0 = time.perf_counter()
            for i in range(e2e_steps):
                dr.dr_step_host(ha, ho, *outs)
            dr.dr_synchronize()
            e2e_s = time.perf_counter() - t0
            te = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
            if world > 1:
                dist.all_reduce(te, op=dist.ReduceOp.MAX)
            e2e_s = float(te.item())
        e2e = {"value": n_glob * e2e_steps / e2e_s, "unit": "env-steps/s",
               "h2d_bytes_per_step": n_glob * (20 + 26) * 4, "d2h_bytes_per_step": n_glob * (20 + 22 + 10 + 3) * 4,
               "api": "dr_step_host (pinned host buffers)", "steps": e2e_steps}

    ctx.close()
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline and not args.profile:
            cpu = cpu_baseline(cfg, args)
        line = {
            "metric": "randomized env-steps/sec", "value": value, "unit": "env-steps/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps,
            "higher_is_better": True, "scaling": cfg["scaling"], "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": cfg["workload"], "n_env_global": n_glob, "n_env_per_gpu": n,
                       "layers": hex(cfg["mask"]), "parallelism": f"env-shard x{world}",
                       "l2": "inputs larger than L2" if cfg["bytes"] * n > 126e6 else "L2-resident (warm)",
                       "cuda_graph_steps": G,
                       "bytes_per_step_per_gpu": cfg["bytes"] * n},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
            "clocks": clocks,
            "stats_check": {"envs_last_step": stats[0], "force_trig_rate": stats[6] / max(stats[0], 1)},
        }
        if cfg["resets"]:
            line["resets_per_sec"] = (n_glob / 10) * args.steps / (elapsed_ms / 1e3)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
