"""bench.py's reference arm (the fp64 oracle on host cores) runs here on CPU: its JSON
line carries the contract's keys, and under torchrun only rank 0 prints (the others exit 0)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(extra_env=None, *args):
    env = dict(os.environ)
    env.update(extra_env or {})
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "2", "--warmup", "1",
           "--cpu-sample-envs", "64"] + list(args)
    return subprocess.run(cmd, capture_output=True, text=True, env=env, cwd=ROOT, timeout=300)


def test_reference_arm_json_line():
    r = _run()
    assert r.returncode == 0, r.stderr
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["metric"] == "randomized env-steps/sec" and d["unit"] == "env-steps/s"
    assert d["value"] > 0 and d["higher_is_better"] is True and d["data"] == "synthetic"
    assert d["config"]["workload"] == "cfg4-1M-envs-full-pipeline"
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] == os.cpu_count() and cb["value"] == d["value"]
    assert "64 envs" in cb["sample"] and "OpenMP" in cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_reference_arm_reset_config():
    r = _run(None, "--config", "reset")
    assert r.returncode == 0, r.stderr
    d = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][0])
    assert d["config"]["workload"] == "cfg5-1M-envs-10pct-resets-per-step" and d["value"] > 0


def test_reference_arm_non_zero_rank_is_silent():
    r = _run({"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"})
    assert r.returncode == 0, r.stderr
    assert not [l for l in r.stdout.splitlines() if l.startswith("{")]


def test_mix_ceiling_reads_the_committed_probe():
    """roofline.mix_ceiling comes from profiles/bw_ceiling.json, written from the
    scripts/bw_ceiling.cu runs in profiles/round2_v6_bw_ceiling.txt."""
    sys.path.insert(0, ROOT)
    import bench
    with open(os.path.join(ROOT, "profiles", "bw_ceiling.json")) as f:
        d = json.load(f)
    txt = open(os.path.join(ROOT, "profiles", "round2_v6_bw_ceiling.txt")).read()
    for mix in ("step_5r_3w", "vision_1r_4w", "copy_1r_1w"):
        assert f'"best_gbs": {d[mix]["gbs"]}' in txt, mix   # the figure is one the probe printed
        m = bench.mix_ceiling(mix, 0.5 * d[mix]["gbs"])
        assert m["gbs"] == d[mix]["gbs"] and abs(m["frac"] - 0.5) < 1e-12
    assert bench.mix_ceiling("no_such_mix", 1.0) is None
