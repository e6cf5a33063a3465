"""The examples run: examples/rl_loop.py (the library inside a rollout loop: policy stand-in,
dr_step, simulator stand-in, dr_reset of ended episodes, vision every 64 steps, stats prints)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_rl_loop_example_runs():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "examples", "rl_loop.py"), "--envs", "8192", "--steps", "100"],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "100 steps of 8192 envs done" in r.stdout, r.stdout
    assert "step 100:" in r.stdout


@pytest.mark.parametrize("name", ["rl_loop.py"])
def test_examples_compile(name):
    """(CPU) the example scripts are valid Python."""
    import py_compile
    py_compile.compile(os.path.join(ROOT, "examples", name), doraise=True)
