"""The boundary from plain C: include/*.h parse as C99 on their own, and examples/dr_step_c.c
(which links libdr.so and the CUDA runtime, no Python) builds here and runs on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CUDA = "/usr/local/cuda"


@pytest.mark.parametrize("hdr", ["dr.h", "dr_vision.h"])
def test_headers_are_self_contained_c99(tmp_path, hdr):
    src = tmp_path / "t.c"
    src.write_text(f'#include "{hdr}"\nint main(void) {{ return 0; }}\n')
    r = subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-pedantic", "-fsyntax-only",
                        "-I" + os.path.join(ROOT, "include"), str(src)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def _build_example(out):
    from paper_1906_11633_b200 import dr
    dr.load()   # builds libdr.so if needed
    pkg = os.path.join(ROOT, "paper_1906_11633_b200")
    cmd = ["gcc", "-std=c99", "-O2", os.path.join(ROOT, "examples", "dr_step_c.c"), "-I" + os.path.join(ROOT, "include"),
           "-I" + os.path.join(CUDA, "include"), "-L" + pkg, "-ldr", "-L" + os.path.join(CUDA, "lib64"), "-lcudart",
           "-Wl,-rpath," + pkg, "-o", str(out)]
    return subprocess.run(cmd, capture_output=True, text=True)


def test_c_example_builds(tmp_path):
    if not os.path.exists(os.path.join(CUDA, "lib64", "libcudart.so")):
        pytest.skip("no CUDA runtime library to link")
    r = _build_example(tmp_path / "dr_step_c")
    assert r.returncode == 0, r.stderr


@pytest.mark.gpu
def test_c_example_runs(tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    exe = tmp_path / "dr_step_c"
    r = _build_example(exe)
    assert r.returncode == 0, r.stderr
    run = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert run.returncode == 0, run.stdout + run.stderr
    assert "envs 4096" in run.stdout and "steps 100" in run.stdout
