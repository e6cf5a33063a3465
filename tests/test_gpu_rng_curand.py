"""Device RNG vs cuRAND on the device: the round function every libdr kernel
draws from (dr_math.cuh philox_rounds, through the C-ABI hook dr_debug_philox_keyed) equals cuRAND's
curand_Philox4x32_10 (Salmon et al., SC'11; the Random123 reference the oracle is pinned to in
tests/test_oracle_rng.py) on 2^24 random (counter, key) pairs plus structured edge pairs.  The cuRAND
side is a test-only kernel (tests/cuda/curand_philox_ref.cu) built here with nvcc."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.fixture(scope="module")
def curand_ref(tmp_path_factory):
    so = str(tmp_path_factory.mktemp("curand") / "libcurand_ref.so")
    nvcc = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")
    subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "--shared", "-Xcompiler", "-fPIC",
                    "-o", so, os.path.join(HERE, "cuda", "curand_philox_ref.cu")], check=True)
    lib = C.CDLL(so)
    lib.curand_philox_ref.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_ulonglong, C.c_void_p]
    lib.curand_philox_ref.restype = C.c_int
    return lib


def _both(torch, lib, ctr, key):
    from paper_1906_11633_b200 import dr
    n = ctr.shape[0]
    got = torch.empty(n, 4, dtype=torch.int32, device="cuda")
    ref = torch.empty(n, 4, dtype=torch.int32, device="cuda")
    dr.dr_debug_philox_keyed(ctr, key, got)
    s = torch.cuda.current_stream().cuda_stream
    assert lib.curand_philox_ref(ctr.data_ptr(), key.data_ptr(), ref.data_ptr(), n, s) == 0
    torch.cuda.synchronize()
    return got, ref


@pytest.mark.gpu
def test_device_philox_equals_curand_2pow24_random_pairs(torch_cuda, curand_ref):
    torch = torch_cuda
    g = torch.Generator(device="cuda").manual_seed(20261017)
    n = 1 << 24
    ctr = torch.randint(-2**31, 2**31, (n, 4), dtype=torch.int64, device="cuda", generator=g).to(torch.int32)
    key = torch.randint(-2**31, 2**31, (n, 2), dtype=torch.int64, device="cuda", generator=g).to(torch.int32)
    got, ref = _both(torch, curand_ref, ctr, key)
    bad = (got != ref).any(dim=1)
    assert int(bad.sum()) == 0, f"{int(bad.sum())} of {n} blocks differ; first at {int(bad.nonzero()[0])}"


@pytest.mark.gpu
def test_device_philox_equals_curand_edge_pairs(torch_cuda, curand_ref):
    """All-zero / all-ones words, single-bit counters and keys, and the counter layout the kernels
    use (global env, t or episode, channel, block) at the top of each range."""
    torch = torch_cuda
    M = 0xFFFFFFFF
    kat = []
    with open(os.path.join(HERE, "golden", "philox4x32_10_kat.txt")) as f:
        for line in f:
            if line.strip() and not line.startswith("#"):
                v = [int(x, 16) for x in line.split()]
                kat.append(((tuple(v[0:4]), tuple(v[4:6])), tuple(v[6:10])))
    rows = [k[0] for k in kat]
    rows += [((0, 0, 0, 0), (0, 0)), ((M, M, M, M), (M, M)), ((M, M, M, M), (0, 0)), ((0, 0, 0, 0), (M, M)),
            ((1048575, 0xFFFFFFFE, 0x10C, 63), (0x89ABCDEF, 0x01234567))]
    rows += [((1 << b if w == 0 else 0, 1 << b if w == 1 else 0, 1 << b if w == 2 else 0, 1 << b if w == 3 else 0),
              (0x9E3779B9, 0xBB67AE85)) for w in range(4) for b in range(32)]
    rows += [((b, b, b, b), (1 << (b % 32), 1 << ((b + 7) % 32))) for b in range(64)]
    ctr = torch.from_numpy(np.array([r[0] for r in rows], dtype=np.uint32).view(np.int32)).cuda()
    key = torch.from_numpy(np.array([r[1] for r in rows], dtype=np.uint32).view(np.int32)).cuda()
    got, ref = _both(torch, curand_ref, ctr, key)
    assert torch.equal(got, ref)
    # and the published Random123 known-answer vectors (tests/golden, as in tests/test_oracle_rng.py)
    g = got.cpu().numpy().view(np.uint32)
    for i, (_, expect) in enumerate(kat):
        assert tuple(int(x) for x in g[i]) == expect
