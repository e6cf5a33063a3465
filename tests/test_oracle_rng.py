"""Pins for the oracle's RNG layer: Philox4x32-10 and the draw transforms.

Pinned against: published Random123 known-answer vectors (tests/golden), cuRAND's own
Philox4x32_10 (an independent library, compiled for the host here), closed forms of the
uniform map, and distribution tests against scipy.stats (independent library CDFs).
"""
import math
import os
import shutil
import subprocess
import tempfile

import numpy as np
import pytest
from scipy import stats

from conftest import GOLDEN


def _kat_rows():
    rows = []
    with open(os.path.join(GOLDEN, "philox4x32_10_kat.txt")) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            v = [int(x, 16) for x in line.split()]
            rows.append((tuple(v[0:4]), tuple(v[4:6]), tuple(v[6:10])))
    return rows


def test_philox_known_answer_vectors(oracle_mod):
    rows = _kat_rows()
    assert len(rows) == 3
    for ctr, key, expect in rows:
        assert oracle_mod.philox(ctr, key) == expect


_CURAND_HOST_SRC = r"""
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define QUALIFIERS static inline __host__ __device__
#include <curand_philox4x32_x.h>
int main() {
  unsigned a, b, c, d, k0, k1;
  while (scanf("%x %x %x %x %x %x", &a, &b, &c, &d, &k0, &k1) == 6) {
    uint4 ctr = make_uint4(a, b, c, d); uint2 key = make_uint2(k0, k1);
    uint4 o = curand_Philox4x32_10(ctr, key);
    printf("%08x %08x %08x %08x\n", o.x, o.y, o.z, o.w);
  }
  return 0;
}
"""


@pytest.mark.skipif(shutil.which("nvcc") is None, reason="nvcc not available")
def test_philox_matches_curand_host(oracle_mod):
    """cuRAND's curand_Philox4x32_10 (curand_philox4x32_x.h), compiled as host code by nvcc,
    must agree word for word with the oracle's from-spec Philox on random (ctr, key)."""
    rng = np.random.default_rng(7)
    vals = rng.integers(0, 2**32, size=(2000, 6), dtype=np.uint64)
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "p.cu")
        exe = os.path.join(d, "p")
        with open(src, "w") as f:
            f.write(_CURAND_HOST_SRC)
        subprocess.check_call(["nvcc", "-O1", "-o", exe, src])
        inp = "\n".join(" ".join(f"{int(x):08x}" for x in row) for row in vals) + "\n"
        out = subprocess.run([exe], input=inp, capture_output=True, text=True, check=True).stdout.split("\n")
    for row, line in zip(vals, out):
        got = oracle_mod.philox(tuple(int(x) for x in row[:4]), tuple(int(x) for x in row[4:6]))
        assert got == tuple(int(x, 16) for x in line.split()), row


def test_uniform_closed_form(oracle_mod):
    # U(x) = ((x >> 9) + 0.5) * 2^-23 : extremes and exact dyadic values
    assert oracle_mod.uniform(0) == 2.0 ** -24
    assert oracle_mod.uniform(0xFFFFFFFF) == 1.0 - 2.0 ** -24
    assert oracle_mod.uniform(0x80000000) == 0.5 + 2.0 ** -24
    assert oracle_mod.uniform(0x000001FF) == 2.0 ** -24   # low 9 bits discarded
    for x in [1 << 9, 12345 << 9, 0xDEADBEEF]:
        assert oracle_mod.uniform(x) == ((x >> 9) + 0.5) / 2 ** 23
    # uniform on (0, 1): 2^23 equally spaced midpoints, mean exactly 1/2
    assert oracle_mod.uniform(0x7FFFFFFF) + oracle_mod.uniform(0x80000000) == 1.0
    # exactly representable in fp32 too: both sides see the identical u
    for x in [0, 0xFFFFFFFF, 0x12345678, 0x9ABCDEF0, 0xFFFFFE00, 0x80000000]:
        u = oracle_mod.uniform(x)
        assert float(np.float32(u)) == u


def _philox_words(oracle_mod, n_blocks, ch=0x77):
    w = np.empty((n_blocks, 4), dtype=np.uint64)
    for b in range(n_blocks):
        w[b] = oracle_mod.philox((b, 3, ch, 0), (0x12345678, 0x9ABCDEF0))
    return w


def test_normals_distribution(oracle_mod):
    """Box-Muller normals from Philox words: KS against scipy's standard normal CDF, and the
    pair (z0, z1) uncorrelated."""
    w = _philox_words(oracle_mod, 20000)
    z = []
    for b in range(w.shape[0]):
        z.extend(oracle_mod.normal_pair(int(w[b, 0]), int(w[b, 1])))
        z.extend(oracle_mod.normal_pair(int(w[b, 2]), int(w[b, 3])))
    z = np.array(z)
    assert abs(z.mean()) < 5 / math.sqrt(len(z))
    assert abs(z.var() - 1.0) < 5 * math.sqrt(2.0 / len(z))
    ks = stats.kstest(z, "norm")
    assert ks.pvalue > 1e-3, ks
    z0, z1 = z[0::2], z[1::2]
    assert abs(np.corrcoef(z0, z1)[0, 1]) < 5 / math.sqrt(len(z0))


def test_normal_pair_polar_identity(oracle_mod):
    # z0^2 + z1^2 = -2 ln U(x) for any y (Box-Muller radius), and atan2(z1, z0) = 2 pi U(y) mod 2 pi
    for x, y in [(0x10000000, 0x40000000), (0xFFFFFF00, 0x00000100), (0x00000000, 0xC0000000)]:
        z0, z1 = oracle_mod.normal_pair(x, y)
        u = oracle_mod.uniform(x)
        assert math.isclose(z0 * z0 + z1 * z1, -2.0 * math.log(u), rel_tol=1e-12)
        ang = math.atan2(z1, z0) % (2 * math.pi)
        assert math.isclose(ang, (2 * math.pi * oracle_mod.uniform(y)) % (2 * math.pi), rel_tol=1e-9, abs_tol=1e-9)


def test_exponential_distribution(oracle_mod):
    """Exp(lambda) is rate-parameterised [Q10]: KS against scipy's expon(scale=1/lambda)."""
    lam = 1250.0
    w = _philox_words(oracle_mod, 10000, ch=0x55).reshape(-1)
    x = np.array([oracle_mod.exponential(int(v), lam) for v in w])
    assert (x > 0).all()
    assert abs(x.mean() - 1 / lam) < 5 * (1 / lam) / math.sqrt(len(x))
    assert stats.kstest(x, "expon", args=(0, 1 / lam)).pvalue > 1e-3


def test_bernoulli_thresholds(oracle_mod):
    # T = floor(p * 2^32); event is x < T
    assert oracle_mod.bernoulli_threshold(0.5) == 2 ** 31                 # delay p = 0.5
    assert oracle_mod.bernoulli_threshold(0.0) == 0
    assert oracle_mod.bernoulli_threshold(1.0) == 2 ** 32
    # dropout: 0.2 per second at the nominal 80 ms step: 1 - exp(-0.016)
    t_drop = oracle_mod.bernoulli_threshold(1.0 - math.exp(-0.2 * 0.08))
    assert t_drop == 68172641
    assert abs(t_drop / 2 ** 32 - 0.015873) < 1e-6


def test_force_probability_table(oracle_mod):
    """Loguniform p on [0.1 %, 10 %] quantised to 65,536 midpoints [Q19]:
    endpoints, monotone, ln p equally spaced, thresholds = floor(p 2^32)."""
    from workload import presets
    from oracle.oracle import Oracle
    orc = Oracle(presets.preset(presets.FORCE), 1, 1)
    p0, p_last = orc.force_p(0), orc.force_p(65535)
    assert math.isclose(p0, 0.001 * math.exp(0.5 / 65536 * math.log(100)), rel_tol=1e-12)
    assert math.isclose(p_last, 0.1 * math.exp(-0.5 / 65536 * math.log(100)), rel_tol=1e-12)
    assert orc.force_threshold(0) == 4295118
    assert orc.force_threshold(65535) == 429481639
    ps = np.array([orc.force_p(j) for j in range(0, 65536, 97)])
    d = np.diff(np.log(ps))
    assert np.allclose(d, d[0], rtol=1e-9)
    for j in [0, 1, 1000, 32767, 65535]:
        assert orc.force_threshold(j) == math.floor(orc.force_p(j) * 2 ** 32)
