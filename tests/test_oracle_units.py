"""Pins for the oracle's per-element rules: backlash, occlusion,
quaternion algebra and the random-rotation draw."""
import math
import os

import numpy as np
import pytest
from scipy.spatial.transform import Rotation

from conftest import GOLDEN


def _backlash_rows():
    rows = []
    with open(os.path.join(GOLDEN, "backlash_hand.txt")) as f:
        for line in f:
            if not line.strip() or line.startswith("#"):
                continue
            lhs, rhs, tol, note = [x.strip() for x in line.split("|", 3)]
            rows.append(([float(x) for x in lhs.split()], [float(x) for x in rhs.split()], float(tol), note))
    return rows


@pytest.mark.parametrize("row", _backlash_rows(), ids=lambda r: r[3][:40])
def test_backlash_hand_examples(oracle_mod, row):
    (s, a, dn, dp, dt), (s_new, alpha, out), tol, note = row
    sn, al, o = oracle_mod.backlash(s, a, dn, dp, dt)
    assert math.isclose(sn, s_new, rel_tol=1e-12, abs_tol=1e-15), note
    assert abs(al - alpha) <= max(tol, 0.0) + 1e-300 if tol else al == alpha, (al, note)
    assert abs(o - out) <= tol + 1e-300 if tol else o == out, (o, note)
    if not tol and out == 0.0:
        # sign of zero: alpha * a keeps a's sign [Q3]
        assert math.copysign(1.0, o) == math.copysign(1.0, out), note


def test_backlash_invariants_random_states(oracle_mod):
    """SPEC.md:219 invariants (as corrected in DESIGN.md [Q5]) on random states:
    s' in [-1,1]; alpha in [0,1]; |out| <= |a|; out*a >= 0; alpha = 1 iff s == sgn(a) at step start
    (or a = s = 0); otherwise alpha <= eps/|sgn(a) - s| (+ rounding)."""
    rng = np.random.default_rng(1)
    n = 40000
    s = rng.uniform(-1, 1, n)
    s[: n // 10] = rng.choice([-1.0, 1.0], n // 10)        # engaged states
    a = rng.uniform(-1, 1, n)
    a[n // 10: n // 10 + 500] = 0.0
    dn = rng.uniform(0, 6, n)
    dp = rng.uniform(0, 6, n)
    dt = rng.uniform(0.08, 0.09, n)
    eps = 1e-12
    for i in range(n):
        sn, al, o = oracle_mod.backlash(s[i], a[i], dn[i], dp[i], dt[i], eps)
        sg = float(a[i] > 0) - float(a[i] < 0)
        assert -1.0 <= sn <= 1.0
        assert 0.0 <= al <= 1.0
        assert abs(o) <= abs(a[i])
        assert o * a[i] >= 0.0
        if s[i] == sg:
            assert al == 1.0
        else:
            assert al <= eps / abs(sg - s[i]) * (1 + 1e-3) + 1e-15, (s[i], a[i], al)
        if sg == 0:
            assert sn == s[i]


def test_occlusion_rules(oracle_mod):
    tips = np.zeros(15, dtype=np.float32)
    for i in range(5):
        tips[3 * i] = 0.1 * i                 # far apart
    obj = np.array([1.0, 1.0, 1.0], dtype=np.float32)
    # occl_dist = 0 -> never occluded (even coincident points)
    t2 = tips.copy()
    t2[3:6] = t2[0:3]
    assert not any(oracle_mod.occluded(t2, obj, 0.0, i) for i in range(5))
    # two fingertips at distance d/2 -> both occluded
    d = 0.015
    t3 = tips.copy()
    t3[3] = t3[0] + d / 2
    t3[4] = t3[1]
    t3[5] = t3[2]
    assert oracle_mod.occluded(t3, obj, d, 0) and oracle_mod.occluded(t3, obj, d, 1)
    assert not oracle_mod.occluded(t3, obj, d, 2)
    # object centre within d of tip 4 -> only tip 4
    obj2 = np.array([t3[12] + 0.01, t3[13], t3[14]], dtype=np.float32)
    assert oracle_mod.occluded(t3, obj2, d, 4) and not oracle_mod.occluded(t3, obj2, d, 3)
    # exact boundary (dyadic, so every fp64 op is exact): r = 2^-6, tips at x = 0 and x = 2^-6
    # -> D = r^2 exactly -> NOT occluded (strict <); one fp32 ulp closer -> occluded.
    r = 2.0 ** -6
    t4 = np.zeros(15, dtype=np.float32)
    for i in range(2, 5):
        t4[3 * i] = 1.0 + i
    t4[3] = np.float32(r)
    assert not oracle_mod.occluded(t4, obj, r, 0)
    t4[3] = np.nextafter(np.float32(r), np.float32(0))
    assert oracle_mod.occluded(t4, obj, r, 0)


def _scipy_mul(a, b):
    # scipy uses scalar-last quaternions; composition R(a) * R(b) == a (x) b (Hamilton product)
    ra = Rotation.from_quat([a[1], a[2], a[3], a[0]])
    rb = Rotation.from_quat([b[1], b[2], b[3], b[0]])
    x, y, z, w = (ra * rb).as_quat()
    return np.array([w, x, y, z])


def test_quat_mul_vs_scipy(oracle_mod):
    rng = np.random.default_rng(3)
    for _ in range(200):
        a = rng.standard_normal(4)
        a /= np.linalg.norm(a)
        b = rng.standard_normal(4)
        b /= np.linalg.norm(b)
        got = np.array(oracle_mod.quat_mul(a, b))
        ref = _scipy_mul(a, b)
        if np.dot(got, ref) < 0:
            ref = -ref
        assert np.allclose(got, ref, atol=1e-12)
    # identity and i*j = k
    assert oracle_mod.quat_mul((1, 0, 0, 0), (0, 1, 0, 0)) == (0, 1, 0, 0)
    assert oracle_mod.quat_mul((0, 1, 0, 0), (0, 0, 1, 0)) == (0, 0, 0, 1)


def test_random_rotation_distribution(oracle_mod):
    """Orientation noise "0.1 rad" read as angle ~ N(0, 0.1^2) about a uniform axis
    [Q15]: unit quaternion; |angle| half-normal with mean 0.1 sqrt(2/pi) (scipy rotvec); axis
    uniform on the sphere (E[axis] = 0, E[axis_z^2] = 1/3)."""
    sigma = 0.1
    n = 20000
    ang, ax = [], []
    for b in range(n):
        w = oracle_mod.philox((b, 0, 0x10B, 0), (1, 2))
        q = np.array(oracle_mod.rotation(sigma, w))
        assert abs(np.linalg.norm(q) - 1.0) < 1e-12
        rv = Rotation.from_quat([q[1], q[2], q[3], q[0]]).as_rotvec()
        th = np.linalg.norm(rv)
        ang.append(th)
        if th > 1e-6:
            ax.append(rv / th)
    ang = np.array(ang)
    ax = np.array(ax)
    assert abs(ang.mean() - sigma * math.sqrt(2 / math.pi)) < 4 * sigma * 0.6 / math.sqrt(n)
    assert abs(np.sqrt((ang ** 2).mean()) - sigma) < 0.02 * sigma
    assert np.all(np.abs(ax.mean(axis=0)) < 4 / math.sqrt(3 * len(ax)) * 1.0)
    assert abs((ax[:, 2] ** 2).mean() - 1 / 3) < 0.01
