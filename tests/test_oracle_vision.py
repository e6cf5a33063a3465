"""Pins for the vision-randomization oracle (oracle/oracle_vision.c) against what the paper and
mathematics fix: the table values (Table vision-randomization), the
normalisation's definition (zero mean / unit variance), linear contrast scaling,
the noise distribution, affine invariance of the normalisation, and the range / frequency
invariants of every appearance draw."""
import json
import math
import os

import numpy as np
import pytest
from scipy import stats

from conftest import GOLDEN
from workload import presets

SEED = presets.SEED_DR


@pytest.fixture(scope="module")
def table():
    with open(os.path.join(GOLDEN, "vision_table.json")) as f:
        return json.load(f)


def _img(n, h, w, c, seed=0, lo=0, hi=256):
    return np.random.default_rng(seed).integers(lo, hi, (n, h, w, c), dtype=np.uint8)


def test_vision_preset_is_the_paper_table(table):
    V = presets.VISION
    assert V["cam_pos_range"] == pytest.approx(table["camera_position_mm"] * 1e-3)
    assert V["cam_rot_max"] == pytest.approx(math.radians(table["camera_rotation_deg"][1]))
    assert V["cam_fov_range"] == pytest.approx(math.radians(table["camera_fov_deg"]))
    assert [V["robot_metallic_lo"], V["robot_metallic_hi"]] == pytest.approx([x / 100 for x in table["robot_metallic_pct"]])
    assert [V["robot_gloss_lo"], V["robot_gloss_hi"]] == pytest.approx([x / 100 for x in table["robot_glossiness_pct"]])
    assert V["obj_hue_range"] == pytest.approx(table["object_hue_pct"] / 100)
    assert V["obj_sat_range"] == pytest.approx(table["object_saturation_pct"] / 100)
    assert V["obj_val_range"] == pytest.approx(table["object_value_pct"] / 100)
    assert [V["obj_metallic_lo"], V["obj_metallic_hi"]] == pytest.approx([x / 100 for x in table["object_metallic_pct"]])
    assert [V["obj_gloss_lo"], V["obj_gloss_hi"]] == pytest.approx([x / 100 for x in table["object_glossiness_pct"]])
    assert [V["lights_min"], V["lights_max"]] == table["number_of_lights"]
    assert [V["light_rel_lo"], V["light_rel_hi"]] == table["light_relative_intensity"]
    assert [V["light_total_lo"], V["light_total_hi"]] == table["total_light_intensity"]
    assert [V["contrast_lo"], V["contrast_hi"]] == pytest.approx([x / 100 for x in table["image_contrast_pct"]])
    assert V["noise_std_lo"] == V["noise_std_hi"] == pytest.approx(table["pixel_noise_pct"] / 100)
    assert presets.VISION_BATCH_SAMPLES * presets.VISION_CAMERAS == table["images_per_batch"]
    assert [presets.VISION_H, presets.VISION_W] == table["image_hw"]


# ---- image augmentation ------------------------------------------------------
def test_normalisation_zero_mean_unit_variance():
    """Contrast pinned to 1 and noise to 0: every image has mean 0 and std 1."""
    from oracle import oracle as O
    P = presets.vision_preset(contrast_lo=1.0, contrast_hi=1.0, noise_std_lo=0.0, noise_std_hi=0.0)
    out, st = O.image_augment(P, SEED, 0, _img(6, 17, 13, 3))
    for i in range(6):
        assert abs(out[i].mean()) < 1e-12
        assert abs(out[i].std() - 1.0) < 1e-12
    assert (st[:, 2] == 1.0).all() and (st[:, 3] == 0.0).all()


def test_contrast_is_linear_scaling():
    """Contrast factor pinned to 0.5 (noise off): output std 0.5, and out = 0.5 x the unit-variance
    image of the same input."""
    from oracle import oracle as O
    x = _img(3, 9, 11, 3, seed=1)
    P1 = presets.vision_preset(contrast_lo=1.0, contrast_hi=1.0, noise_std_lo=0.0, noise_std_hi=0.0)
    Ph = presets.vision_preset(contrast_lo=0.5, contrast_hi=0.5, noise_std_lo=0.0, noise_std_hi=0.0)
    o1, _ = O.image_augment(P1, SEED, 0, x)
    oh, _ = O.image_augment(Ph, SEED, 0, x)
    for i in range(3):
        assert abs(oh[i].std() - 0.5) < 1e-12
    assert np.array_equal(oh, 0.5 * o1)


def test_normalisation_affine_invariance():
    """Normalisation removes any positive affine map of the intensities: x and 2x + 10 give the same
    augmented image for the same seed (a wrong mean or std would not cancel)."""
    from oracle import oracle as O
    x = _img(4, 10, 10, 3, seed=2, hi=120)
    y = (2 * x.astype(np.int32) + 10).astype(np.uint8)
    ox, _ = O.image_augment(presets.vision_preset(), SEED, 5, x)
    oy, _ = O.image_augment(presets.vision_preset(), SEED, 5, y)
    assert np.abs(ox - oy).max() < 1e-12


def test_constant_image_is_noise_only():
    """Degenerate variance: a constant image normalises to 0 (std floored), so with noise off the
    output is all zeros, and with noise s the output is s z."""
    from oracle import oracle as O
    x = np.full((2, 40, 40, 3), 77, np.uint8)
    o0, st = O.image_augment(presets.vision_preset(noise_std_lo=0.0, noise_std_hi=0.0), SEED, 0, x)
    assert (o0 == 0.0).all() and (st[:, 1] == 0.0).all()
    o1, _ = O.image_augment(presets.vision_preset(noise_std_lo=0.25, noise_std_hi=0.25), SEED, 0, x)
    z = o1.reshape(-1) / 0.25
    assert abs(z.mean()) < 4 / math.sqrt(z.size)
    assert abs(z.std() - 1.0) < 4 / math.sqrt(2 * z.size)
    assert stats.kstest(z, "norm").pvalue > 1e-3


def test_noise_independent_across_pixels_and_images():
    """Per-pixel noise is i.i.d.: neighbouring elements (same Philox block and across blocks) and the
    same pixel of two images are uncorrelated."""
    from oracle import oracle as O
    x = np.full((2, 64, 64, 3), 50, np.uint8)
    o, _ = O.image_augment(presets.vision_preset(noise_std_lo=1.0, noise_std_hi=1.0), SEED, 3, x)
    a = o[0].reshape(-1)
    bound = 5 / math.sqrt(a.size)
    for lag in (1, 2, 3, 4, 5):
        assert abs(np.corrcoef(a[:-lag], a[lag:])[0, 1]) < bound
    assert abs(np.corrcoef(o[0].reshape(-1), o[1].reshape(-1))[0, 1]) < bound


def test_per_image_draw_distributions():
    """Contrast factor ~ U[0.5, 1.5] and noise std ~ U[lo, hi], one draw per image (Table
    vision-randomization "image contrast adjustment 50%-150%")."""
    from oracle import oracle as O
    x = _img(4000, 1, 1, 1, seed=3)
    _, st = O.image_augment(presets.vision_preset(noise_std_lo=0.05, noise_std_hi=0.2), SEED, 0, x)
    assert st[:, 2].min() >= 0.5 and st[:, 2].max() <= 1.5
    assert stats.kstest((st[:, 2] - 0.5) / 1.0, "uniform").pvalue > 1e-3
    assert stats.kstest((st[:, 3] - 0.05) / 0.15, "uniform").pvalue > 1e-3


def test_partition_invariance_images():
    """Results depend on the global image id, not on how a batch is split: images [0, 6) in one
    call equal [0, 2) + [2, 6) with image_offset 2."""
    from oracle import oracle as O
    x = _img(6, 5, 7, 3, seed=4)
    P = presets.vision_preset()
    a, sa = O.image_augment(P, SEED, 9, x)
    b1, s1 = O.image_augment(P, SEED, 9, x[:2])
    b2, s2 = O.image_augment(P, SEED, 9, x[2:], image_offset=2)
    assert np.array_equal(a, np.concatenate([b1, b2]))
    assert np.array_equal(sa, np.concatenate([s1, s2]))


# ---- appearance draws (Table vision-randomization) ------------------------------
@pytest.fixture(scope="module")
def scenes():
    from oracle import oracle as O
    return O.scene_draw(presets.vision_preset(), SEED, 7, 60000)


def test_scene_fields_inside_their_ranges(scenes):
    V = presets.VISION
    S = scenes
    pos = S[:, 0:9]
    assert np.abs(pos).max() <= V["cam_pos_range"]
    assert stats.kstest(pos[:, 0] / (2 * V["cam_pos_range"]) + 0.5, "uniform").pvalue > 1e-3
    q = S[:, 9:21].reshape(-1, 3, 4)
    assert np.allclose(np.linalg.norm(q, axis=2), 1.0, atol=1e-12)
    ang = 2 * np.arccos(np.clip(q[:, :, 0], -1, 1))
    assert ang.max() <= V["cam_rot_max"] + 1e-12
    assert stats.kstest(ang.reshape(-1) / V["cam_rot_max"], "uniform").pvalue > 1e-3
    assert np.abs(S[:, 21:24]).max() <= V["cam_fov_range"]
    assert S[:, 24:27].min() > 0 and S[:, 24:27].max() < 1
    assert V["robot_metallic_lo"] <= S[:, 27].min() and S[:, 27].max() <= V["robot_metallic_hi"]
    assert V["robot_gloss_lo"] <= S[:, 28].min() and S[:, 28].max() <= V["robot_gloss_hi"]
    h, s, v = S[:, 29], S[:, 30], S[:, 31]
    assert h.min() >= 0 and h.max() < 1
    # hue wraps: calibrated 0.005 +- 0.01 -> a quarter of the draws land in [0.995, 1)
    assert abs((h > 0.5).mean() - 0.25) < 0.01
    # saturation clamps: 0.9 + U[-0.15, 0.15] exceeds 1 with probability 1/6
    assert abs((s == 1.0).mean() - 1 / 6) < 0.01 and s.max() == 1.0
    assert v.min() >= 0.35 and v.max() <= 0.65
    assert 0.05 <= S[:, 32].min() and S[:, 32].max() <= 0.15
    assert 0.05 <= S[:, 33].min() and S[:, 33].max() <= 0.15


def test_scene_lights(scenes):
    S = scenes
    n = S[:, 34].astype(int)
    assert set(np.unique(n)) == {4, 5, 6}
    for k in (4, 5, 6):
        assert abs((n == k).mean() - 1 / 3) < 0.02   # "number of lights 4-6", uniform
    d = S[:, 35:53].reshape(-1, 6, 3)
    I = S[:, 53:59]
    for k in (4, 5, 6):
        m = n == k
        dk = d[m][:, :k]
        assert np.allclose(np.linalg.norm(dk, axis=2), 1.0, atol=1e-12)
        assert dk[:, :, 2].min() > 0          # upper half-sphere
        assert (d[m][:, k:] == 0).all() and (I[m][:, k:] == 0).all()
    # hemisphere area-uniform: z ~ U[0, 1]
    z = d[n == 6][:, :, 2].reshape(-1)
    assert stats.kstest(z, "uniform").pvalue > 1e-3
    tot = S[:, 59]
    assert tot.min() >= 0 and tot.max() <= 15
    assert np.allclose(I.sum(axis=1), tot, rtol=1e-12, atol=1e-12)
    # relative intensities in [1, 5]: ratios of two lights lie in [1/5, 5]
    r = I[:, 1] / I[:, 0]
    assert r.min() >= 0.2 - 1e-12 and r.max() <= 5 + 1e-12
    assert (S[:, 60:64] == 0).all()


# ---- vision-model pose augmentation ----------------------
def _qmul(a, b):
    w1, x1, y1, z1 = a.T
    w2, x2, y2, z2 = b.T
    return np.stack([w1 * w2 - x1 * x2 - y1 * y2 - z1 * z2, w1 * x2 + x1 * w2 + y1 * z2 - z1 * y2,
                     w1 * y2 - x1 * z2 + y1 * w2 + z1 * x2, w1 * z2 + x1 * y2 - y1 * x2 + z1 * w2], axis=1)


def test_pose_augment_branches():
    """Keep the pose 20 %, rotate 90 deg about a main (body) axis 40 %, jitter position and rotation
    40 %: branch frequencies, exact identity, the relative rotation q_in^-1 q_out is
    exactly 90 deg about +-e_x / e_y / e_z with the position unchanged, and the jitter's position
    noise is N(0, pos_std^2) with a half-normal rotation angle."""
    from oracle import oracle as O
    P = presets.pose_preset()
    n = 100000
    x = presets.poses(n, seed=3)
    out, br = O.pose_augment(P, SEED, 2, x)
    f = np.bincount(br, minlength=3) / n
    assert np.abs(f - np.array([0.2, 0.4, 0.4])).max() < 0.01
    xin = x.astype(np.float64)
    k0, k1, k2 = br == 0, br == 1, br == 2
    assert np.array_equal(out[k0], xin[k0])
    assert np.array_equal(out[k1, :3], xin[k1, :3])
    conj = xin[k1, 3:] * np.array([1, -1, -1, -1])
    rel = _qmul(conj, out[k1, 3:])
    rel /= np.linalg.norm(rel, axis=1, keepdims=True)                       # inputs are unit to float32 only
    assert np.abs(np.abs(rel[:, 0]) - math.sqrt(0.5)).max() < 1e-12        # angle exactly 90 deg
    ax = np.abs(rel[:, 1:]) > 1e-9
    assert (ax.sum(axis=1) == 1).all()                                      # about one body axis
    cnt = ax.sum(axis=0) / ax.shape[0]
    assert np.abs(cnt - 1 / 3).max() < 0.015
    z = (out[k2, :3] - xin[k2, :3]) / P["pos_std"]
    assert stats.kstest(z.reshape(-1), "norm").pvalue > 1e-3
    qn = np.linalg.norm(out[:, 3:], axis=1)
    assert np.abs(qn - 1).max() < 1e-6                                      # float32 inputs, unit to ~1e-7
    rel2 = _qmul(out[k2, 3:], xin[k2, 3:] * np.array([1, -1, -1, -1]))     # q_j = q_out q_in^-1 (world frame)
    ang = 2 * np.arccos(np.clip(np.abs(rel2[:, 0]) / np.linalg.norm(rel2, axis=1), -1, 1))
    assert abs(ang.mean() - P["rot_std"] * math.sqrt(2 / math.pi)) < 4 * P["rot_std"] / math.sqrt(ang.size)


# ---- simulator-provided occlusion bits ---------------------------------
def test_simulator_occlusion_mask_drives_the_hold():
    """With the simulator's occlusion bits installed, the occluded count is their popcount, and a
    flagged tip returns exactly its previous reading ("last available reading");
    with the OCCLUSION layer off the bits are ignored."""
    from oracle.oracle import Oracle
    from workload.presets import DROPOUT, FULL, OCCLUSION
    n, T = 32, 6
    from workload import gen
    acts, obs = gen.frames(n, T)
    o = Oracle(presets.preset(FULL & ~DROPOUT), n, SEED)
    rng = np.random.default_rng(0)
    m = o.set_occlusion_mask(np.zeros(n, np.uint8))
    prev = o.step(acts[0], obs[0])["out_obs"]
    for t in range(1, T):
        m[:] = rng.integers(0, 32, n)
        r = o.step(acts[t], obs[t])
        assert r["stats"][4] == sum(bin(int(v)).count("1") for v in m)
        for i in range(5):
            held = (m >> i) & 1 == 1
            assert np.array_equal(r["out_obs"][held, 4 + 3 * i:7 + 3 * i], prev[held, 4 + 3 * i:7 + 3 * i])
        prev = r["out_obs"]
    o.close()
    o = Oracle(presets.preset(FULL & ~DROPOUT & ~OCCLUSION), n, SEED)
    o.set_occlusion_mask(np.full(n, 31, np.uint8))
    o.step(acts[0], obs[0])
    assert o.step(acts[1], obs[1])["stats"][4] == 0
    o.close()
