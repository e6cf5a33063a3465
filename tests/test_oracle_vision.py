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
