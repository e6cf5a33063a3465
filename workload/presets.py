"""Parameter presets: values quoted from the paper's tables, plus the DESIGN.md readings for
what the paper leaves open.  Data only -- no thresholds, tables or transforms are computed here.

Citations: PAPER.md line numbers of /root/reference/PAPER.md ("Randomizations" appendix).
"""
from __future__ import annotations

import copy

# Layer bits
TIMING, ACT_NOISE, DELAY, BACKLASH, OBS_NOISE = 1 << 0, 1 << 1, 1 << 2, 1 << 3, 1 << 4
DROPOUT, OCCLUSION, FORCE, PHYS = 1 << 5, 1 << 6, 1 << 7, 1 << 8
ALL = 0x1FF
# SURVEY.md §8(f) rank 2 variants (not in the paper's randomization set, so not in FULL)
SMOOTH, SUBSTEP_BACKLASH = 1 << 9, 1 << 10
FULL = ALL
# config 2: "backlash + action/obs noise"; TIMING is needed because backlash uses dt.
CFG2 = TIMING | ACT_NOISE | BACKLASH | OBS_NOISE

LAYER_NAMES = {
    "TIMING": TIMING, "ACT_NOISE": ACT_NOISE, "DELAY": DELAY, "BACKLASH": BACKLASH,
    "OBS_NOISE": OBS_NOISE, "DROPOUT": DROPOUT, "OCCLUSION": OCCLUSION, "FORCE": FORCE,
    "PHYS": PHYS,
}

# physical-parameter descriptor kinds (SPEC.md:126 schema; the paper's table is missing)
PHYS_FIXED, PHYS_UNIFORM_SCALE, PHYS_LOGUNIFORM_SCALE, PHYS_ADD_GAUSS, PHYS_MUL_LOGNORMAL = 0, 1, 2, 3, 4

N_ACT, N_TIPS, N_SUB, MAX_PHYS = 20, 5, 10, 256
OBS_IN, OBS_OUT = 26, 22

SEED_DR = 1906011633      # library seed S_DR
SEED_WORKLOAD = 1808000177  # workload seed S_W


def default_phys_table():
    """[Q20] The paper's physical-parameter table is absent.  Synthetic P = 256
    slots (~264 calibrated values): kinds cycle UNIFORM_SCALE(0.5, 1.5),
    LOGUNIFORM_SCALE(0.3, 3), ADD_GAUSS(0.15), MUL_LOGNORMAL(0.2) (SPEC.md:224 defaults);
    base value 0.5 + 0.01 * index.  Slot 0 is the object mass (base 0.5 kg).
    Parity unpinned: a workload choice."""
    kinds = [
        (PHYS_UNIFORM_SCALE, 0.5, 1.5),
        (PHYS_LOGUNIFORM_SCALE, 0.3, 3.0),
        (PHYS_ADD_GAUSS, 0.15, 0.0),
        (PHYS_MUL_LOGNORMAL, 0.2, 0.0),
    ]
    table = []
    for i in range(MAX_PHYS):
        k, a, b = kinds[i % 4]
        table.append((k, a, b, 0.5 + 0.01 * i))
    return table


PAPER = {
    # Table action-noise, "percentage of the action range"; range = 2 [Q8]
    "act_sigma_uadd": 0.10,   # 5 %   uncorrelated additive
    "act_sigma_cadd": 0.03,   # 1.5 % correlated additive
    "act_sigma_mult": 0.015,  # 1.5 % uncorrelated multiplicative (unitless)
    "delay_prob": 0.5,
    # timing
    "dt_base": 0.008, "lambda_lo": 1250.0, "lambda_hi": 10000.0, "step_nominal": 0.08,
    # backlash; calibrated widths not given [Q21]
    "delta_cal_neg": [3.5 + 0.1 * j for j in range(N_ACT)],
    "delta_cal_pos": [4.0 + 0.1 * j for j in range(N_ACT)],
    "delta_jitter_std": 0.1, "backlash_eps": 1e-12,
    # Table obs-noise, metres / radians
    "tip_corr": 1e-3, "tip_uncorr": 2e-3, "obj_corr": 5e-3, "obj_uncorr": 1e-3,
    "rot_corr": 0.1, "rot_uncorr": 0.1, "tip_marker": 3e-3, "base_marker": 1e-3,
    "base_marker_to_tips": 1,  # [Q14]
    # PhaseSpace errors; hold = ceil(1 s / 80 ms) = 13 steps [Q11]; 15 mm [Q13]
    "dropout_rate_hz": 0.2, "dropout_hold_steps": 13, "occl_dist": 0.015,
    # random forces
    "force_p_lo": 0.001, "force_p_hi": 0.1, "force_accel_std": 1.0, "force_decay_per_step": 0.99,
    # action smoothing: "exponential moving average ... coefficient of 0.3 per 80ms" [Q25]
    "act_smooth_coef": 0.3,
    # physical parameters [Q20]
    "n_phys": MAX_PHYS, "mass_index": 0, "phys": default_phys_table(),
    "layer_mask": FULL,
}


def preset(layer_mask: int = FULL, **overrides) -> dict:
    """A deep copy of the paper preset with ``layer_mask`` and any field overrides."""
    p = copy.deepcopy(PAPER)
    p["layer_mask"] = int(layer_mask)
    for k, v in overrides.items():
        if k not in p:
            raise KeyError(f"unknown parameter {k!r}")
        p[k] = v
    return p


# ---- vision randomizations: Table vision-randomization -------------------------
import math as _math  # noqa: E402

VISION = {
    "cam_pos_range": 1.5e-3,                      # "camera position +-1.5 mm"
    "cam_rot_max": 3.0 * _math.pi / 180.0,        # "camera rotation 0-3 deg around a random axis"
    "cam_fov_range": 1.0 * _math.pi / 180.0,      # "camera field of view +-1 deg" (radians)
    "robot_metallic_lo": 0.05, "robot_metallic_hi": 0.25,   # "robot material metallic level 5%-25%"
    "robot_gloss_lo": 0.0, "robot_gloss_hi": 1.0,           # "robot material glossiness level 0%-100%"
    # calibrated object HSV: "around calibrated values from real-world measurements",
    # values not given -- workload choice (parity unpinned), picked so hue wraps and saturation clamps
    "obj_hue_cal": 0.005, "obj_sat_cal": 0.9, "obj_val_cal": 0.5,
    "obj_hue_range": 0.01, "obj_sat_range": 0.15, "obj_val_range": 0.15,   # "+-1 %", "+-15 %", "+-15 %"
    "obj_metallic_lo": 0.05, "obj_metallic_hi": 0.15,       # "object metallic level 5%-15%"
    "obj_gloss_lo": 0.05, "obj_gloss_hi": 0.15,             # "object glossiness level 5%-15%"
    "lights_min": 4, "lights_max": 6,                       # "number of lights 4-6"
    "light_rel_lo": 1.0, "light_rel_hi": 5.0,               # "light relative intensity 1-5"
    "light_total_lo": 0.0, "light_total_hi": 15.0,          # "total light intensity 0-15"
    "contrast_lo": 0.5, "contrast_hi": 1.5,                 # "image contrast adjustment 50%-150%"
    "noise_std_lo": 0.1, "noise_std_hi": 0.1,               # "additive per-pixel Gaussian noise +-10%" [V6]
    "std_floor": 1e-8,                                      # constant images
}
# the paper's vision batch: 64 samples x 3 cameras = 192 RGB images of 200 x 200 x 8-bit
VISION_BATCH_SAMPLES, VISION_CAMERAS, VISION_H, VISION_W, VISION_C = 64, 3, 200, 200, 3


def vision_preset(**overrides) -> dict:
    p = copy.deepcopy(VISION)
    for k, v in overrides.items():
        if k not in p:
            raise KeyError(f"unknown vision parameter {k!r}")
        p[k] = v
    return p


# vision-model training pose augmentation: keep 20 %, rotate 90 deg about a main axis
# 40 %, jitter position + rotation 40 %.  Jitter stds are not given in the paper (SPEC.md:632's
# 5 mm / 0.05 rad) -- parity unpinned workload choice.
POSE_AUG = {"p_keep": 0.2, "p_rot90": 0.4, "pos_std": 5e-3, "rot_std": 0.05}


def pose_preset(**overrides) -> dict:
    p = dict(POSE_AUG)
    for k, v in overrides.items():
        if k not in p:
            raise KeyError(f"unknown pose-augmentation parameter {k!r}")
        p[k] = v
    return p


def poses(n: int, seed: int = SEED_WORKLOAD):
    """Seeded object poses [n][7] float32: position around the palm + a uniform unit quaternion."""
    import numpy as np
    rng = np.random.default_rng(seed)
    out = np.empty((n, 7))
    out[:, 0:3] = np.array([0.0, 0.04, 0.03]) + 0.01 * rng.standard_normal((n, 3))
    q = rng.standard_normal((n, 4))
    out[:, 3:7] = q / np.linalg.norm(q, axis=1, keepdims=True)
    return out.astype(np.float32)
