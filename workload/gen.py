"""Seeded synthetic Shadow-hand-shaped inputs (SURVEY.md §8(d) recipe).

* actions[e][j] = -1 + (2k+1)/11, k ~ U{0..10}: the paper's 11-bin action grid (PAPER.md:591,
  731; bin centres SPEC.md:103).  Includes exact 0 (k = 5) and values near +-1.
* raw_obs[e] = [tips 5x3, object position 3, object quaternion (w,x,y,z) 4, goal quaternion 4]
  in metres, hand frame: fingertips at nominal points on an arc ~25 mm apart plus N(0, (5 mm)^2)
  per axis per frame; object at (0, 0.04, 0.03) + N(0, (10 mm)^2) -- giving ~7 % occluded tips
  at r = 15 mm (SURVEY aim 2-10 %); quaternions uniform
  (normalised N(0, I4)).
* Frames: a ring of F frames; step t uses frame t mod F.

No randomization arithmetic of the method lives here.
"""
from __future__ import annotations

import numpy as np

from .presets import N_ACT, N_TIPS, OBS_IN, SEED_WORKLOAD

# nominal fingertip points: arc of radius 0.1 m, 0.25 rad apart (chord 24.9 mm)
_ARC_R = 0.10
_ARC_STEP = 0.25
TIP_NOMINAL = np.array(
    [[_ARC_R * np.sin((i - 2) * _ARC_STEP), -0.03 + _ARC_R * np.cos((i - 2) * _ARC_STEP), 0.03]
     for i in range(N_TIPS)], dtype=np.float64)
OBJ_NOMINAL = np.array([0.0, 0.04, 0.03])
TIP_JITTER = 0.005
OBJ_JITTER = 0.010


def actions(rng: np.random.Generator, n_env: int) -> np.ndarray:
    k = rng.integers(0, 11, size=(n_env, N_ACT))
    return (-1.0 + (2.0 * k + 1.0) / 11.0).astype(np.float32)


def _unit_quats(rng: np.random.Generator, n: int) -> np.ndarray:
    q = rng.standard_normal((n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    return q


def raw_obs(rng: np.random.Generator, n_env: int) -> np.ndarray:
    o = np.empty((n_env, OBS_IN), dtype=np.float64)
    tips = TIP_NOMINAL[None, :, :] + TIP_JITTER * rng.standard_normal((n_env, N_TIPS, 3))
    o[:, 0:15] = tips.reshape(n_env, 15)
    o[:, 15:18] = OBJ_NOMINAL[None, :] + OBJ_JITTER * rng.standard_normal((n_env, 3))
    o[:, 18:22] = _unit_quats(rng, n_env)
    o[:, 22:26] = _unit_quats(rng, n_env)
    return o.astype(np.float32)


def frames(n_env: int, n_frames: int, seed: int = SEED_WORKLOAD):
    """(actions [F][n][20] f32, raw_obs [F][n][26] f32), C-contiguous."""
    rng = np.random.default_rng(seed)
    acts = np.empty((n_frames, n_env, N_ACT), dtype=np.float32)
    obs = np.empty((n_frames, n_env, OBS_IN), dtype=np.float32)
    for f in range(n_frames):
        acts[f] = actions(rng, n_env)
        obs[f] = raw_obs(rng, n_env)
    return acts, obs


def reset_mask_ring(n_env: int, t: int, period: int = 10) -> np.ndarray:
    """Config 5 deterministic reset pattern: env e resets at step t when (e + t) mod period == 0."""
    e = np.arange(n_env)
    return ((e + t) % period == 0).astype(np.uint8)


def reset_mask_bernoulli(rng: np.random.Generator, n_env: int, prob: float = 0.1) -> np.ndarray:
    return (rng.random(n_env) < prob).astype(np.uint8)


def occlusion_rate(obs: np.ndarray, r: float = 0.015) -> float:
    """Fraction of fingertips with another tip or the object centre closer than r (reporting
    helper for the generator's recipe; float64 numpy, not the method's exact test)."""
    tips = obs[..., 0:15].reshape(obs.shape[:-1] + (N_TIPS, 3)).astype(np.float64)
    obj = obs[..., 15:18].astype(np.float64)
    occ = np.zeros(tips.shape[:-1], dtype=bool)
    for i in range(N_TIPS):
        for j in range(N_TIPS):
            if i != j:
                occ[..., i] |= np.sum((tips[..., i, :] - tips[..., j, :]) ** 2, axis=-1) < r * r
        occ[..., i] |= np.sum((tips[..., i, :] - obj) ** 2, axis=-1) < r * r
    return float(occ.mean())


def images(n: int, h: int, w: int, c: int, seed: int = SEED_WORKLOAD) -> np.ndarray:
    """Synthetic rendered-like u8 images [n][h][w][c] (the paper's camera frames are 200 x 200 x
    8-bit RGB): a per-image linear gradient background, a few flat-coloured
    rectangles (a block / hand stand-in), plus mild sensor-like noise, clipped to [0, 255].
    Per-image brightness and contrast vary, so the normalisation sees a spread of means / stds."""
    rng = np.random.default_rng(seed)
    yy = np.linspace(0.0, 1.0, h)[:, None, None]
    xx = np.linspace(0.0, 1.0, w)[None, :, None]
    out = np.empty((n, h, w, c), dtype=np.uint8)
    for i in range(n):
        base = rng.uniform(20, 200, size=(1, 1, c))
        gy, gx = rng.uniform(-60, 60, size=(2, 1, 1, c))
        img = base + gy * yy + gx * xx
        for _ in range(rng.integers(1, 4)):
            y0, x0 = rng.integers(0, h), rng.integers(0, w)
            y1, x1 = min(h, y0 + rng.integers(1, max(2, h // 2))), min(w, x0 + rng.integers(1, max(2, w // 2)))
            img[y0:y1, x0:x1, :] = rng.uniform(0, 255, size=c)
        img = img + rng.normal(0.0, 3.0, size=(h, w, c))
        out[i] = np.clip(np.rint(img), 0, 255).astype(np.uint8)
    return out
