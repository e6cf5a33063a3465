"""ctypes wrapper of liboracle.so -- TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` / ``--impl reference``
legs may import this module.  It declares its own struct layouts (mirroring oracle.h) and
imports nothing from the product package ``paper_1906_11633_b200``.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
LIB_OMP_PATH = os.path.join(HERE, "liboracle_omp.so")   # same source, -fopenmp: per-env loops over all cores
SOURCES = [os.path.join(HERE, "oracle.c"), os.path.join(HERE, "oracle_vision.c")]
HEADERS = [os.path.join(HERE, "oracle.h")]

N_ACT, N_TIPS, N_SUB, MAX_PHYS, OBS_IN, OBS_OUT, N_STATS = 20, 5, 10, 256, 26, 22, 32


def build(force: bool = False) -> str:
    """gcc -O2 -ffp-contract=off: plain scalar fp64, no FMA contraction.  Built twice: single-thread
    (liboracle.so) and with -fopenmp (liboracle_omp.so, the all-core CPU baseline)."""
    newest = max(os.path.getmtime(p) for p in SOURCES + HEADERS)
    for path, extra in ((LIB_PATH, []), (LIB_OMP_PATH, ["-fopenmp"])):
        if force or not os.path.exists(path) or os.path.getmtime(path) < newest:
            cmd = ["gcc", "-O2", "-std=c99", "-D_DEFAULT_SOURCE", "-ffp-contract=off", "-fno-fast-math",
                   "-fPIC", "-shared", "-Wall", "-Wno-unknown-pragmas"] + extra + ["-o", path] + SOURCES + ["-lm"]
            subprocess.check_call(cmd)
    return LIB_PATH


class PhysDesc(C.Structure):
    _fields_ = [("kind", C.c_int32), ("a", C.c_double), ("b", C.c_double), ("base", C.c_double)]


class OrcParams(C.Structure):
    _fields_ = [
        ("layer_mask", C.c_uint32),
        ("act_sigma_uadd", C.c_double), ("act_sigma_cadd", C.c_double),
        ("act_sigma_mult", C.c_double), ("delay_prob", C.c_double),
        ("dt_base", C.c_double), ("lambda_lo", C.c_double), ("lambda_hi", C.c_double),
        ("step_nominal", C.c_double),
        ("delta_cal_neg", C.c_double * N_ACT), ("delta_cal_pos", C.c_double * N_ACT),
        ("delta_jitter_std", C.c_double), ("backlash_eps", C.c_double),
        ("tip_corr", C.c_double), ("tip_uncorr", C.c_double), ("obj_corr", C.c_double),
        ("obj_uncorr", C.c_double), ("rot_corr", C.c_double), ("rot_uncorr", C.c_double),
        ("tip_marker", C.c_double), ("base_marker", C.c_double),
        ("base_marker_to_tips", C.c_int32),
        ("dropout_rate_hz", C.c_double), ("dropout_hold_steps", C.c_int32), ("occl_dist", C.c_double),
        ("force_p_lo", C.c_double), ("force_p_hi", C.c_double), ("force_accel_std", C.c_double),
        ("force_decay_per_step", C.c_double),
        ("n_phys", C.c_int32), ("mass_index", C.c_int32),
        ("phys", PhysDesc * MAX_PHYS),
        ("act_smooth_coef", C.c_double),
    ]


class OrcEnv(C.Structure):
    _fields_ = [
        ("gid", C.c_int64), ("episode", C.c_uint32),
        ("delay_bits", C.c_uint32), ("p_index", C.c_uint32), ("t_force", C.c_uint32), ("_pad0", C.c_uint32),
        ("p_force", C.c_double), ("lambda_", C.c_double), ("mass", C.c_double),
        ("dneg", C.c_double * N_ACT), ("dpos", C.c_double * N_ACT), ("c_act", C.c_double * N_ACT),
        ("off_tip", C.c_double * 15), ("c_obj", C.c_double * 3), ("q_c", C.c_double * 4),
        ("phys", C.c_double * MAX_PHYS),
        ("prev", C.c_double * N_ACT), ("slack", C.c_double * N_ACT), ("last", C.c_double * 15),
        ("has_last", C.c_int32), ("timer", C.c_int32 * N_TIPS),
        ("f_trig", C.c_double * 3), ("k_f", C.c_uint32), ("_pad1", C.c_uint32),
        ("ema", C.c_double * N_ACT),
    ]


class OrcVisionParams(C.Structure):
    _fields_ = [(n, C.c_double) for n in (
        "cam_pos_range", "cam_rot_max", "cam_fov_range", "robot_metallic_lo", "robot_metallic_hi",
        "robot_gloss_lo", "robot_gloss_hi", "obj_hue_cal", "obj_sat_cal", "obj_val_cal", "obj_hue_range",
        "obj_sat_range", "obj_val_range", "obj_metallic_lo", "obj_metallic_hi", "obj_gloss_lo", "obj_gloss_hi")] + [
        ("lights_min", C.c_int32), ("lights_max", C.c_int32)] + [(n, C.c_double) for n in (
        "light_rel_lo", "light_rel_hi", "light_total_lo", "light_total_hi", "contrast_lo", "contrast_hi",
        "noise_std_lo", "noise_std_hi", "std_floor")]


class OrcPoseAugParams(C.Structure):
    _fields_ = [("p_keep", C.c_double), ("p_rot90", C.c_double), ("pos_std", C.c_double), ("rot_std", C.c_double)]


SCENE_WORDS = 64

_libs = {}


def lib(omp: bool = False):
    """The single-thread oracle library, or (omp=True) the -fopenmp build of the same source."""
    if omp not in _libs:
        build()
        L = C.CDLL(LIB_OMP_PATH if omp else LIB_PATH)
        dp, fp, u8p = C.POINTER(C.c_double), C.POINTER(C.c_float), C.POINTER(C.c_uint8)
        L.orc_init.argtypes = [C.POINTER(OrcParams), C.c_int64, C.POINTER(C.c_int64), C.c_uint64,
                               C.POINTER(C.c_void_p)]
        L.orc_init.restype = C.c_int
        L.orc_free.argtypes = [C.c_void_p]
        L.orc_scene_draw.argtypes = [C.POINTER(OrcVisionParams), C.c_uint64, C.c_uint64, C.c_int64, C.c_int64, dp]
        L.orc_scene_draw.restype = C.c_int
        L.orc_image_augment.argtypes = [C.POINTER(OrcVisionParams), C.c_uint64, C.c_uint64, C.c_int64, u8p,
                                        C.c_int64, C.c_int32, C.c_int32, C.c_int32, dp, dp]
        L.orc_image_augment.restype = C.c_int
        L.orc_pose_augment.argtypes = [C.POINTER(OrcPoseAugParams), C.c_uint64, C.c_uint64, C.c_int64, fp, C.c_int64,
                                       dp, u8p]
        L.orc_pose_augment.restype = C.c_int
        L.orc_update_params.argtypes = [C.c_void_p, C.POINTER(OrcParams)]
        L.orc_update_params.restype = C.c_int
        L.orc_reset.argtypes = [C.c_void_p, u8p]
        L.orc_reset.restype = C.c_int
        L.orc_step.argtypes = [C.c_void_p, fp, fp, dp, dp, dp, dp, dp, dp]
        L.orc_step.restype = C.c_int
        L.orc_step_sub.argtypes = [C.c_void_p, fp, fp, dp, dp, dp, dp, dp, dp, dp]
        L.orc_step_sub.restype = C.c_int
        L.orc_set_occlusion_mask.argtypes = [C.c_void_p, u8p]
        L.orc_step_index.argtypes = [C.c_void_p]
        L.orc_step_index.restype = C.c_uint64
        L.orc_set_step_index.argtypes = [C.c_void_p, C.c_uint64]
        L.orc_get_env.argtypes = [C.c_void_p, C.c_int64, C.POINTER(OrcEnv)]
        L.orc_get_env.restype = C.c_int
        L.orc_set_env.argtypes = [C.c_void_p, C.c_int64, C.POINTER(OrcEnv)]
        L.orc_set_env.restype = C.c_int
        L.orc_force_threshold.argtypes = [C.c_void_p, C.c_uint32]
        L.orc_force_threshold.restype = C.c_uint64
        L.orc_force_p.argtypes = [C.c_void_p, C.c_uint32]
        L.orc_force_p.restype = C.c_double
        L.orc_philox.argtypes = [C.POINTER(C.c_uint32), C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]
        L.orc_uniform.argtypes = [C.c_uint32]
        L.orc_uniform.restype = C.c_double
        L.orc_normal_pair.argtypes = [C.c_uint32, C.c_uint32, dp, dp]
        L.orc_exponential.argtypes = [C.c_uint32, C.c_double]
        L.orc_exponential.restype = C.c_double
        L.orc_rotation.argtypes = [C.c_double, C.POINTER(C.c_uint32), dp]
        L.orc_quat_mul.argtypes = [dp, dp, dp]
        L.orc_backlash.argtypes = [C.c_double] * 6 + [dp, dp, dp]
        L.orc_occluded.argtypes = [fp, fp, C.c_double, C.c_int]
        L.orc_occluded.restype = C.c_int
        L.orc_bernoulli_threshold.argtypes = [C.c_double]
        L.orc_bernoulli_threshold.restype = C.c_uint64
        _libs[omp] = L
    return _libs[omp]


def make_params(preset: dict) -> OrcParams:
    p = OrcParams()
    for name, _ in OrcParams._fields_:
        if name in ("phys", "delta_cal_neg", "delta_cal_pos"):
            continue
        setattr(p, name, preset[name])
    for j in range(N_ACT):
        p.delta_cal_neg[j] = preset["delta_cal_neg"][j]
        p.delta_cal_pos[j] = preset["delta_cal_pos"][j]
    for i, (k, a, b, base) in enumerate(preset["phys"]):
        p.phys[i].kind, p.phys[i].a, p.phys[i].b, p.phys[i].base = k, a, b, base
    return p


def _ptr(a, ct):
    return a.ctypes.data_as(C.POINTER(ct)) if a is not None else None


# ---- scalar hooks --------------------------------------------------------------------------
def philox(ctr, key):
    c = (C.c_uint32 * 4)(*ctr)
    k = (C.c_uint32 * 2)(*key)
    o = (C.c_uint32 * 4)()
    lib().orc_philox(c, k, o)
    return tuple(o)


def uniform(x):
    return lib().orc_uniform(x)


def normal_pair(x, y):
    z0, z1 = C.c_double(), C.c_double()
    lib().orc_normal_pair(x, y, C.byref(z0), C.byref(z1))
    return z0.value, z1.value


def exponential(x, lam):
    return lib().orc_exponential(x, lam)


def rotation(sigma, words):
    w = (C.c_uint32 * 4)(*words)
    q = (C.c_double * 4)()
    lib().orc_rotation(sigma, w, q)
    return tuple(q)


def quat_mul(a, b):
    A, B, O = (C.c_double * 4)(*a), (C.c_double * 4)(*b), (C.c_double * 4)()
    lib().orc_quat_mul(A, B, O)
    return tuple(O)


def backlash(s, a, dneg, dpos, dt, eps=1e-12):
    sn, al, out = C.c_double(), C.c_double(), C.c_double()
    lib().orc_backlash(s, a, dneg, dpos, dt, eps, C.byref(sn), C.byref(al), C.byref(out))
    return sn.value, al.value, out.value


def occluded(tips15, obj3, r, tip):
    t = np.ascontiguousarray(tips15, dtype=np.float32)
    o = np.ascontiguousarray(obj3, dtype=np.float32)
    return bool(lib().orc_occluded(_ptr(t, C.c_float), _ptr(o, C.c_float), r, tip))


def bernoulli_threshold(p):
    return lib().orc_bernoulli_threshold(p)


# ---- vision randomization (Table vision-randomization) ----------------------
def make_vision_params(preset: dict) -> OrcVisionParams:
    p = OrcVisionParams()
    for name, _ in OrcVisionParams._fields_:
        setattr(p, name, preset[name])
    return p


def scene_draw(preset: dict, seed: int, batch: int, n: int, sample_offset: int = 0):
    """[n][64] fp64 appearance draws (field order: oracle.h orc_scene_draw)."""
    p = make_vision_params(preset)
    out = np.zeros((n, SCENE_WORDS))
    rc = lib().orc_scene_draw(C.byref(p), C.c_uint64(seed), C.c_uint64(batch), sample_offset, n,
                              _ptr(out, C.c_double))
    if rc != 0:
        raise ValueError(f"orc_scene_draw failed: {rc}")
    return out


def image_augment(preset: dict, seed: int, batch: int, images, image_offset: int = 0):
    """images: u8 [n][H][W][C] -> (fp64 [n][H][W][C], fp64 [n][4] = mean, std, contrast, noise std)."""
    x = np.ascontiguousarray(images, dtype=np.uint8)
    n, h, w, c = x.shape
    p = make_vision_params(preset)
    out = np.empty(x.shape, dtype=np.float64)
    st = np.empty((n, 4))
    rc = lib().orc_image_augment(C.byref(p), C.c_uint64(seed), C.c_uint64(batch), image_offset,
                                 _ptr(x, C.c_uint8), n, h, w, c, _ptr(out, C.c_double), _ptr(st, C.c_double))
    if rc != 0:
        raise ValueError(f"orc_image_augment failed: {rc}")
    return out, st


def pose_augment(preset: dict, seed: int, batch: int, poses, offset: int = 0):
    """poses float32 [n][7] (pos, quat wxyz) -> (fp64 [n][7], branch u8 [n])."""
    x = np.ascontiguousarray(poses, dtype=np.float32)
    n = x.shape[0]
    p = OrcPoseAugParams(*(preset[k] for k in ("p_keep", "p_rot90", "pos_std", "rot_std")))
    out = np.empty((n, 7))
    br = np.empty(n, dtype=np.uint8)
    rc = lib().orc_pose_augment(C.byref(p), C.c_uint64(seed), C.c_uint64(batch), offset, _ptr(x, C.c_float), n,
                                _ptr(out, C.c_double), _ptr(br, C.c_uint8))
    if rc != 0:
        raise ValueError(f"orc_pose_augment failed: {rc}")
    return out, br


# ---- context -------------------------------------------------------------------------------
class Oracle:
    """fp64 CPU oracle over a list of global env ids (any subset of a larger run)."""

    def __init__(self, preset: dict, n_env: int, seed: int, gids=None, omp: bool = False):
        """omp=True: the all-core (-fopenmp) build of the same oracle (bit-identical results)."""
        L = self._L = lib(omp)
        self._params = make_params(preset)
        self.n = int(n_env)
        if gids is None:
            gids = np.arange(self.n, dtype=np.int64)
        self.gids = np.ascontiguousarray(gids, dtype=np.int64)
        assert self.gids.shape == (self.n,)
        h = C.c_void_p()
        rc = L.orc_init(C.byref(self._params), self.n, _ptr(self.gids, C.c_int64), C.c_uint64(seed), C.byref(h))
        if rc != 0:
            raise ValueError(f"orc_init failed: {rc}")
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            self._L.orc_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_occlusion_mask(self, mask):
        """Simulator occlusion bits [n] u8 (bit i = tip i), or None for the distance rule.  The
        array is kept alive here and re-read at every step (update it in place)."""
        self._occl = None if mask is None else np.ascontiguousarray(mask, dtype=np.uint8)
        self._L.orc_set_occlusion_mask(self._h, None if self._occl is None else _ptr(self._occl, C.c_uint8))
        return self._occl

    def update_params(self, preset: dict):
        """Swap the parameter set mid-run: later draws use it."""
        self._params = make_params(preset)
        rc = self._L.orc_update_params(self._h, C.byref(self._params))
        if rc != 0:
            raise ValueError(f"orc_update_params failed: {rc}")

    def reset(self, mask=None):
        m = None if mask is None else np.ascontiguousarray(mask, dtype=np.uint8)
        if m is not None:
            assert m.shape == (self.n,)
        rc = self._L.orc_reset(self._h, _ptr(m, C.c_uint8))
        assert rc == 0

    def step(self, actions, raw_obs, want_margin=False, want_sub=False):
        a = np.ascontiguousarray(actions, dtype=np.float32)
        o = np.ascontiguousarray(raw_obs, dtype=np.float32)
        assert a.shape == (self.n, N_ACT) and o.shape == (self.n, OBS_IN)
        out = {
            "out_actions": np.empty((self.n, N_ACT)),
            "out_obs": np.empty((self.n, OBS_OUT)),
            "out_dt": np.empty((self.n, N_SUB)),
            "out_force": np.empty((self.n, 3)),
            "stats": np.empty(N_STATS),
        }
        margin = np.empty((self.n, N_ACT)) if want_margin else None
        sub = np.empty((self.n, N_SUB, N_ACT)) if want_sub else None
        dp = C.c_double
        rc = self._L.orc_step_sub(self._h, _ptr(a, C.c_float), _ptr(o, C.c_float),
                                _ptr(out["out_actions"], dp), _ptr(sub, dp), _ptr(out["out_obs"], dp),
                                _ptr(out["out_dt"], dp), _ptr(out["out_force"], dp),
                                _ptr(out["stats"], dp), _ptr(margin, dp))
        if want_sub:
            out["out_actions_sub"] = sub
        assert rc == 0
        if want_margin:
            out["margin"] = margin
        return out

    @property
    def step_index(self):
        return self._L.orc_step_index(self._h)

    @step_index.setter
    def step_index(self, t):
        self._L.orc_set_step_index(self._h, t)

    def env(self, i) -> dict:
        e = OrcEnv()
        assert self._L.orc_get_env(self._h, i, C.byref(e)) == 0
        d = {}
        for name, ty in OrcEnv._fields_:
            if name.startswith("_pad"):
                continue
            v = getattr(e, name)
            if hasattr(v, "_length_"):
                v = np.array(v[:])
            d["lambda" if name == "lambda_" else name] = v
        return d

    def set_env(self, i, d: dict):
        """State import of env i from a dict shaped like env(i) (missing keys keep their value)."""
        e = OrcEnv()
        assert self._L.orc_get_env(self._h, i, C.byref(e)) == 0
        for name, _ in OrcEnv._fields_:
            key = "lambda" if name == "lambda_" else name
            if name.startswith("_pad") or key not in d:
                continue
            v = d[key]
            cur = getattr(e, name)
            if hasattr(cur, "_length_"):
                vals = np.asarray(v).ravel()
                assert len(vals) == cur._length_, name
                for k in range(cur._length_):
                    cur[k] = vals[k].item()
            else:
                setattr(e, name, v.item() if hasattr(v, "item") else v)
        assert self._L.orc_set_env(self._h, i, C.byref(e)) == 0

    def force_threshold(self, j):
        return self._L.orc_force_threshold(self._h, j)

    def force_p(self, j):
        return self._L.orc_force_p(self._h, j)
