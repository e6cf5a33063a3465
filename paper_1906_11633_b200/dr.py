"""Thin Python binding of libdr.so (include/dr.h) -- argument marshalling only.

Every function has the C-ABI name and argument order.  Tensors must be CUDA, fp32 (u8 for the
reset mask), C-contiguous and of the documented shape; their data pointers are passed straight
through.  PyTorch provides device memory, streams and process groups; every step of the
randomization pipeline runs in the CUDA kernels of libdr.so.  There is no fallback: if the
shared library is missing or fails to load, ``load()`` raises.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libdr.so")
# A/B experiments load an alternative in-tree build (e.g. variants/libdr_m6.so); never a fallback.
_LIB_OVERRIDE = os.environ.get("DR_LIB")

ABI_VERSION = 2
N_STAT_SLOTS = 4
N_ACT, N_TIPS, N_SUB, MAX_PHYS, OBS_IN, OBS_OUT, N_STATS = 20, 5, 10, 256, 26, 22, 32
TIMING, ACT_NOISE, DELAY, BACKLASH, OBS_NOISE = 1, 2, 4, 8, 16
DROPOUT, OCCLUSION, FORCE, PHYS, ALL = 32, 64, 128, 256, 0x1FF
SMOOTH, SUBSTEP_BACKLASH, ALL_EXT = 512, 1024, 0x7FF

STATUS = {0: "DR_OK", -1: "DR_EINVAL", -2: "DR_ENOTINIT", -3: "DR_EALREADY", -4: "DR_ENOMEM",
          -5: "DR_ECUDA", -6: "DR_EUNSUPPORTED"}

STAT_NAMES = {0: "envs", 1: "delayed", 2: "drop_init", 3: "masked", 4: "occluded", 5: "held",
              6: "force_trig", 7: "rail_hits", 8: "alpha_one", 9: "alpha_lt1", 10: "resets",
              11: "act_clamps", 16: "sum_dt", 17: "sum_dt2", 18: "sum_da", 19: "sum_da2",
              20: "sum_abs_bl", 21: "sum_zu2", 22: "sum_ztip2", 23: "sum_f2"}


class DRError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


class PhysDesc(C.Structure):
    _fields_ = [("kind", C.c_uint32), ("_pad", C.c_uint32), ("a", C.c_double), ("b", C.c_double),
                ("base", C.c_double)]


class DrParams(C.Structure):
    _fields_ = [
        ("abi_version", C.c_uint32), ("struct_size", C.c_uint32), ("layer_mask", C.c_uint32), ("_pad0", C.c_uint32),
        ("n_act", C.c_int32), ("n_tips", C.c_int32), ("n_substeps", C.c_int32), ("_pad1", C.c_int32),
        ("env_offset", C.c_int64), ("n_env_global", C.c_int64),
        ("act_sigma_uadd", C.c_double), ("act_sigma_cadd", C.c_double), ("act_sigma_mult", C.c_double),
        ("delay_prob", C.c_double),
        ("dt_base", C.c_double), ("lambda_lo", C.c_double), ("lambda_hi", C.c_double), ("step_nominal", C.c_double),
        ("delta_cal_neg", C.c_double * N_ACT), ("delta_cal_pos", C.c_double * N_ACT),
        ("delta_jitter_std", C.c_double), ("backlash_eps", C.c_double),
        ("tip_corr", C.c_double), ("tip_uncorr", C.c_double), ("obj_corr", C.c_double), ("obj_uncorr", C.c_double),
        ("rot_corr", C.c_double), ("rot_uncorr", C.c_double), ("tip_marker", C.c_double), ("base_marker", C.c_double),
        ("base_marker_to_tips", C.c_int32), ("dropout_hold_steps", C.c_int32),
        ("dropout_rate_hz", C.c_double), ("occl_dist", C.c_double),
        ("force_p_lo", C.c_double), ("force_p_hi", C.c_double), ("force_accel_std", C.c_double),
        ("force_decay_per_step", C.c_double),
        ("act_smooth_coef", C.c_double),
        ("n_phys", C.c_int32), ("mass_index", C.c_int32),
        ("phys", PhysDesc * MAX_PHYS),
        ("workspace", C.c_void_p), ("workspace_bytes", C.c_size_t), ("stream", C.c_void_p),
    ]


class DrEnvState(C.Structure):
    _fields_ = [
        ("episode", C.c_uint32), ("delay_bits", C.c_uint32), ("p_index", C.c_uint32), ("t_force", C.c_uint32),
        ("flags", C.c_uint32), ("k_f", C.c_uint32), ("lambda_", C.c_float), ("mass", C.c_float),
        ("dneg", C.c_float * N_ACT), ("dpos", C.c_float * N_ACT), ("c_act", C.c_float * N_ACT),
        ("off_tip", C.c_float * 15), ("c_obj", C.c_float * 3), ("q_c", C.c_float * 4),
        ("prev", C.c_float * N_ACT), ("slack", C.c_float * N_ACT), ("last", C.c_float * 15),
        ("f_trig", C.c_float * 3), ("ema", C.c_float * N_ACT),
    ]


_lib = None


def load():
    """Load libdr.so (building it first if the sources are newer).  Raises if unavailable."""
    global _lib
    if _lib is not None:
        return _lib
    from . import build as _build
    try:
        _build.build()
    except Exception as ex:  # nvcc missing on a box with a prebuilt .so is fine
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libdr.so missing and cannot be built: {ex}") from ex
    L = C.CDLL(os.path.join(PKG, _LIB_OVERRIDE) if _LIB_OVERRIDE else LIB_PATH)
    vp, fp = C.c_void_p, C.c_void_p
    L.dr_params_default.argtypes = [C.POINTER(DrParams)]
    L.dr_init.argtypes = [C.POINTER(DrParams), C.c_int64, C.c_uint64]
    L.dr_reset.argtypes = [vp]
    L.dr_update_params.argtypes = [C.POINTER(DrParams)]
    L.dr_step.argtypes = [fp] * 6
    L.dr_step_host.argtypes = [fp] * 6
    L.dr_step_substeps.argtypes = [fp] * 7
    L.dr_finalize.argtypes = []
    L.dr_workspace_bytes.argtypes = [C.POINTER(DrParams), C.c_int64]
    L.dr_workspace_bytes.restype = C.c_size_t
    L.dr_set_stream.argtypes = [vp]
    L.dr_set_occlusion_input.argtypes = [vp]
    L.dr_synchronize.argtypes = []
    L.dr_phys_params.restype = C.c_void_p
    L.dr_n_phys.restype = C.c_int
    L.dr_stats.argtypes = [C.c_int]
    L.dr_stats.restype = C.c_void_p
    L.dr_set_stats_buffer.argtypes = [vp]
    L.dr_step_index.restype = C.c_uint64
    L.dr_step_index_sync.restype = C.c_uint64
    L.dr_set_step_index.argtypes = [C.c_uint64]
    L.dr_state_bytes.restype = C.c_size_t
    L.dr_state_export.argtypes = [vp, C.c_int64, C.c_int64]
    L.dr_state_import.argtypes = [vp, C.c_int64, C.c_int64]
    L.dr_last_error.restype = C.c_char_p
    L.dr_kernel_launches.restype = C.c_uint64
    L.dr_abi_version.restype = C.c_uint32
    L.dr_phys_export.argtypes = [vp, C.c_int64, C.c_int64]
    L.dr_debug_philox.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, vp]
    L.dr_debug_philox.restype = C.c_int
    L.dr_debug_philox_keyed.argtypes = [vp, vp, vp, C.c_uint64, vp]
    L.dr_debug_philox_keyed.restype = C.c_int
    for f in ("dr_params_default", "dr_init", "dr_update_params", "dr_reset", "dr_step", "dr_step_substeps", "dr_step_host", "dr_finalize",
              "dr_set_stream", "dr_set_occlusion_input", "dr_synchronize", "dr_set_stats_buffer", "dr_set_step_index",
              "dr_state_export", "dr_state_import", "dr_phys_export"):
        getattr(L, f).restype = C.c_int
    if L.dr_abi_version() != ABI_VERSION:
        raise RuntimeError("libdr.so ABI version mismatch")
    _lib = L
    return L


def _check(rc):
    if rc != 0:
        raise DRError(rc, load().dr_last_error().decode())
    return rc


def _ptr(t, shape=None, dtype=None, name="tensor"):
    """Data pointer of a CUDA tensor after checking dtype/shape/contiguity (marshalling only)."""
    if t is None:
        return None
    import torch
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name}: expected a torch.Tensor")
    if not t.is_cuda:
        raise ValueError(f"{name}: must be a CUDA tensor")
    if dtype is not None and t.dtype != dtype:
        raise ValueError(f"{name}: dtype {t.dtype} != {dtype}")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name}: shape {tuple(t.shape)} != {tuple(shape)}")
    if not t.is_contiguous():
        raise ValueError(f"{name}: must be contiguous")
    return C.c_void_p(t.data_ptr())


# ---------------------------------------------------------------------------------------------
# parameters
# ---------------------------------------------------------------------------------------------
def dr_params_default() -> DrParams:
    p = DrParams()
    _check(load().dr_params_default(C.byref(p)))
    return p


def params_from_preset(preset: dict, env_offset: int = 0, n_env_global: int = 0, stream=None,
                       workspace=None) -> DrParams:
    """Fill a DrParams from a workload preset dict (field names match dr.h)."""
    p = dr_params_default()
    for name, _ in DrParams._fields_:
        if name in preset and name not in ("phys", "delta_cal_neg", "delta_cal_pos"):
            setattr(p, name, preset[name])
    for j in range(N_ACT):
        p.delta_cal_neg[j] = preset["delta_cal_neg"][j]
        p.delta_cal_pos[j] = preset["delta_cal_pos"][j]
    for i, (k, a, b, base) in enumerate(preset["phys"]):
        p.phys[i].kind, p.phys[i].a, p.phys[i].b, p.phys[i].base = k, a, b, base
    p.env_offset = env_offset
    p.n_env_global = n_env_global
    if stream is not None:
        p.stream = C.c_void_p(stream)
    if workspace is not None:
        p.workspace = C.c_void_p(workspace.data_ptr())
        p.workspace_bytes = workspace.numel() * workspace.element_size()
    return p


# ---------------------------------------------------------------------------------------------
# C-ABI functions, same names
# ---------------------------------------------------------------------------------------------
def dr_init(params: DrParams, n_env: int, seed: int):
    return _check(load().dr_init(C.byref(params), n_env, seed))


def dr_update_params(params: DrParams):
    return _check(load().dr_update_params(C.byref(params)))


def dr_reset(env_mask=None, n_env=None):
    m = None
    if env_mask is not None:
        import torch
        m = _ptr(env_mask, (n_env,) if n_env else None, torch.uint8, "env_mask")
    return _check(load().dr_reset(m))


def dr_step(actions, raw_obs, out_actions, out_obs, out_dt, out_force):
    import torch
    n = actions.shape[0]
    f = torch.float32
    return _check(load().dr_step(_ptr(actions, (n, N_ACT), f, "actions"), _ptr(raw_obs, (n, OBS_IN), f, "raw_obs"),
                                 _ptr(out_actions, (n, N_ACT), f, "out_actions"),
                                 _ptr(out_obs, (n, OBS_OUT), f, "out_obs"), _ptr(out_dt, (n, N_SUB), f, "out_dt"),
                                 _ptr(out_force, (n, 3), f, "out_force")))


def dr_step_substeps(actions, raw_obs, out_actions, out_actions_sub, out_obs, out_dt, out_force):
    import torch
    n = actions.shape[0]
    f = torch.float32
    return _check(load().dr_step_substeps(
        _ptr(actions, (n, N_ACT), f, "actions"), _ptr(raw_obs, (n, OBS_IN), f, "raw_obs"),
        _ptr(out_actions, (n, N_ACT), f, "out_actions"), _ptr(out_actions_sub, (n, N_SUB, N_ACT), f, "out_actions_sub"),
        _ptr(out_obs, (n, OBS_OUT), f, "out_obs"), _ptr(out_dt, (n, N_SUB), f, "out_dt"),
        _ptr(out_force, (n, 3), f, "out_force")))


def _host_ptr(t, shape, name):
    import torch
    if t.is_cuda or t.dtype != torch.float32 or tuple(t.shape) != tuple(shape) or not t.is_contiguous():
        raise ValueError(f"{name}: expected a contiguous host float32 tensor of shape {shape}")
    return C.c_void_p(t.data_ptr())


def dr_step_host(actions, raw_obs, out_actions, out_obs, out_dt, out_force):
    n = actions.shape[0]
    return _check(load().dr_step_host(_host_ptr(actions, (n, N_ACT), "actions"),
                                      _host_ptr(raw_obs, (n, OBS_IN), "raw_obs"),
                                      _host_ptr(out_actions, (n, N_ACT), "out_actions"),
                                      _host_ptr(out_obs, (n, OBS_OUT), "out_obs"),
                                      _host_ptr(out_dt, (n, N_SUB), "out_dt"),
                                      _host_ptr(out_force, (n, 3), "out_force")))


def dr_finalize():
    return _check(load().dr_finalize())


def dr_workspace_bytes(params: DrParams, n_env: int) -> int:
    return load().dr_workspace_bytes(C.byref(params), n_env)


def dr_set_stream(stream_handle: int):
    return _check(load().dr_set_stream(C.c_void_p(stream_handle)))


def dr_set_occlusion_input(mask=None, n_env=None):
    """mask: CUDA uint8 [n_env] (bit i = tip i occluded), or None for the distance rule."""
    import torch
    m = None if mask is None else _ptr(mask, (n_env,) if n_env else None, torch.uint8, "occl_mask")
    return _check(load().dr_set_occlusion_input(m))


def dr_synchronize():
    return _check(load().dr_synchronize())


def dr_phys_params() -> int:
    return load().dr_phys_params() or 0


def dr_n_phys() -> int:
    return load().dr_n_phys()


def dr_stats(slot: int) -> int:
    return load().dr_stats(slot) or 0


def dr_set_stats_buffer(buf=None):
    import torch
    return _check(load().dr_set_stats_buffer(None if buf is None else _ptr(buf, (N_STAT_SLOTS, N_STATS), torch.float64,
                                                                           "stats")))


def dr_step_index() -> int:
    return load().dr_step_index()


def dr_step_index_sync() -> int:
    return load().dr_step_index_sync()


def dr_set_step_index(t: int):
    return _check(load().dr_set_step_index(t))


def dr_state_bytes() -> int:
    return load().dr_state_bytes()


def dr_state_export(env_lo: int = 0, env_hi: int = 0):
    """Returns a ctypes array of DrEnvState (blocking)."""
    n = env_hi - env_lo if (env_lo or env_hi) else dr_state_bytes() // C.sizeof(DrEnvState)
    buf = (DrEnvState * n)()
    _check(load().dr_state_export(C.cast(buf, C.c_void_p), env_lo, env_hi))
    return buf


def dr_state_import(states, env_lo: int = 0, env_hi: int = 0):
    return _check(load().dr_state_import(C.cast(states, C.c_void_p), env_lo, env_hi))


def dr_last_error() -> str:
    return load().dr_last_error().decode()


def dr_kernel_launches() -> int:
    return load().dr_kernel_launches()


# ---------------------------------------------------------------------------------------------
# helpers (marshalling of results; no arithmetic of the method)
# ---------------------------------------------------------------------------------------------
def states_to_numpy(states) -> dict:
    """ctypes DrEnvState array -> dict of numpy arrays (field name -> [n, ...])."""
    import numpy as np
    raw = np.frombuffer(states, dtype=np.uint32).reshape(len(states), -1)
    out, off = {}, 0
    for name, ty in DrEnvState._fields_:
        n = ty._length_ if hasattr(ty, "_length_") else 1
        col = raw[:, off:off + n]
        if (hasattr(ty, "_type_") and ty._type_ is C.c_float) or ty is C.c_float:
            col = col.view(np.float32)
        out["lambda" if name == "lambda_" else name] = col if n > 1 else col[:, 0]
        off += n
    return out


def dr_debug_philox(domain: int, channel: int, block: int, out):
    import torch
    return _check(load().dr_debug_philox(domain, channel, block, _ptr(out, None, torch.int32, "out")))


def dr_debug_philox_keyed(ctr, key, out, stream=None):
    """ctr, out: CUDA int32 [n][4]; key: CUDA int32 [n][2] (uint32 bit patterns)."""
    import torch
    n = ctr.shape[0]
    s = stream if stream is not None else torch.cuda.current_stream()
    return _check(load().dr_debug_philox_keyed(_ptr(ctr, (n, 4), torch.int32, "ctr"), _ptr(key, (n, 2), torch.int32, "key"),
                                               _ptr(out, (n, 4), torch.int32, "out"), n, C.c_void_p(s.cuda_stream)))


def dr_phys_export(env_lo: int = 0, env_hi: int = 0):
    """[hi - lo][n_phys] float32 numpy copy of the episode's physical parameters (blocking)."""
    import numpy as np
    n_phys = dr_n_phys()
    n = env_hi - env_lo if (env_lo or env_hi) else dr_state_bytes() // C.sizeof(DrEnvState)
    out = np.empty((n, n_phys), dtype=np.float32)
    _check(load().dr_phys_export(out.ctypes.data_as(C.c_void_p), env_lo, env_hi))
    return out
