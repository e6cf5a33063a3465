"""Thin binding of libdr.so's vision randomizations (include/dr_vision.h) -- marshalling only.

Context-free calls: each takes the seed, the batch index and a CUDA stream (default: torch's
current stream).  Tensors must be CUDA, contiguous, of the documented dtype and shape.
"""
from __future__ import annotations

import ctypes as C

from . import dr

SCENE_WORDS = 64
N_CAMERAS, MAX_LIGHTS = 3, 6

_FIELDS = [(n, C.c_double) for n in (
    "cam_pos_range", "cam_rot_max", "cam_fov_range", "robot_metallic_lo", "robot_metallic_hi",
    "robot_gloss_lo", "robot_gloss_hi", "obj_hue_cal", "obj_sat_cal", "obj_val_cal", "obj_hue_range",
    "obj_sat_range", "obj_val_range", "obj_metallic_lo", "obj_metallic_hi", "obj_gloss_lo", "obj_gloss_hi")] + [
    ("lights_min", C.c_int32), ("lights_max", C.c_int32)] + [(n, C.c_double) for n in (
    "light_rel_lo", "light_rel_hi", "light_total_lo", "light_total_hi", "contrast_lo", "contrast_hi",
    "noise_std_lo", "noise_std_hi", "std_floor")]


class DrVisionParams(C.Structure):
    _fields_ = [("abi_version", C.c_uint32), ("struct_size", C.c_uint32)] + _FIELDS


class DrPoseAugParams(C.Structure):
    _fields_ = [("abi_version", C.c_uint32), ("struct_size", C.c_uint32), ("p_keep", C.c_double),
                ("p_rot90", C.c_double), ("pos_std", C.c_double), ("rot_std", C.c_double)]


_ready = False


def _lib():
    global _ready
    L = dr.load()
    if not _ready:
        vp = C.c_void_p
        L.dr_vision_params_default.argtypes = [C.POINTER(DrVisionParams)]
        L.dr_scene_draw_batch.argtypes = [C.POINTER(DrVisionParams), C.c_uint64, C.c_uint64, C.c_int64, C.c_int64, vp, vp]
        L.dr_image_augment.argtypes = [C.POINTER(DrVisionParams), C.c_uint64, C.c_uint64, C.c_int64, vp, C.c_int64,
                                       C.c_int32, C.c_int32, C.c_int32, vp, vp, vp]
        L.dr_total_kernel_launches.restype = C.c_uint64
        L.dr_pose_aug_params_default.argtypes = [C.POINTER(DrPoseAugParams)]
        L.dr_pose_augment.argtypes = [C.POINTER(DrPoseAugParams), C.c_uint64, C.c_uint64, C.c_int64, vp, C.c_int64,
                                      vp, vp, vp]
        for f in ("dr_vision_params_default", "dr_scene_draw_batch", "dr_image_augment", "dr_pose_aug_params_default",
                  "dr_pose_augment"):
            getattr(L, f).restype = C.c_int
        _ready = True
    return L


def dr_vision_params_default() -> DrVisionParams:
    p = DrVisionParams()
    dr._check(_lib().dr_vision_params_default(C.byref(p)))
    return p


def params_from_preset(preset: dict) -> DrVisionParams:
    p = dr_vision_params_default()
    for name, _ in _FIELDS:
        if name in preset:
            setattr(p, name, preset[name])
    return p


def _stream(stream):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def dr_scene_draw_batch(params: DrVisionParams, seed: int, batch_index: int, out, sample_offset: int = 0,
                        stream=None):
    """out: CUDA int32/float32 tensor [n][64] (the dr_scene_draw records)."""
    n = out.shape[0]
    ptr = dr._ptr(out, (n, SCENE_WORDS), None, "out")
    return dr._check(_lib().dr_scene_draw_batch(C.byref(params), C.c_uint64(seed), C.c_uint64(batch_index),
                                                sample_offset, n, ptr, _stream(stream)))


def dr_image_augment(params: DrVisionParams, seed: int, batch_index: int, images, out, img_stats=None,
                     image_offset: int = 0, stream=None):
    """images: CUDA uint8 [n][H][W][C]; out: CUDA float32 same shape; img_stats: float32 [n][4] or None."""
    import torch
    n, h, w, c = images.shape
    ip = dr._ptr(images, None, torch.uint8, "images")
    op = dr._ptr(out, (n, h, w, c), torch.float32, "out")
    sp = dr._ptr(img_stats, (n, 4), torch.float32, "img_stats") if img_stats is not None else None
    return dr._check(_lib().dr_image_augment(C.byref(params), C.c_uint64(seed), C.c_uint64(batch_index), image_offset,
                                             ip, n, h, w, c, op, sp, _stream(stream)))


def dr_total_kernel_launches() -> int:
    return _lib().dr_total_kernel_launches()


def scene_fields(rec):
    """[n][64] float32 numpy view of dr_scene_draw records -> dict of named fields."""
    import numpy as np
    r = np.asarray(rec, dtype=np.float32)
    return {
        "cam_pos": r[:, 0:9].reshape(-1, 3, 3), "cam_quat": r[:, 9:21].reshape(-1, 3, 4), "cam_fov": r[:, 21:24],
        "robot_rgb": r[:, 24:27], "robot_metallic": r[:, 27], "robot_gloss": r[:, 28], "obj_hsv": r[:, 29:32],
        "obj_metallic": r[:, 32], "obj_gloss": r[:, 33], "n_lights": r[:, 34].view(np.uint32),
        "light_dir": r[:, 35:53].reshape(-1, 6, 3), "light_intensity": r[:, 53:59], "total_intensity": r[:, 59],
    }


def dr_pose_aug_params_default() -> DrPoseAugParams:
    p = DrPoseAugParams()
    dr._check(_lib().dr_pose_aug_params_default(C.byref(p)))
    return p


def pose_params_from_preset(preset: dict) -> DrPoseAugParams:
    p = dr_pose_aug_params_default()
    for k in ("p_keep", "p_rot90", "pos_std", "rot_std"):
        if k in preset:
            setattr(p, k, preset[k])
    return p


def dr_pose_augment(params: DrPoseAugParams, seed: int, batch_index: int, pose_in, pose_out, branch_out=None,
                    sample_offset: int = 0, stream=None):
    """pose_in / pose_out: CUDA float32 [n][7]; branch_out: CUDA uint8 [n] or None."""
    import torch
    n = pose_in.shape[0]
    ip = dr._ptr(pose_in, (n, 7), torch.float32, "pose_in")
    op = dr._ptr(pose_out, (n, 7), torch.float32, "pose_out")
    bp = dr._ptr(branch_out, (n,), torch.uint8, "branch_out") if branch_out is not None else None
    return dr._check(_lib().dr_pose_augment(C.byref(params), C.c_uint64(seed), C.c_uint64(batch_index), sample_offset,
                                            ip, n, op, bp, _stream(stream)))
