/*
 * dr_vision.h -- C-ABI of libdr.so's vision randomizations: the
 * appearance draws of Table vision-randomization and the post-render image
 * augmentation of PAPER.md:127-129, batched on an NVIDIA B200 (sm_100a).
 *
 * These calls are context-free (no dr_init needed): each takes its seed, batch index and CUDA
 * stream explicitly and enqueues one kernel.  Draws use Philox4x32-10 keyed by the seed with
 * counter (global sample / image id, batch index, channel, block) -- channels 0x201-0x202 for
 * images, 0x301-0x303 for scene draws -- so results depend only on
 * (seed, batch index, global id), never on how a batch is split across calls or GPUs.
 *
 * Pointers are DEVICE pointers owned by the caller (PyTorch) and must stay alive until the
 * enqueued work completes in stream order.  Errors: DR_EINVAL (dr_last_error() names the field),
 * DR_EUNSUPPORTED (image larger than the cluster-resident limit), DR_ECUDA (launch error).
 * Readings of what the paper leaves open are DESIGN.md V1-V6.
 */
#ifndef DR_VISION_H
#define DR_VISION_H

#include <stddef.h>
#include <stdint.h>

#include "dr.h"

#ifdef __cplusplus
extern "C" {
#endif

#define DR_VIS_N_CAMERAS  3  /* "number of cameras 3" */
#define DR_VIS_MAX_LIGHTS 6  /* "number of lights 4-6" */
/* Largest image dr_image_augment keeps on chip: 8 CTAs of one cluster x 200 KB of shared memory. */
#define DR_VIS_MAX_IMAGE_BYTES (8 * 200 * 1024)

typedef struct {
    uint32_t abi_version, struct_size;   /* DR_ABI_VERSION, sizeof(dr_vision_params) */
    /* Table vision-randomization; lengths in metres, angles in radians */
    double cam_pos_range;                /* 1.5e-3: per-axis offset U[-r, r]               [V1] */
    double cam_rot_max;                  /* 3 deg: angle U[0, max] about a uniform axis     [V2] */
    double cam_fov_range;                /* 1 deg: offset U[-r, r] */
    double robot_metallic_lo, robot_metallic_hi;   /* 0.05, 0.25 */
    double robot_gloss_lo, robot_gloss_hi;         /* 0, 1 */
    double obj_hue_cal, obj_sat_cal, obj_val_cal;  /* calibrated HSV in [0, 1]  */
    double obj_hue_range, obj_sat_range, obj_val_range;  /* 0.01, 0.15, 0.15: additive [V3] */
    double obj_metallic_lo, obj_metallic_hi;       /* 0.05, 0.15 */
    double obj_gloss_lo, obj_gloss_hi;             /* 0.05, 0.15 */
    int32_t lights_min, lights_max;                /* 4, 6 (0 <= min <= max <= 6)          [V4] */
    double light_rel_lo, light_rel_hi;             /* 1, 5 */
    double light_total_lo, light_total_hi;         /* 0, 15                                [V5] */
    /* post-render augmentation (Table rows "image contrast adjustment",
     * "additive per-pixel Gaussian noise") [V6] */
    double contrast_lo, contrast_hi;     /* 0.5, 1.5: factor per image */
    double noise_std_lo, noise_std_hi;   /* 0.1, 0.1: noise std per image, normalized units */
    double std_floor;                    /* 1e-8: normalisation divides by max(std, floor) */
} dr_vision_params;

/* One sample's appearance draws, 64 words (256 bytes). */
typedef struct {
    float cam_pos[DR_VIS_N_CAMERAS][3];   /* position offsets, m */
    float cam_quat[DR_VIS_N_CAMERAS][4];  /* rotation offsets (w, x, y, z) */
    float cam_fov[DR_VIS_N_CAMERAS];      /* field-of-view offsets, rad */
    float robot_rgb[3];
    float robot_metallic, robot_gloss;
    float obj_hsv[3];                     /* hue wrapped to [0, 1), saturation / value clamped to [0, 1] */
    float obj_metallic, obj_gloss;
    uint32_t n_lights;
    float light_dir[DR_VIS_MAX_LIGHTS][3];  /* unit directions on the upper half-sphere (z > 0); 0 past n_lights */
    float light_intensity[DR_VIS_MAX_LIGHTS];  /* sum = total_intensity; 0 past n_lights */
    float total_intensity;
    float _pad[4];
} dr_scene_draw;

/* The paper's values (Table vision-randomization) and the DESIGN.md calibrated-HSV workload choice. */
int dr_vision_params_default(dr_vision_params* p);

/* Appearance draws for samples [sample_offset, sample_offset + n_samples) of batch batch_index:
 * out_dev[n_samples] (device, 16-byte aligned).  One thread per sample, fp64 arithmetic rounded
 * to fp32 on output.  Asynchronous on `stream` (cudaStream_t, NULL = legacy default). */
int dr_scene_draw_batch(const dr_vision_params* p, uint64_t seed, uint64_t batch_index, int64_t sample_offset,
                        int64_t n_samples, dr_scene_draw* out_dev, void* stream);

/* Post-render augmentation of n_images u8 images, row-major
 * [n_images][height][width][channels], image i having global id image_offset + i:
 *   out = f * (x - mean) / max(std, floor) + s * z,   f ~ U[contrast], s ~ U[noise], z ~ N(0, 1)
 * per element, mean / population std over the whole image.  out: device fp32, same shape.
 * img_stats: device fp32 [n_images][4] = (mean, std, f, s), or NULL.
 * One thread-block cluster per image: the image is read from HBM once (TMA bulk copies into the
 * cluster's shared memory), reduced through distributed shared memory, and written once.
 * DR_EUNSUPPORTED if height * width * channels > DR_VIS_MAX_IMAGE_BYTES.  Asynchronous.
 * Launched with programmatic dependent launch: a call directly behind another dr_image_augment
 * on the same stream reads its images while that call is still writing (and writes early too
 * when neither call's buffers overlap the other's); the results are those of stream order. */
int dr_image_augment(const dr_vision_params* p, uint64_t seed, uint64_t batch_index, int64_t image_offset,
                     const uint8_t* images, int64_t n_images, int32_t height, int32_t width, int32_t channels,
                     float* out, float* img_stats, void* stream);

/* Vision-model training pose augmentation. */
typedef struct {
    uint32_t abi_version, struct_size;   /* DR_ABI_VERSION, sizeof(dr_pose_aug_params) */
    double p_keep;     /* 0.2: "leave the object pose as is with 20% probability" */
    double p_rot90;    /* 0.4: "rotate the object by 90 deg around its main axes with 40% probability" */
    double pos_std;    /* 5e-3 m: position jitter per axis (not given in the paper)  [Q28] */
    double rot_std;    /* 0.05 rad: rotation jitter angle about a uniform axis (not given) */
} dr_pose_aug_params;

int dr_pose_aug_params_default(dr_pose_aug_params* p);

/* Per sample i (global id sample_offset + i) of batch batch_index, pose_in [n][7] = (position xyz,
 * unit quaternion wxyz), device fp32:
 *   branch 0 (p_keep):  pose unchanged;
 *   branch 1 (p_rot90): q <- q (x) r, r = exactly 90 deg about one of the object's own axes (uniform
 *                       axis and sign); position unchanged;
 *   branch 2 (rest):    position + N(0, pos_std^2) per axis and q <- q_j (x) q with q_j an angle
 *                       N(0, rot_std^2) about a uniform axis ("jitter ... both the position and
 *                       rotation independently").
 * The branch is an exact integer decision on one Philox word (channel 0x401).  pose_out [n][7]
 * device fp32 (may alias pose_in); branch_out [n] device u8 or NULL.  Asynchronous on `stream`. */
int dr_pose_augment(const dr_pose_aug_params* p, uint64_t seed, uint64_t batch_index, int64_t sample_offset,
                    const float* pose_in, int64_t n, float* pose_out, uint8_t* branch_out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* DR_VISION_H */
