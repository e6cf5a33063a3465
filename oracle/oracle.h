/*
 * oracle.h -- plain, slow, fp64 CPU oracle of the per-env-step domain-randomization
 * pipeline ("Randomizations" appendix).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load liboracle.so.  The product path
 * (include/dr.h + paper_1906_11633_b200/) never includes, links or calls anything here,
 * and this file includes nothing from the product path: the oracle re-declares its
 * own parameter struct, implements its own Philox4x32-10 from the Salmon et al.
 * (SC'11) specification, its own draw transforms, and its own host-side threshold
 * tables.  Every function cites the passage it follows.
 *
 * Arithmetic: fp64 throughout, scalar, one env at a time, compiled with
 * -O2 -ffp-contract=off (no FMA contraction), so the occlusion distance test is the
 * exactly-rounded ((dx*dx + dy*dy) + dz*dz) the readings in DESIGN.md fix.
 *
 * Parity pins: see tests/test_oracle_*.py.  Unpinned by the paper (workload choices,
 * DESIGN.md "parity unpinned"): the physical-parameter table (table
 * missing) and the calibrated backlash widths (values not given).
 */
#ifndef DR_ORACLE_H
#define DR_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_N_ACT      20   /* Shadow hand actuators */
#define ORC_N_TIPS     5    /* fingertips */
#define ORC_N_SUB      10   /* MuJoCo substeps per env step */
#define ORC_MAX_PHYS   256
#define ORC_OBS_IN     26   /* raw_obs row: tips 15, obj pos 3, obj quat 4 (w,x,y,z), goal quat 4 */
#define ORC_OBS_OUT    22   /* policy obs row: rel goal 4, tips 15, obj pos 3 */
#define ORC_N_STATS    32

/* layer bits (same meaning as DESIGN.md's table; declared independently here) */
#define ORC_TIMING     (1u << 0)
#define ORC_ACT_NOISE  (1u << 1)
#define ORC_DELAY      (1u << 2)
#define ORC_BACKLASH   (1u << 3)
#define ORC_OBS_NOISE  (1u << 4)
#define ORC_DROPOUT    (1u << 5)
#define ORC_OCCLUSION  (1u << 6)
#define ORC_FORCE      (1u << 7)
#define ORC_PHYS       (1u << 8)
/* SURVEY.md §8(f) rank 2 variants (off in the paper's FULL set) */
#define ORC_SMOOTH     (1u << 9)   /* EMA action smoothing, 0.3 per 80 ms */
#define ORC_SUBSTEP_BL (1u << 10)  /* backlash updated once per substep with dt_k */

/* physical-parameter descriptor kinds (SPEC.md:126 schema; table itself missing) */
#define ORC_PHYS_FIXED            0
#define ORC_PHYS_UNIFORM_SCALE    1
#define ORC_PHYS_LOGUNIFORM_SCALE 2
#define ORC_PHYS_ADD_GAUSS        3
#define ORC_PHYS_MUL_LOGNORMAL    4

typedef struct {
    int32_t kind;
    double a, b, base;
} orc_phys_desc;

typedef struct {
    uint32_t layer_mask;
    /* action noise + delay, Table action-noise */
    double act_sigma_uadd, act_sigma_cadd, act_sigma_mult, delay_prob;
    /* timing */
    double dt_base, lambda_lo, lambda_hi, step_nominal;
    /* backlash */
    double delta_cal_neg[ORC_N_ACT], delta_cal_pos[ORC_N_ACT];
    double delta_jitter_std, backlash_eps;
    /* observation noise, Table obs-noise PAPER.md:29-45 (metres / radians) */
    double tip_corr, tip_uncorr, obj_corr, obj_uncorr, rot_corr, rot_uncorr;
    double tip_marker, base_marker;
    int32_t base_marker_to_tips;
    /* PhaseSpace errors */
    double dropout_rate_hz;
    int32_t dropout_hold_steps;
    double occl_dist;
    /* random forces */
    double force_p_lo, force_p_hi, force_accel_std, force_decay_per_step;
    /* physical parameters */
    int32_t n_phys, mass_index;
    orc_phys_desc phys[ORC_MAX_PHYS];
    /* action smoothing coefficient per 80 ms step (PAPER.md:743 footnote: 0.3) */
    double act_smooth_coef;
} orc_params;

/* One environment's episode record + mutable state, fp64. */
typedef struct {
    int64_t  gid;          /* global env id (Philox counter word 0) */
    uint32_t episode;      /* k_e */
    /* ---- episode record (reset draws) ---- */
    uint32_t delay_bits;   /* bit j = actuator j delayed */
    uint32_t p_index;      /* j_p = x >> 16 */
    uint32_t t_force;      /* floor(p_j * 2^32) (saturated to 2^32-1 only if p=1) */
    uint32_t _pad0;
    double   p_force;      /* p_j */
    double   lambda;
    double   mass;
    double   dneg[ORC_N_ACT], dpos[ORC_N_ACT];
    double   c_act[ORC_N_ACT];
    double   off_tip[ORC_N_TIPS * 3];
    double   c_obj[3];
    double   q_c[4];
    double   phys[ORC_MAX_PHYS];
    /* ---- mutable state ---- */
    double   prev[ORC_N_ACT];
    double   slack[ORC_N_ACT];
    double   last[ORC_N_TIPS * 3];
    int32_t  has_last;
    int32_t  timer[ORC_N_TIPS];
    double   f_trig[3];
    uint32_t k_f;
    uint32_t _pad1;
    double   ema[ORC_N_ACT];   /* smoothed action (ORC_SMOOTH) */
} orc_env;

typedef struct orc_ctx orc_ctx;

/* ---- context API (mirrors the shape of the product ABI; host memory only) ---- */
int  orc_init(const orc_params* p, int64_t n_env, const int64_t* gids, uint64_t seed, orc_ctx** out);
void orc_free(orc_ctx* c);
int  orc_update_params(orc_ctx* c, const orc_params* p); /* mid-run parameter swap */
int  orc_reset(orc_ctx* c, const uint8_t* mask);          /* NULL = all envs */
/* One env step for all envs of the context.  Outputs may be NULL.
 * bl_margin [n][20]: fp64 |(s + a_n*d*dt_env) - sgn(a_n)| (the backlash rail margin: where fp32 and
 * fp64 may clamp differently), or on a rail hit from s != sgn(a_n) the smaller |sgn(a_n) - s| (where
 * alpha = eps / (|sgn - s| + eps) is ill-conditioned in s); +inf when sgn(a_n) = 0 or BACKLASH off --
 * used by tests to classify knife-edge gate decisions (diagnostic only: no output depends on it). */
int  orc_step(orc_ctx* c, const float* actions, const float* raw_obs,
              double* out_actions, double* out_obs, double* out_dt, double* out_force,
              double* stats, double* bl_margin);
/* Same step with the per-substep actions [n][10][20] of ORC_SUBSTEP_BL (may be NULL). */
int  orc_step_sub(orc_ctx* c, const float* actions, const float* raw_obs,
                  double* out_actions, double* out_actions_sub, double* out_obs, double* out_dt,
                  double* out_force, double* stats, double* bl_margin);
/* Simulator-provided occlusion: bit i of mask[e] = fingertip marker i of
 * env e occluded this step (the simulator's collision-site rule) replaces the distance
 * rule; NULL restores it.  The array (n bytes) is read at every later orc_step. */
void     orc_set_occlusion_mask(orc_ctx* c, const uint8_t* mask);
uint64_t orc_step_index(const orc_ctx* c);
void     orc_set_step_index(orc_ctx* c, uint64_t t);
int      orc_get_env(const orc_ctx* c, int64_t i, orc_env* dst);
int      orc_set_env(orc_ctx* c, int64_t i, const orc_env* src);   /* state import (gid kept) */
int64_t  orc_n_env(const orc_ctx* c);
uint64_t orc_force_threshold(const orc_ctx* c, uint32_t j); /* T_j of the 65,536-entry table */
double   orc_force_p(const orc_ctx* c, uint32_t j);

/* ---- scalar hooks (pinned individually by tests) ---- */
void   orc_philox(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
double orc_uniform(uint32_t x);
void   orc_normal_pair(uint32_t x, uint32_t y, double* z0, double* z1);
double orc_exponential(uint32_t x, double lambda);
void   orc_rotation(double sigma, const uint32_t w[4], double q[4]);
void   orc_quat_mul(const double a[4], const double b[4], double out[4]);
void   orc_backlash(double s, double a, double dneg, double dpos, double dt, double eps,
                    double* s_new, double* alpha, double* out);
int    orc_occluded(const float* tips15, const float* obj3, double r, int tip);
uint64_t orc_bernoulli_threshold(double p);

/* ---- vision randomization (Table vision-randomization) ----
 * Appearance draws per sample and the post-render image augmentation per camera image;
 * readings V1-V6 in DESIGN.md.  Draws: Philox keyed by the seed, counter = (global sample or
 * image id, batch index, channel, block), channels below. */
#define ORC_VIS_N_CAMERAS  3
#define ORC_VIS_MAX_LIGHTS 6
#define ORC_SCENE_WORDS    64   /* scene record: see orc_scene_draw */
typedef struct {
    double cam_pos_range, cam_rot_max, cam_fov_range;            /* 1.5 mm, 3 deg, 1 deg */
    double robot_metallic_lo, robot_metallic_hi, robot_gloss_lo, robot_gloss_hi;
    double obj_hue_cal, obj_sat_cal, obj_val_cal;                 /* calibrated HSV in [0, 1] */
    double obj_hue_range, obj_sat_range, obj_val_range;           /* 0.01, 0.15, 0.15 */
    double obj_metallic_lo, obj_metallic_hi, obj_gloss_lo, obj_gloss_hi;
    int32_t lights_min, lights_max;                               /* 4, 6 */
    double light_rel_lo, light_rel_hi, light_total_lo, light_total_hi;   /* 1..5, 0..15 */
    double contrast_lo, contrast_hi;                              /* 0.5, 1.5 */
    double noise_std_lo, noise_std_hi;                            /* 0.1, 0.1 (normalized units) */
    double std_floor;                                             /* 1e-8 */
} orc_vision_params;

/* Appearance draws of samples [sample_offset, sample_offset + n): out [n][64] fp64, fields in
 * the order cam_pos[3][3], cam_quat[3][4], cam_fov[3], robot_rgb[3], robot_metallic,
 * robot_gloss, obj_hsv[3], obj_metallic, obj_gloss, n_lights, light_dir[6][3],
 * light_intensity[6], total_intensity, 4 zero pad words. */
int orc_scene_draw(const orc_vision_params* p, uint64_t seed, uint64_t batch, int64_t sample_offset, int64_t n,
                   double* out);
/* Post-render augmentation of n u8 images [n][H][W][C]: normalise each image
 * to zero mean / unit variance, scale by a contrast factor, add per-pixel Gaussian noise.
 * out [n][H][W][C] fp64; img_stats [n][4] = (mean, std, contrast, noise std), may be NULL. */
int orc_image_augment(const orc_vision_params* p, uint64_t seed, uint64_t batch, int64_t image_offset,
                      const uint8_t* images, int64_t n, int32_t h, int32_t w, int32_t c, double* out,
                      double* img_stats);

/* Vision-model training pose augmentation: per sample,
 * keep the pose (p_keep = 20 %), rotate the object 90 deg about one of its body axes (p_rot90 =
 * 40 %), or jitter position and rotation independently with Gaussian noise (the remaining 40 %).
 * pose_in [n][7] = position xyz, unit quaternion wxyz; pose_out [n][7] fp64; branch [n] = 0/1/2. */
typedef struct {
    double p_keep, p_rot90;      /* 0.2, 0.4 */
    double pos_std, rot_std;     /* jitter: 5 mm per axis, 0.05 rad about a uniform axis (values not in the paper) */
} orc_pose_aug_params;
int orc_pose_augment(const orc_pose_aug_params* p, uint64_t seed, uint64_t batch, int64_t offset,
                     const float* pose_in, int64_t n, double* pose_out, uint8_t* branch);

/* stats slot indices */
enum {
    ORC_S_ENVS = 0, ORC_S_DELAYED = 1, ORC_S_DROP_INIT = 2, ORC_S_MASKED = 3, ORC_S_OCCLUDED = 4,
    ORC_S_HELD = 5, ORC_S_FORCE_TRIG = 6, ORC_S_RAIL_HITS = 7, ORC_S_ALPHA_ONE = 8,
    ORC_S_ALPHA_LT1 = 9, ORC_S_RESETS = 10, ORC_S_ACT_CLAMPS = 11,
    ORC_S_SUM_DT = 16, ORC_S_SUM_DT2 = 17, ORC_S_SUM_DA = 18, ORC_S_SUM_DA2 = 19,
    ORC_S_SUM_ABS_BL = 20, ORC_S_SUM_ZU2 = 21, ORC_S_SUM_ZTIP2 = 22, ORC_S_SUM_F2 = 23
};

#ifdef __cplusplus
}
#endif
#endif
