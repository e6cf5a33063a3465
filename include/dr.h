/*
 * dr.h -- C-ABI of libdr.so: the batched per-environment-step domain-randomization pipeline of
 * the "Randomizations" appendix on an NVIDIA B200 (sm_100a).
 *
 * One context per process, bound to the CUDA device current at dr_init (one process per GPU,
 * the torchrun model).  All calls are ASYNCHRONOUS on the library stream (dr_set_stream /
 * dr_params.stream) unless stated: they validate, enqueue and return.  Not thread-safe.
 *
 * Per-env arrays passed to dr_step / dr_reset are DEVICE pointers, row-major [n_env][C],
 * fp32 unless noted, 16-byte aligned, owned by the caller (PyTorch), and must stay alive until
 * the enqueued work completes in stream order.  Inputs are never written (the
 * noise reaches the policy inputs only; the caller's clean copy is the value-function view).
 *
 * Error behaviour: every entry point returns a dr_status (or a sentinel for pointer/size
 * getters); dr_last_error() names the offending field or CUDA error.  DR_ECUDA is sticky.
 * No per-element checks run on the hot path: NaN/out-of-range inputs propagate (actions are
 * clamped to [-1, 1] after action noise).  Quaternion inputs are assumed unit.
 *
 * The RNG conventions (Philox4x32-10 keyed by the seed, counter = (global env id, step t or
 * episode k_e, channel, block)) and every reading of the paper used here are written down in
 * DESIGN.md; results depend only on (seed, global env id, t, k_e), never on the GPU count.
 */
#ifndef DR_H
#define DR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DR_ABI_VERSION 2u

#define DR_N_ACT       20  /* actuators of the Shadow hand */
#define DR_N_TIPS      5   /* fingertip markers */
#define DR_N_SUBSTEPS  10  /* MuJoCo substeps per env step */
#define DR_MAX_PHYS    256 /* physical-parameter slots (~264 calibrated values) */
#define DR_OBS_IN      26  /* raw_obs row: tips[5][3], obj_pos[3], obj_quat[4] (w,x,y,z), goal_quat[4] */
#define DR_OBS_OUT     22  /* out_obs row (policy view, Table policy-inputs):
                              noisy relative goal[4] (w,x,y,z; w >= 0), noisy tips[5][3], noisy obj_pos[3] */
#define DR_N_STATS     32  /* per-step statistics vector, fp64 */

typedef enum {
    DR_OK = 0,
    DR_EINVAL = -1,        /* invalid argument / parameter (dr_last_error names it) */
    DR_ENOTINIT = -2,      /* no context: call dr_init first */
    DR_EALREADY = -3,      /* dr_init on an initialised context */
    DR_ENOMEM = -4,        /* device or host allocation failed, or workspace too small */
    DR_ECUDA = -5,         /* CUDA launch/API error (sticky until dr_finalize) */
    DR_EUNSUPPORTED = -6   /* shape the v1 kernels do not specialise (n_act != 20, ...) */
} dr_status;

/* layer_mask bits: each randomization of PAPER.md:1-115 can be disabled (identity branch,
 * no draws consumed, no bytes moved for its state). */
enum {
    DR_TIMING    = 1u << 0, /* dt = 8 ms + Exp(lambda) per substep, lambda ~ U[1250,10000] per episode */
    DR_ACT_NOISE = 1u << 1, /* additive/multiplicative action noise (Table action-noise) */
    DR_DELAY     = 1u << 2, /* per-actuator one-step action delay, p = 0.5 per episode */
    DR_BACKLASH  = 1u << 3, /* backlash slack model */
    DR_OBS_NOISE = 1u << 4, /* correlated + uncorrelated obs noise, marker misplacement */
    DR_DROPOUT   = 1u << 5, /* fingertip marker dropout 0.2/s for 1 s */
    DR_OCCLUSION = 1u << 6, /* marker occlusion -> hold last reading */
    DR_FORCE     = 1u << 7, /* random forces on the object */
    DR_PHYS      = 1u << 8, /* per-episode physical parameters */
    DR_ALL       = 0x1FFu,  /* the paper's randomization set */
    /* variants, off unless requested: */
    DR_SMOOTH    = 1u << 9, /* EMA smoothing of the policy action, 0.3 per 80 ms, before delay/noise */
    DR_SUBSTEP_BACKLASH = 1u << 10, /* backlash slack updated once per substep with dt_k;
                                       requires dr_step_substeps */
    DR_ALL_EXT   = 0x7FFu
};

/* physical-parameter descriptor (SPEC.md:126 schema; the paper's table is missing) */
enum {
    DR_PHYS_FIXED = 0,            /* v = base */
    DR_PHYS_UNIFORM_SCALE = 1,    /* v = base * U[a, b] */
    DR_PHYS_LOGUNIFORM_SCALE = 2, /* v = base * exp(U[ln a, ln b]) */
    DR_PHYS_ADD_GAUSS = 3,        /* v = base + a * N(0,1) */
    DR_PHYS_MUL_LOGNORMAL = 4     /* v = base * exp(a * N(0,1)) */
};
typedef struct {
    uint32_t kind;
    uint32_t _pad;
    double a, b, base;
} dr_phys_desc;

/* Parameters.  Host struct, copied at dr_init.  Fill with dr_params_default() (the paper's
 * values) and override.  abi_version = DR_ABI_VERSION, struct_size = sizeof(dr_params). */
typedef struct dr_params {
    uint32_t abi_version, struct_size, layer_mask, _pad0;
    int32_t  n_act, n_tips, n_substeps, _pad1;       /* must be 20, 5, 10 (else DR_EUNSUPPORTED) */
    int64_t  env_offset;                             /* global id of local env 0 (multi-GPU shard) */
    int64_t  n_env_global;                           /* total envs over all ranks (0 = n_env) */
    /* action noise + delay: Table action-noise, range 2 */
    double act_sigma_uadd;       /* 0.10  (5 % of range) */
    double act_sigma_cadd;       /* 0.03  (1.5 % of range), per episode */
    double act_sigma_mult;       /* 0.015 (unitless) */
    double delay_prob;           /* 0.5 */
    /* timing */
    double dt_base;              /* 0.008 s */
    double lambda_lo, lambda_hi; /* 1250, 10000 (1/s, rate) */
    double step_nominal;         /* 0.08 s: the dropout rate's time base */
    /* backlash */
    double delta_cal_neg[DR_N_ACT], delta_cal_pos[DR_N_ACT]; /* calibrated widths (>= 0) */
    double delta_jitter_std;     /* 0.1 */
    double backlash_eps;         /* 1e-12; must be in [0, 1e-8] (DR_EINVAL otherwise) */
    /* observation noise std, metres / radians (Table obs-noise) */
    double tip_corr, tip_uncorr, obj_corr, obj_uncorr, rot_corr, rot_uncorr, tip_marker, base_marker;
    int32_t base_marker_to_tips; /* 1: hand-base marker error shifts all tips (Q14) */
    int32_t dropout_hold_steps;  /* 13 = ceil(1 s / 80 ms), <= 15 */
    /* PhaseSpace errors */
    double dropout_rate_hz;      /* 0.2 */
    double occl_dist;            /* 0.015 m (>= 0; 0 disables) */
    /* random forces */
    double force_p_lo, force_p_hi;  /* 0.001, 0.1 (loguniform), 0 < lo <= hi <= 1 */
    double force_accel_std;         /* 1.0 m/s^2 (times the object mass) */
    double force_decay_per_step;    /* 0.99 per 80 ms step, in (0, 1] */
    /* action smoothing (DR_SMOOTH) */
    double act_smooth_coef;         /* 0.3: a_s <- (1 - c) a_s + c a per step, in [0, 1] */
    /* physical parameters */
    int32_t n_phys, mass_index;     /* 1 <= n_phys <= 256; phys[mass_index] is the object mass */
    dr_phys_desc phys[DR_MAX_PHYS];
    /* memory / stream (PyTorch-owned) */
    void*  workspace;               /* NULL: the library cudaMallocs its state */
    size_t workspace_bytes;         /* >= dr_workspace_bytes(params, n_env) when workspace != NULL */
    void*  stream;                  /* cudaStream_t; NULL = legacy default stream */
} dr_params;

/* Exported per-env state (dr_state_export / dr_state_import), 672 bytes. */
typedef struct {
    uint32_t episode;        /* k_e: number of resets since dr_init */
    uint32_t delay_bits;     /* bit j: actuator j delayed this episode */
    uint32_t p_index;        /* j_p: index of the episode's force probability in the 65,536 table */
    uint32_t t_force;        /* force trigger threshold floor(p * 2^32) */
    uint32_t flags;          /* bits 4i..4i+3: dropout timer of tip i; bit 20: has_last */
    uint32_t k_f;            /* steps since the last force trigger (saturates at 65535) */
    float lambda, mass;
    float dneg[DR_N_ACT], dpos[DR_N_ACT], c_act[DR_N_ACT];
    float off_tip[DR_N_TIPS * 3], c_obj[3], q_c[4];
    float prev[DR_N_ACT], slack[DR_N_ACT], last[DR_N_TIPS * 3], f_trig[3];
    float ema[DR_N_ACT];     /* smoothed action (DR_SMOOTH) */
} dr_env_state;

/* Stats slot indices (dr_stats).  Integer counts are exact (held in fp64 < 2^53). */
enum {
    DR_S_ENVS = 0, DR_S_DELAYED = 1, DR_S_DROP_INIT = 2, DR_S_MASKED = 3, DR_S_OCCLUDED = 4,
    DR_S_HELD = 5, DR_S_FORCE_TRIG = 6, DR_S_RAIL_HITS = 7, DR_S_ALPHA_ONE = 8, DR_S_ALPHA_LT1 = 9,
    DR_S_RESETS = 10, DR_S_ACT_CLAMPS = 11,
    DR_S_SUM_DT = 16, DR_S_SUM_DT2 = 17, DR_S_SUM_DA = 18, DR_S_SUM_DA2 = 19, DR_S_SUM_ABS_BL = 20,
    DR_S_SUM_ZU2 = 21, DR_S_SUM_ZTIP2 = 22, DR_S_SUM_F2 = 23
};

/* Fill *p with the paper's values (tables cited above), layer_mask = DR_ALL, the DESIGN.md
 * synthetic physics table and calibrated widths.  Returns DR_OK. */
int dr_params_default(dr_params* p);

/* Create the context: validate (DR_EINVAL naming the field: any std < 0, lo > hi, probabilities
 * outside [0,1], decay outside (0,1], occl_dist < 0, calibrated delta < 0, dt_base <= 0, base
 * mass <= 0, n_env < 1 or > 2^31, env_offset + n_env > n_env_global), allocate or adopt the
 * workspace, upload constants, then enqueue episode 0 sampling for every env. */
int dr_init(const dr_params* params, int64_t n_env, uint64_t seed);

/* On-the-fly parameter update ("change randomization parameters during training", ORRB's
 * adaptive randomization).  Validates *params like dr_init (same DR_EINVAL
 * messages); layer_mask, n_phys, env_offset and n_env_global must equal the context's
 * (DR_EINVAL otherwise); workspace and stream fields are ignored.  The new constants and
 * tables are uploaded in stream order on the library stream, so every dr_step / dr_reset
 * enqueued after this call sees them and every one enqueued before does not:
 *   - per-step draws (action-noise stds, substep base dt, dropout rate and hold, occlusion
 *     radius, uncorrelated obs noise, force accel std and decay) change from the next dr_step;
 *   - per-episode draws (calibrated backlash widths and jitter, lambda range, force p range,
 *     correlated noise, delay probability, physics descriptors) change at each env's next
 *     reset: the current episode records are not resampled.
 * Not graph-capturable (host tables are staged synchronously).  Asynchronous otherwise. */
int dr_update_params(const dr_params* params);

/* Episode reset: for every env with
 * env_mask[e] != 0 (device u8 [n_env]; NULL = all), k_e += 1, then resample its episode record
 * and physical parameters and zero its state.  Asynchronous. */
int dr_reset(const uint8_t* env_mask);

/* One environment step for all n_env envs, one fused kernel:
 *   actions     [n][20] in   policy actions in [-1, 1]
 *   raw_obs     [n][26] in   true fingertip/object state (see DR_OBS_IN)
 *   out_actions [n][20] out  delayed, noised, clamped, backlash-gated actions for the simulator
 *   out_obs     [n][22] out  policy observation (see DR_OBS_OUT)
 *   out_dt      [n][10] out  substep durations, s
 *   out_force   [n][3]  out  force on the object, N
 * The global step counter t advances by one in stream order (device-resident, so a CUDA graph
 * of dr_step calls advances it on every replay).  Jobs of up to 16,384 envs (n_env_global) run a
 * latency-mode kernel (8 warps split a 32-env group's transform), larger jobs the throughput
 * kernel (one thread per env, persistent tiles); the environment variable DR_STEP_MODE =
 * throughput | latency, read at dr_init, forces either.  Both give the same results within the
 * parity contract, and every shard of a job runs the same one.  The step (and reset) kernels are
 * launched with programmatic dependent launch: they wait for the previous kernel in the stream
 * before touching memory, so ordering is unchanged (DR_PDL=0 at dr_init: plain launches).
 * Asynchronous. */
int dr_step(const float* actions, const float* raw_obs, float* out_actions, float* out_obs,
            float* out_dt, float* out_force);

/* dr_step for contexts with DR_SUBSTEP_BACKLASH (DR_EINVAL otherwise; dr_step returns DR_EINVAL
 * for such contexts): the backlash slack model runs once per MuJoCo substep k with that
 * substep's dt_k ("each of the substeps", 104 "dt"), the noised action held over
 * the step, so the simulator receives one gated action per substep:
 *   out_actions_sub [n][10][20] out  alpha_k * a_n for substep k
 *   out_actions     [n][20]     out  the last substep's action (= out_actions_sub[:, 9])
 * Other arguments as dr_step.  Asynchronous. */
int dr_step_substeps(const float* actions, const float* raw_obs, float* out_actions, float* out_actions_sub,
                     float* out_obs, float* out_dt, float* out_force);

/* End-to-end variant on HOST buffers (same layouts): copies inputs host->device, runs dr_step,
 * copies outputs device->host through two library-owned device buffer sets.  Pipelined over
 * consecutive calls: the H2D of call t runs on a library copy stream, the step on the library
 * stream, the D2H on a second copy stream, ordered by events, so call t+1's upload overlaps call
 * t's download and compute.  Asynchronous if the host buffers are pinned (cudaHostAlloc / torch
 * pin_memory): the caller must not modify an input buffer or read an output buffer of a call
 * until dr_synchronize(), which waits for all three streams.  If raw_obs directly follows
 * actions in host memory (one [n][20 + 26] allocation), the upload is one copy; if out_obs,
 * out_dt and out_force directly follow out_actions (one [n][20 + 22 + 10 + 3] allocation, n even),
 * the download is one copy -- fewer per-copy latencies for small n.  DR_EINVAL for
 * DR_SUBSTEP_BACKLASH contexts. */
int dr_step_host(const float* actions, const float* raw_obs, float* out_actions, float* out_obs,
                 float* out_dt, float* out_force);

/* Destroy the context (frees library-owned memory; never the caller's workspace).  Blocking. */
int dr_finalize(void);

/* ---- auxiliaries ---- */
size_t   dr_workspace_bytes(const dr_params* params, int64_t n_env); /* 0 on invalid input */
int      dr_set_stream(void* cuda_stream);          /* later calls enqueue on this stream */
/* Simulator-provided occlusion: occl_mask_dev is a device u8 [n_env]
 * array whose bit i says fingertip marker i of env e is occluded this step (the simulator's
 * collision-site rule); with DR_OCCLUSION on it replaces the 15 mm distance rule
 * (Q13 / Q27).  Every later dr_step reads the array in stream order, so the caller
 * refreshes its contents before each step.  NULL restores the distance rule. */
int      dr_set_occlusion_input(const uint8_t* occl_mask_dev);
int      dr_synchronize(void);                      /* blocking: wait for the library stream */
const float*  dr_phys_params(void);   /* device [n_env][n_phys] fp32, row-major; valid in stream order */
int      dr_n_phys(void);
/* Per-step stats (see DR_S_*) of the step with index t land in slot t % DR_STAT_SLOTS (a ring of
 * 4): device [32] fp64, complete when step t's kernel is.  Step t's kernel also clears slot
 * (t + 1) % 4 for the next step, so a caller all-reducing slot t % 4 (NCCL, overlapped with later
 * steps) must have finished before step t + 3 is enqueued.  Counts are exact; the moment slots
 * are sums of per-CTA partials rounded to a power-of-two quantum chosen from n_env_global (so the
 * order-free fp64 atomic sum is exact and deterministic; ~1e-12 relative).  dr_set_stats_buffer
 * lets the caller own the [4][32] fp64 device buffer (e.g. a torch tensor it all-reduces with
 * NCCL); NULL restores the internal one. */
#define DR_STAT_SLOTS 4
const double* dr_stats(int slot);
int      dr_set_stats_buffer(double* dev_buf);
uint64_t dr_step_index(void);               /* host count of enqueued steps (== device t unless graph-replayed) */
/* Blocking: waits for the library stream and returns the device step counter t (the index of the
 * next step; CUDA-graph replays of dr_step advance it too), and resets the host count to it.  The
 * stats of the last completed step are then in slot (t - 1) % DR_STAT_SLOTS. */
uint64_t dr_step_index_sync(void);
int      dr_set_step_index(uint64_t t);     /* blocking; for resume (also clears the stats ring) */
size_t   dr_state_bytes(void);              /* sizeof(dr_env_state) * n_env */
/* Blocking copies of per-env state for envs [env_lo, env_hi) (local indices); lo = hi = 0
 * means all envs.  host_dst / host_src hold (hi - lo) dr_env_state records. */
int      dr_state_export(void* host_dst, int64_t env_lo, int64_t env_hi);
int      dr_state_import(const void* host_src, int64_t env_lo, int64_t env_hi);
/* Blocking copy of phys rows [env_lo, env_hi) (lo = hi = 0: all) into host_dst [(hi-lo)][n_phys] fp32. */
int      dr_phys_export(void* host_dst, int64_t env_lo, int64_t env_hi);
const char* dr_last_error(void);
/* Launches of library kernels enqueued since dr_init (host count; graph replays not counted). */
uint64_t dr_kernel_launches(void);
/* Every libdr kernel launch of the process (context calls and the context-free vision calls). */
uint64_t dr_total_kernel_launches(void);
/* Test hook: out_dev[e][0..3] = the device Philox4x32-10 block the kernels draw for counter
 * (global id of env e, domain, channel, block) under the context's seed.  out_dev: device
 * uint32 [n_env][4].  Asynchronous.  Lets tests check the RNG words bit-exactly. */
int      dr_debug_philox(uint32_t domain, uint32_t channel, uint32_t block, uint32_t* out_dev);
/* Test hook (no context needed): out_dev[i] = Philox4x32-10(counter ctr_dev[i][0..3], key
 * key_dev[i][0..1]) computed by the same device round function every kernel uses (Salmon et al.,
 * SC'11; the RNG of DESIGN.md "RNG conventions"), round keys built from the key in registers.
 * ctr_dev / out_dev: device uint32 [n][4], 16-byte aligned; key_dev: device uint32 [n][2], 8-byte
 * aligned; n <= 2^32.  Asynchronous on `stream` (cudaStream_t, NULL = legacy default stream).
 * Lets tests check the device RNG against cuRAND's curand_Philox4x32_10 on arbitrary pairs. */
int      dr_debug_philox_keyed(const uint32_t* ctr_dev, const uint32_t* key_dev, uint32_t* out_dev, uint64_t n,
                               void* stream);
uint32_t dr_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* DR_H */
