// dr_internal.h -- shared between the host library (dr_api.cu) and the kernels (dr_kernels.cu).
// Device data layout: tiled structure-of-arrays ("AoSoA").
//   rec  : episode record, [n_tiles][REC_PLANES][TILE] 4-byte words
//   st   : mutable per-env state, [n_tiles][ST_PLANES][TILE]
//   phys : [n_env][n_phys] fp32, row-major (the simulator reads rows)
// Within a tile, plane k of env e sits at k * TILE + (e % TILE): a warp's 32 consecutive envs
// read one 128-byte line per plane (coalesced), every plane offset from an env's base is a
// compile-time immediate (no per-access address arithmetic), and a tile's whole record /
// state is one contiguous block (one bulk copy / L2 prefetch).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace dr {

constexpr int N_ACT = 20, N_TIPS = 5, N_SUB = 10, MAX_PHYS = 256, OBS_IN = 26, OBS_OUT = 22;
constexpr int N_STATS = 32;
constexpr int N_STAT_SLOTS = 4;     // stats ring: step t accumulates into slot t % 4 (DESIGN.md §8 "Stats")
constexpr int TILE = 128;           // envs per CTA tile (one thread per env)
constexpr uint32_t RUNTIME_MASK = 0xFFFFFFFFu;

// ---- record planes (read by the step kernel: 86 of them) ----
enum : int {
    REC_DELAY = 0,   // u32 delay bits
    REC_INVLAM = 1,  // 1/lambda (the step only needs the reciprocal rate)
    REC_TFORCE = 2,  // u32 force threshold
    REC_MASS = 3,
    REC_DNEG = 4,    // 20
    REC_DPOS = 24,   // 20
    REC_CACT = 44,   // 20
    REC_OFFTIP = 64, // 15
    REC_COBJ = 79,   // 3
    REC_QC = 82,     // 4
    REC_STEP_PLANES = 86,
    // not read by the step kernel
    REC_LAMBDA = 86,
    REC_PINDEX = 87, // u32
    REC_EPISODE = 88,// u32
    REC_PLANES = 89
};
// ---- state planes (read + written by the step kernel) ----
enum : int {
    ST_PREV = 0,     // 20
    ST_SLACK = 20,   // 20
    ST_LAST = 40,    // 15
    ST_FLAGS = 55,   // u32: tip i timer in bits 4i..4i+3, has_last in bit 20
    ST_FTRIG = 56,   // 3
    ST_KF = 59,      // u32
    ST_EMA = 60,     // 20: smoothed action (DR_SMOOTH)
    ST_PLANES = 80
};
constexpr uint32_t HAS_LAST_BIT = 1u << 20;
// Set by the reset kernel instead of zeroing the 60 state planes ("slack s initialized
// to 0; force vector zeroed"): the step kernel reads a fresh env's state as all-zero and writes it
// back, so a reset costs one scattered state word instead of sixty.
constexpr uint32_t FRESH_BIT = 1u << 21;

// AoSoA addressing: word offset of env e's plane 0; plane k is at + k * TILE.
__host__ __device__ __forceinline__ size_t rec_index(uint32_t e) {
    return (size_t)(e / TILE) * (REC_PLANES * TILE) + (e % TILE);
}
__host__ __device__ __forceinline__ size_t st_index(uint32_t e) {
    return (size_t)(e / TILE) * (ST_PLANES * TILE) + (e % TILE);
}
constexpr size_t PLANE = TILE;   // plane stride in words

// Philox channels
enum : uint32_t {
    CH_STEP = 0x01,   // 16 step words: substeps 0-9, dropout tips 10-14, force trigger 15
    CH_ACT_UADD = 0x02, CH_ACT_MULT = 0x03,   // 0x04 retired (dropout words live in CH_STEP)
    CH_TIP_NOISE = 0x05, CH_OBJ_NOISE = 0x06, CH_ROT_NOISE = 0x07, CH_FORCE = 0x08,
    CH_PHYS_U = 0x101, CH_DELAY = 0x102, CH_BACKLASH = 0x103, CH_LAMBDA = 0x104,
    CH_FORCE_P = 0x105, CH_CORR_ACT = 0x106, CH_CORR_TIP = 0x107, CH_MARKER_TIP = 0x108,
    CH_MARKER_BASE = 0x109, CH_CORR_OBJ = 0x10A, CH_CORR_ROT = 0x10B, CH_PHYS_N = 0x10C
};

// Constants uploaded once at dr_init (warp-uniform accesses only -> __constant__).
struct DevConst {
    uint32_t layer_mask;
    uint32_t n_env;
    uint64_t pitch;
    uint32_t env_offset;
    uint32_t hold_steps;
    uint32_t rk0[10], rk1[10];        // Philox round keys (key schedule precomputed on host)
    unsigned long long t_delay, t_drop;
    float su, sc, sm;                 // action noise stds
    float dt_base, lam_lo, lam_range;
    float dcal_neg[N_ACT], dcal_pos[N_ACT], jitter;
    float eps;
    float tip_corr, tip_uncorr, obj_corr, obj_uncorr, rot_corr, rot_uncorr, tip_marker, base_marker;
    int32_t base_to_tips;
    int32_t occl_on;
    double occl_r2;
    float occl_r2_lo, occl_r2_hi;      // r^2 (1 -+ 1e-5): fp32 fast-path decision band
    uint32_t occl_exact_only;          // r^2 outside the fp32 normal range: always exact fp64
    float accel_std;
    float smooth_c, smooth_keep;       // EMA: a_s <- smooth_keep * a_s + smooth_c * a
    double mq_scale[8], mq_inv[8];     // moment slots 16..23: CTA sums are rounded to multiples of
                                       // mq_inv (a power of 2) so the fp64 atomic totals are exact
    int32_t n_phys, mass_index;
    int32_t n_phys_u, n_phys_n;       // counts of uniform-kind / normal-kind params
    int32_t n_rs_philox, n_rs_pairs;  // reset task-table lengths (host-built, layer-dependent)
};

// Reset task tables (built on the host at dr_init, staged in shared memory by the reset kernel):
//   philox task : slot | blk << 8 | channel << 16        (one Philox block per entry)
//   pair task   : slot | pair << 8 | zbuf_base << 16     (one Box-Muller pair per entry)
//   phys entry  : float4 (A, B, C0, C1) + src word: v = C0 + C1 * f, f = (exp?) 2^(A + B x) : A + B x, where
//                 x = U(word src) for uniform kinds or z[src] for normal kinds
//                 (src bit 31: normal kind, bit 30: exp, bits 0..29: index)
constexpr int RS_MAX_PHILOX = 161, RS_MAX_PAIRS = 128 + 50;
// Philox block slots of one reset env (shared-memory layout; the task table says which are live)
enum : int {
    SL_PHYS_U = 0,        // up to 64 blocks (256 uniform-kind params)
    SL_PHYS_N = 64,       // up to 64 blocks (256 normal-kind params)
    SL_DELAY = 128,       // 5
    SL_BACKLASH = 133,    // 10 (40 normals)
    SL_LAMBDA = 143,      // 1
    SL_FORCE_P = 144,     // 1
    SL_CORR_ACT = 145,    // 5
    SL_CORR_TIP = 150,    // 4
    SL_MARKER_TIP = 154,  // 4
    SL_MARKER_BASE = 158, // 1
    SL_CORR_OBJ = 159,    // 1
    SL_CORR_ROT = 160,    // 1
    SL_COUNT = 161
};
// z buffer of one reset env: normal n of a channel at its base + n
enum : int {
    ZB_PHYS = 0,    // by normal rank, up to 256
    ZB_BL = 256,    // 40: delta_-1 normals 0..19, delta_+1 normals 20..39
    ZB_CA = 296,    // 20
    ZB_CT = 316,    // 16 (15 used)
    ZB_MT = 332,    // 16 (15 used)
    ZB_MB = 348,    // 4 (3 used)
    ZB_CO = 352,    // 4 (3 used)
    ZB_COUNT = 356
};
constexpr uint32_t RS_SRC_NORMAL = 1u << 31, RS_SRC_EXP = 1u << 30, RS_SRC_DRAW = 1u << 29, RS_SRC_IDX = (1u << 29) - 1u;

// Pointers of the device workspace.
struct DevPtrs {
    uint32_t* rec;            // [n_tiles][REC_PLANES][TILE]
    uint32_t* st;             // [n_tiles][ST_PLANES][TILE]
    float* phys;              // [n_env][n_phys]
    // physics descriptor table (global, lane-indexed in the reset kernel)
    uint32_t* pd_kind_rank;   // [256]: kind | (rank << 8)
    float* pd_a;              // [256]  a (or ln a for loguniform)
    float* pd_b;              // [256]  b (or ln b - ln a for loguniform)
    float* pd_base;           // [256]
    uint32_t* t_tab;          // [65536] force thresholds
    uint32_t* rs_philox;      // [RS_MAX_PHILOX] reset Philox tasks
    uint32_t* rs_pairs;       // [RS_MAX_PAIRS] reset Box-Muller pair tasks
    float4* rs_phys;          // [256] physics coefficients
    uint32_t* rs_src;         // [256] physics draw source
    double* dec_tab;          // [512]: 0.99^j (j < 256), then 0.99^(256 i)
    double* stats;            // [N_STAT_SLOTS][N_STATS] (internal or caller-owned)
    unsigned long long* ctl;  // [0] = step t, [1] = CTAs started counter, [2] = resets pending
    const uint8_t* occl_in;   // simulator occlusion bits per env (dr_set_occlusion_input) or NULL
};

// error / launch bookkeeping shared by every C-ABI entry point (dr_api.cu)
int set_error(int code, const char* fmt, ...);   // records the message for dr_last_error(), returns code
void count_launch();                              // one library kernel enqueued

// launchers (dr_kernels.cu)
cudaError_t upload_const(const DevConst& c, cudaStream_t s);
cudaError_t launch_reset(const DevPtrs& p, const uint8_t* mask, bool first, uint32_t n_env,
                         int grid, cudaStream_t s);
cudaError_t launch_step(const DevPtrs& p, uint32_t layer_mask, const float* actions,
                        const float* raw_obs, float* out_actions, float* out_obs, float* out_dt,
                        float* out_force, float* out_sub, uint32_t n_env, int grid, cudaStream_t s);
cudaError_t launch_export(const DevPtrs& p, void* dst, uint32_t lo, uint32_t hi, cudaStream_t s);
cudaError_t launch_import(const DevPtrs& p, const void* src, uint32_t lo, uint32_t hi, cudaStream_t s);
cudaError_t launch_debug_philox(uint32_t n_env, uint32_t dom, uint32_t ch, uint32_t blk, uint32_t* out,
                                cudaStream_t s);
int step_max_ctas_per_sm(uint32_t layer_mask);
void set_step_prefetch(int mode);
void set_step_pipe(int mode);
void set_step_mode(int mode);   // 0 throughput, 1 latency
int step_mode();
// latency mode up to this many envs per job (n_env_global).  Measured (profiles/round1_notes.md):
// 4,096 envs 7.3 us vs 9.6 us per step; 65,536 envs 26 us vs 21 us -- so only small jobs
constexpr int64_t LAT_MAX_ENVS = 16384;
constexpr int LAT_ENVS_PER_CTA = 32;
int reset_max_ctas_per_sm();
void set_reset_version(int v);
void set_pdl(bool on);            // programmatic dependent launch of the step / reset kernels (DR_PDL, default on)
int reset_grid_for(uint32_t n_env, int sm_count);
constexpr int RESET_THREADS = 256;
constexpr int STEP_THREADS = TILE;
#ifndef DR_STEP_MIN_CTAS
#define DR_STEP_MIN_CTAS 4
#endif
// __launch_bounds__ occupancy target: 4 CTAs/SM (<= 128 regs) measured fastest with the
// warp-cooperative ring (4.10e9 vs 4.04e9 env-steps/s at 3 CTAs/SM; profiles/round1_notes.md)
constexpr int STEP_MIN_CTAS = DR_STEP_MIN_CTAS;
#ifndef DR_SFU_NORMALS
#define DR_SFU_NORMALS 1
#endif
// step-kernel normals for actions / fingertips / object / rotation axis take the Box-Muller angle
// from the SFU (dr_device.cuh: box_muller_sfu); force and reset draws never do
constexpr bool kSfuNormals = DR_SFU_NORMALS != 0;

}  // namespace dr
