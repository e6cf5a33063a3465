// dr_internal.h -- shared between the host library (dr_api.cu) and the kernels (dr_kernels.cu).
// Device data layout:
//   rec  : episode record, [n_tiles][REC_GROUPS][TILE][8] 4-byte words: record word w of env e is
//          word w % 8 of the 32-byte group w / 8 of that env (halves swapped when bit 2 of e is set,
//          rec_off), so the eight words of a group are one DRAM sector of ONE env.  A reset rewrites whole sectors (no L2 read-fill of partially
//          written sectors), and the step reads a group of its 32 consecutive envs as 1 KB of
//          contiguous memory (16-byte cp.async per half group, coalesced).
//   st   : mutable per-env state, [n_tiles][ST_PLANES][TILE] (plane k of env e at k * TILE + e % TILE:
//          a warp's 32 consecutive envs read and write one 128-byte line per plane)
//   phys : [n_env][n_phys] fp32, row-major (the simulator reads rows)
// A tile's whole record / state is one contiguous block.
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

// ---- record words (REC_WORDS per env, 12 sector groups of 8).  Grouped by the step kernel's phases
// (dr_step.cuh): group 0 = the S0 scalars + c_act 0..3, groups 1..5 = (delta-1, delta+1) of actuators
// 4b..4b+3, groups 6..7 = c_act 4..19, groups 8..10 = the observation offsets (+ lambda, p-index),
// group 11 = the episode counter (the step never reads it).
enum : int {
    REC_DELAY = 0,   // u32 delay bits
    REC_INVLAM = 1,  // 1/lambda (the step only needs the reciprocal rate)
    REC_TFORCE = 2,  // u32 force threshold
    REC_MASS = 3,
    REC_G_BL = 1,    // groups 1..5: words 8 + 8b + q = delta-1 of actuator 4b + q, 12 + 8b + q = delta+1
    REC_OFFTIP = 64, // 15
    REC_COBJ = 79,   // 3
    REC_QC = 82,     // 4
    REC_LAMBDA = 86,
    REC_PINDEX = 87, // u32
    REC_EPISODE = 88,// u32
    REC_STEP_GROUPS = 11,   // groups 0..10 are read by the step kernel
    REC_GROUPS = 12,
    REC_WORDS = 8 * REC_GROUPS
};
__host__ __device__ constexpr int rec_dneg(int j) { return 8 + 8 * (j >> 2) + (j & 3); }
__host__ __device__ constexpr int rec_dpos(int j) { return 12 + 8 * (j >> 2) + (j & 3); }
__host__ __device__ constexpr int rec_cact(int j) { return j < 4 ? 4 + j : 44 + j; }
// Word offset of record word w of env e from the env's base (rec_index): group w / 8, word w % 8 --
// with the two 16-byte halves of every group swapped for envs with bit 2 of e set.  The step kernel
// copies groups into shared memory sector by sector (a sector must land contiguously) and thread e
// reads its half h at chunk h ^ swz: within a quarter-warp, envs 0-3 and 4-7 of each 8 then hit
// different 16-byte bank groups (an LDS.128 of the same logical half is conflict-free).
__host__ __device__ constexpr uint32_t rec_swz(uint32_t e) { return ((e >> 2) & 1u) << 2; }
__host__ __device__ constexpr size_t rec_off(uint32_t e, int w) {
    return (size_t)(w >> 3) * (TILE * 8) + ((uint32_t)(w & 7) ^ rec_swz(e));
}
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

// word offset of env e's record word 0 (record word w at + rec_off(w))
__host__ __device__ __forceinline__ size_t rec_index(uint32_t e) {
    return (size_t)(e / TILE) * (REC_WORDS * TILE) + (size_t)(e % TILE) * 8;
}
// AoSoA state addressing: word offset of env e's plane 0; plane k is at + k * TILE.
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
};

// Physics table of the reset kernel (built on the host at dr_init): per parameter q, rs_phys[q] =
// (A, B, C0, C1) and rs_src[q] = draw-buffer offset of its x | exp flag (bit 31), with
// v = C0 + C1 * f(A + B x), f = 2^(.) for the exp kinds (A, B in log2 units), x = the u-th uniform
// (offset u), the n-th normal (offset 256 + n) or the constant 0 (offset 512, draw-free kinds).
constexpr uint32_t RS_EXP = 1u << 31;
constexpr uint32_t RS_OFF_NORMAL = MAX_PHYS, RS_OFF_ZERO = 2 * MAX_PHYS;
// Buffer word of the i-th uniform (or, + RS_OFF_NORMAL, the i-th normal): draw j of Philox block b
// (i = 4 b + j) at j * 64 + b, bank-conflict-free for the reset's physics-row evaluation.
constexpr uint32_t rs_slot(uint32_t i) { return (i & 3u) * 64u + (i >> 2); }

// Pointers of the device workspace.
struct DevPtrs {
    uint32_t* rec;            // [n_tiles][REC_GROUPS][TILE][8]
    uint32_t* st;             // [n_tiles][ST_PLANES][TILE]
    float* phys;              // [n_env][n_phys]
    uint32_t* t_tab;          // [65536] force thresholds
    float4* rs_phys;          // [256] physics coefficients (A, B, C0, C1)
    uint32_t* rs_src;         // [256] physics draw-buffer offset | RS_EXP
    double* dec_tab;          // [512]: 0.99^j (j < 256), then 0.99^(256 i)
    double* stats;            // [N_STAT_SLOTS][N_STATS] (internal or caller-owned)
    unsigned long long* ctl;  // [0] = step t (host-visible), [2] = resets pending, [4] = CTA-start tickets
    uint32_t* done;           // [N_STAT_SLOTS]: CTAs of the step that owns stats slot i that finished their atomics
    uint32_t* cta_done;       // [max CTAs]: steps whose CTA of this index has finished (dr_step.cuh)
    uint32_t* cta_ready;      // [max CTAs]: steps whose CTA of this index has published its state stores
    const uint8_t* occl_in;   // simulator occlusion bits per env (dr_set_occlusion_input) or NULL
};

// error / launch bookkeeping shared by every C-ABI entry point (dr_api.cu)
int set_error(int code, const char* fmt, ...);   // records the message for dr_last_error(), returns code
void count_launch();                              // one library kernel enqueued
// The last libdr kernel enqueued on each stream (dr_api.cu), for programmatic-dependent-launch
// decisions: an image augmentation may write early only behind the previous augmentation of its
// stream (dr_vision.cu), and a chained step only directly behind a step of its context.
struct AugRec {
    const void* images;
    size_t img_bytes;
    const void* out;
    size_t out_bytes;
    const void* st;
    size_t st_bytes;
};
enum : int { LAUNCH_UNKNOWN = -1, LAUNCH_OTHER = 0, LAUNCH_AUGMENT = 1, LAUNCH_STEP = 2 };
// aug: the augmentation's buffers (kind LAUNCH_AUGMENT), or NULL with kind LAUNCH_OTHER / LAUNCH_STEP
void note_stream_launch(void* stream, const AugRec* aug, int kind = LAUNCH_OTHER);
bool last_launch_is_augment(void* stream, AugRec* prev);    // and, if so, its buffers
int last_launch_kind(void* stream);                         // LAUNCH_* (UNKNOWN if not in the table)

// launchers (dr_kernels.cu)
cudaError_t upload_const(const DevConst& c, cudaStream_t s);
cudaError_t launch_reset(const DevPtrs& p, const uint8_t* mask, bool first, uint32_t n_env,
                         int grid, cudaStream_t s, bool early_scan = false);
cudaError_t launch_step(const DevPtrs& p, uint32_t layer_mask, const float* actions,
                        const float* raw_obs, float* out_actions, float* out_obs, float* out_dt,
                        float* out_force, float* out_sub, uint32_t n_env, int grid, int chain, cudaStream_t s);
// (re)arm the step protocol at step index t for a step grid of `grid` CTAs (dr_init, dr_set_step_index)
cudaError_t launch_sync_init(const DevPtrs& p, uint64_t t, int grid, int max_ctas, cudaStream_t s);
cudaError_t launch_export(const DevPtrs& p, void* dst, uint32_t lo, uint32_t hi, cudaStream_t s);
cudaError_t launch_import(const DevPtrs& p, const void* src, uint32_t lo, uint32_t hi, cudaStream_t s);
cudaError_t launch_debug_philox(uint32_t n_env, uint32_t dom, uint32_t ch, uint32_t blk, uint32_t* out,
                                cudaStream_t s);
cudaError_t launch_debug_philox_keyed(const uint32_t* ctr, const uint32_t* key, uint32_t* out, unsigned long long n,
                                      cudaStream_t s);
int step_max_ctas_per_sm(uint32_t layer_mask);
void set_step_mode(int mode);   // 0 throughput, 1 latency
int step_mode();
// latency mode up to this many envs per job (n_env_global).  Measured (profiles/round1_notes.md):
// 4,096 envs 7.3 us vs 9.6 us per step; 65,536 envs 26 us vs 21 us -- so only small jobs
constexpr int64_t LAT_MAX_ENVS = 16384;
constexpr int LAT_ENVS_PER_CTA = 32;
void set_pdl(bool on);            // programmatic dependent launch of the step / reset kernels (DR_PDL, default on)
int reset_grid_for(uint32_t n_env, int sm_count);
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
