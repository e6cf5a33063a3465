// dr_kernels.cu -- sm_100a kernels of the domain-randomization pipeline.
// One translation unit (the __constant__ parameters are shared by every kernel):
//   dr_reset.cuh : reset_kernel -- episode-reset sampling, warp-cooperative
//   dr_step.cuh  : step_kernel<LayerMask, Prefetch> -- the fused per-env-step transform
//   below        : checkpoint export/import, the Philox test hook, and the host launchers.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "dr_device.cuh"
#include "dr_internal.h"

namespace dr {

template <uint32_t L>
__device__ __forceinline__ bool on(uint32_t bit) {
    if constexpr (L == RUNTIME_MASK) return (c_dc.layer_mask & bit) != 0;
    else return (L & bit) != 0;
}

enum : uint32_t {
    B_TIMING = 1u << 0, B_ACT_NOISE = 1u << 1, B_DELAY = 1u << 2, B_BACKLASH = 1u << 3,
    B_OBS_NOISE = 1u << 4, B_DROPOUT = 1u << 5, B_OCCLUSION = 1u << 6, B_FORCE = 1u << 7,
    B_PHYS = 1u << 8, B_SMOOTH = 1u << 9, B_SUBSTEP = 1u << 10
};
// layers that own per-env state planes (their state is "fresh" = zero after a reset)
constexpr uint32_t B_STATEFUL = B_DELAY | B_BACKLASH | B_DROPOUT | B_OCCLUSION | B_FORCE | B_SMOOTH;

#include "dr_reset.cuh"
#include "dr_step.cuh"
#include "dr_step_lat.cuh"

// =====================================================================================
// Export / import (dr_env_state, 168 words per env).  A FRESH env exports its logical state
// (all zero); import writes explicit state (clears FRESH).
// =====================================================================================
constexpr int EXP_WORDS = 168;

__global__ void export_kernel(DevPtrs p, uint32_t* __restrict__ dst, uint32_t lo, uint32_t hi) {
    const uint32_t e = lo + blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= hi) return;
    constexpr size_t P = PLANE;
    const uint32_t* R = p.rec + rec_index(e);
    const uint32_t* S = p.st + st_index(e);
    uint32_t* o = dst + (size_t)(e - lo) * EXP_WORDS;
    const uint32_t flags = S[ST_FLAGS * P];
    const bool fresh = flags & FRESH_BIT;
    o[0] = R[REC_EPISODE * P];
    o[1] = R[REC_DELAY * P];
    o[2] = R[REC_PINDEX * P];
    o[3] = R[REC_TFORCE * P];
    o[4] = fresh ? 0u : flags;
    o[5] = fresh ? 0u : S[ST_KF * P];
    o[6] = R[REC_LAMBDA * P];
    o[7] = R[REC_MASS * P];
    for (int i = 0; i < REC_STEP_PLANES - REC_DNEG; ++i) o[8 + i] = R[(REC_DNEG + i) * P];   // 82 words
    for (int i = 0; i < ST_FLAGS; ++i) o[90 + i] = fresh ? 0u : S[i * P];                     // 55 words
    for (int i = 0; i < 3; ++i) o[145 + i] = fresh ? 0u : S[(ST_FTRIG + i) * P];
    for (int i = 0; i < N_ACT; ++i) o[148 + i] = fresh ? 0u : S[(ST_EMA + i) * P];
}

__global__ void import_kernel(DevPtrs p, const uint32_t* __restrict__ src, uint32_t lo, uint32_t hi) {
    const uint32_t e = lo + blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= hi) return;
    constexpr size_t P = PLANE;
    uint32_t* R = p.rec + rec_index(e);
    uint32_t* S = p.st + st_index(e);
    const uint32_t* o = src + (size_t)(e - lo) * EXP_WORDS;
    R[REC_EPISODE * P] = o[0];
    R[REC_DELAY * P] = o[1];
    R[REC_PINDEX * P] = o[2];
    R[REC_TFORCE * P] = o[3];
    S[ST_FLAGS * P] = o[4] & ~FRESH_BIT;
    S[ST_KF * P] = o[5];
    R[REC_LAMBDA * P] = o[6];
    const float lam = __uint_as_float(o[6]);
    R[REC_INVLAM * P] = __float_as_uint(lam > 0.f ? 1.0f / lam : 0.f);
    R[REC_MASS * P] = o[7];
    for (int i = 0; i < REC_STEP_PLANES - REC_DNEG; ++i) R[(REC_DNEG + i) * P] = o[8 + i];
    for (int i = 0; i < ST_FLAGS; ++i) S[i * P] = o[90 + i];
    for (int i = 0; i < 3; ++i) S[(ST_FTRIG + i) * P] = o[145 + i];
    for (int i = 0; i < N_ACT; ++i) S[(ST_EMA + i) * P] = o[148 + i];
}

__global__ void debug_philox_kernel(uint32_t n_env, uint32_t dom, uint32_t ch, uint32_t blk, uint4* __restrict__ out) {
    const uint32_t e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e < n_env) out[e] = philox(c_dc.env_offset + e, dom, ch, blk);
}

// =====================================================================================
// launchers
// =====================================================================================
cudaError_t upload_const(const DevConst& c, cudaStream_t s) {
    return cudaMemcpyToSymbolAsync(c_dc, &c, sizeof(DevConst), 0, cudaMemcpyHostToDevice, s);
}

// Reset kernel (DR_RESET at dr_init, A/B): 6 = thread-per-env record chain + warp-per-env physics
// rows (reset_kernel_h, default; config 5 reset + step 0.418-0.425 ms vs v3's 0.458-0.460),
// 3 = thread per resetting env over a compacted list (reset_kernel_t), 5 = task-split over
// (task, env) items (reset_kernel_v5), 2 = warp per resetting env in four lane-parallel phases
// (reset_kernel).
// Step and reset kernels go out with cudaLaunchAttributeProgrammaticStreamSerialization: each waits
// (griddepcontrol.wait) for the previous kernel before its first global access, so consecutive
// steps overlap launch latency with the previous grid's tail (dr_device.cuh).  DR_PDL=0: plain launches.
static bool g_pdl = true;
void set_pdl(bool on) { g_pdl = on; }

template <typename... KArgs, typename... Args>
static cudaError_t launch_k(void (*kernel)(KArgs...), int grid, int block, size_t smem, cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)grid, 1, 1);
    cfg.blockDim = dim3((unsigned)block, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = g_pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, args...);
}

static int g_reset_v = 6;
void set_reset_version(int v) { g_reset_v = (v == 2 || v == 3 || v == 5) ? v : 6; }

cudaError_t launch_reset(const DevPtrs& p, const uint8_t* mask, bool first, uint32_t n_env, int grid,
                         cudaStream_t s) {
    const int f = first ? 1 : 0;
    if (g_reset_v == 2) return launch_k(reset_kernel, grid, RESET_THREADS, 0, s, p, mask, f, n_env);
    if (g_reset_v == 5) {
        // per-CTA range: the envs split evenly over the grid, in whole 32-env chunks, <= R5_RANGE
        const uint32_t per = (uint32_t)(((unsigned long long)n_env + grid - 1) / grid);
        const uint32_t range = std::min<uint32_t>(R5_RANGE, std::max<uint32_t>(32u, (per + 31u) & ~31u));
        return launch_k(reset_kernel_v5, grid, R5_THREADS, 0, s, p, mask, f, n_env, range);
    }
    if (g_reset_v == 6) return launch_k(reset_kernel_h, grid, RH_THREADS, 0, s, p, mask, f, n_env);
    return launch_k(reset_kernel_t, grid, RT_THREADS, 0, s, p, mask, f, n_env);
}

int reset_grid_for(uint32_t n_env, int sm_count) {
    int n = 0;
    if (g_reset_v == 2) {
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, reset_kernel, RESET_THREADS, 0) != cudaSuccess || n < 1) n = 1;
        const long long chunks = (n_env + 31) / 32;
        return (int)std::max<long long>(1, std::min<long long>((chunks + 7) / 8, (long long)sm_count * n));
    }
    if (g_reset_v == 5) {
        // one resident wave: as many CTAs as fit (6 per SM), fewer for small jobs (>= 32 envs each)
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, reset_kernel_v5, R5_THREADS, 0) != cudaSuccess || n < 1) n = 1;
        const long long ranges = (n_env + 31) / 32;
        return (int)std::max<long long>(1, std::min<long long>(ranges, (long long)sm_count * n));
    }
    if (g_reset_v == 6) {
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, reset_kernel_h, RH_THREADS, 0) != cudaSuccess || n < 1) n = 1;
        const long long ranges = (n_env + RH_RANGE - 1) / RH_RANGE;
        return (int)std::max<long long>(1, std::min<long long>(ranges, (long long)sm_count * n));
    }
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, reset_kernel_t, RT_THREADS, 0) != cudaSuccess || n < 1) n = 1;
    const long long ranges = (n_env + RT_RANGE - 1) / RT_RANGE;
    return (int)std::max<long long>(1, std::min<long long>(ranges, (long long)sm_count * n));
}

static constexpr uint32_t MASK_FULL = 0xFFu;  // PHYS does not affect the step
static constexpr uint32_t MASK_CFG2 = B_TIMING | B_ACT_NOISE | B_BACKLASH | B_OBS_NOISE;

typedef void (*StepFn)(const DevPtrs, const float*, const float*, float*, float*, float*, float*, float*, uint32_t);

// Optional TMA bulk L2 prefetch policy of the step kernel (DR_PREFETCH=0/1/2; A/B experiments).
// Measured on B200 at 1M envs with the v1 kernel: 0 = none 2.48e9 env-steps/s, 1 = current tile
// 2.10e9, 2 = next tile 1.92e9; the cp.async phase ring (v3+) makes it moot.
static int g_prefetch = 0;

void set_step_prefetch(int mode) { g_prefetch = (mode < 0 || mode > 2) ? 0 : mode; }

// Ring pipeline of the step kernel (DR_PIPE at dr_init): 2 = warp-cooperative 16-byte cp.async.cg
// ring (step_kernel_warp, default), 0 = per-thread 4-byte cp.async ring (step_kernel), 1 = CTA-wide
// TMA bulk-copy ring (step_kernel_tma).  Measured on B200, 1M envs, full pipeline
// (profiles/round1_notes.md), env-steps/s at 3 / 4 CTAs per SM:
//   pipe 2: 4.04e9 / 4.10e9   pipe 0: 3.65e9 / 3.47e9   pipe 1: - / 3.27e9
// Pipe 2 issues 4x fewer LDGSTS and bypasses L1 (the 4-byte .ca copies of pipe 0 allocate L1 lines,
// which thrash once 4 CTAs leave ~24 KB of L1); pipe 1 couples the CTA's warps (a slot is refilled
// only after the slowest warp releases it).
static int g_pipe = 2;

void set_step_pipe(int mode) { g_pipe = (mode < 0 || mode > 2) ? 2 : mode; }

#ifndef DR_WARP_PF
#define DR_WARP_PF 0
#endif
#ifndef DR_WARP_XT
#define DR_WARP_XT 1   // cross-tile pipelining of S0 / A0 (A/B)
#endif
static StepFn step_fn_warp(uint32_t m) {
    if (m == MASK_FULL) return step_kernel_warp<MASK_FULL, DR_WARP_PF, DR_WARP_XT != 0>;
    if (m == MASK_CFG2) return step_kernel_warp<MASK_CFG2, DR_WARP_PF, DR_WARP_XT != 0>;
    return step_kernel_warp<RUNTIME_MASK, DR_WARP_PF, DR_WARP_XT != 0>;
}

template <int PF>
static StepFn step_fn_pf(uint32_t m) {
    if (m == MASK_FULL) return step_kernel<MASK_FULL, PF>;
    if (m == MASK_CFG2) return step_kernel<MASK_CFG2, PF>;
    return step_kernel<RUNTIME_MASK, PF>;
}

static StepFn step_fn_tma(uint32_t m) {
    if (m == MASK_FULL) return step_kernel_tma<MASK_FULL>;
    if (m == MASK_CFG2) return step_kernel_tma<MASK_CFG2>;
    return step_kernel_tma<RUNTIME_MASK>;
}

// Step mode (chosen at dr_init from n_env_global): 0 = throughput (one thread per
// env, persistent tiles), 1 = latency (8 warps split one 32-env group's transform).
static int g_step_mode = 0;
void set_step_mode(int mode) { g_step_mode = mode ? 1 : 0; }
int step_mode() { return g_step_mode; }

static StepFn step_fn_lat(uint32_t m) {
    if (m == MASK_FULL) return step_kernel_lat<MASK_FULL>;
    if (m == MASK_CFG2) return step_kernel_lat<MASK_CFG2>;
    return step_kernel_lat<RUNTIME_MASK>;
}

static StepFn step_fn(uint32_t layer_mask) {
    // PHYS does not affect the step; the variants (SMOOTH, SUBSTEP) run the runtime-mask kernel
    const uint32_t m = layer_mask & 0x6FFu;
    if (g_step_mode == 1) return step_fn_lat(m);
    if (g_pipe == 1) return step_fn_tma(m);
    if (g_pipe == 2) return step_fn_warp(m);
    if (g_prefetch == 0) return step_fn_pf<0>(m);
    if (g_prefetch == 2) return step_fn_pf<2>(m);
    return step_fn_pf<1>(m);
}

static size_t step_dyn_smem() { return g_step_mode == 1 ? 0 : (g_pipe == 1 ? STEP_TMA_DYN_SMEM : STEP_DYN_SMEM); }
static int step_threads() { return g_step_mode == 1 ? LAT_THREADS : STEP_THREADS; }

// the phase ring is dynamic shared memory (static + dynamic > 48 KB needs the opt-in attribute)
static StepFn step_fn_ready(uint32_t layer_mask) {
    StepFn f = step_fn(layer_mask);
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)step_dyn_smem());
    return f;
}

int step_max_ctas_per_sm(uint32_t layer_mask) {
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, step_fn_ready(layer_mask), step_threads(), step_dyn_smem()) !=
        cudaSuccess)
        return 1;
    return n > 0 ? n : 1;
}

int reset_max_ctas_per_sm() {
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, reset_kernel, RESET_THREADS, 0) != cudaSuccess) return 1;
    return n > 0 ? n : 1;
}

cudaError_t launch_step(const DevPtrs& p, uint32_t layer_mask, const float* actions, const float* raw_obs,
                        float* out_actions, float* out_obs, float* out_dt, float* out_force, float* out_sub,
                        uint32_t n_env, int grid, cudaStream_t s) {
    return launch_k(step_fn(layer_mask), grid, step_threads(), step_dyn_smem(), s, p, actions, raw_obs, out_actions,
                    out_obs, out_dt, out_force, out_sub, n_env);
}

cudaError_t launch_debug_philox(uint32_t n_env, uint32_t dom, uint32_t ch, uint32_t blk, uint32_t* out, cudaStream_t s) {
    debug_philox_kernel<<<(n_env + 127) / 128, 128, 0, s>>>(n_env, dom, ch, blk, reinterpret_cast<uint4*>(out));
    return cudaGetLastError();
}

cudaError_t launch_export(const DevPtrs& p, void* dst, uint32_t lo, uint32_t hi, cudaStream_t s) {
    const uint32_t n = hi - lo;
    export_kernel<<<(n + 127) / 128, 128, 0, s>>>(p, static_cast<uint32_t*>(dst), lo, hi);
    return cudaGetLastError();
}

cudaError_t launch_import(const DevPtrs& p, const void* src, uint32_t lo, uint32_t hi, cudaStream_t s) {
    const uint32_t n = hi - lo;
    import_kernel<<<(n + 127) / 128, 128, 0, s>>>(p, static_cast<const uint32_t*>(src), lo, hi);
    return cudaGetLastError();
}

}  // namespace dr
