// dr_kernels.cu -- sm_100a kernels of the domain-randomization pipeline.
// One translation unit (the __constant__ parameters are shared by every kernel):
//   dr_reset.cuh    : reset_kernel -- episode-reset sampling
//   dr_step.cuh     : step_kernel_warp<LayerMask> -- the fused per-env-step transform (throughput mode)
//   dr_step_lat.cuh : step_kernel_lat<LayerMask> -- the same transform, 8 warps per 32 envs (latency mode)
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
// Export / import (dr_env_state, 168 words per env, include/dr.h).  A FRESH env exports its logical
// state (all zero); import writes explicit state (clears FRESH), then import_phys_kernel re-derives
// the imported envs' physics rows from (seed, global id, imported episode index): the rows are a
// pure function of those (PAPER.md:7-8 draws, keyed like every reset draw), so a resumed context
// holds the same rows as the one that was exported (under the same parameters).
// dr_env_state words: 0 episode, 1 delay, 2 p-index, 3 t_force, 4 flags, 5 k_f, 6 lambda, 7 mass,
// 8 dneg[20], 28 dpos[20], 48 c_act[20], 68 off_tip[15], 83 c_obj[3], 86 q_c[4], 90 prev[20],
// 110 slack[20], 130 last[15], 145 f_trig[3], 148 ema[20].
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
    o[0] = R[rec_off(e, REC_EPISODE)];
    o[1] = R[rec_off(e, REC_DELAY)];
    o[2] = R[rec_off(e, REC_PINDEX)];
    o[3] = R[rec_off(e, REC_TFORCE)];
    o[4] = fresh ? 0u : flags;
    o[5] = fresh ? 0u : S[ST_KF * P];
    o[6] = R[rec_off(e, REC_LAMBDA)];
    o[7] = R[rec_off(e, REC_MASS)];
    for (int j = 0; j < N_ACT; ++j) {
        o[8 + j] = R[rec_off(e, rec_dneg(j))];
        o[28 + j] = R[rec_off(e, rec_dpos(j))];
        o[48 + j] = R[rec_off(e, rec_cact(j))];
    }
    for (int i = 0; i < 22; ++i) o[68 + i] = R[rec_off(e, REC_OFFTIP + i)];                        // off_tip, c_obj, q_c
    for (int i = 0; i < ST_FLAGS; ++i) o[90 + i] = fresh ? 0u : S[i * P];                     // prev, slack, last
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
    R[rec_off(e, REC_EPISODE)] = o[0];
    R[rec_off(e, REC_DELAY)] = o[1];
    R[rec_off(e, REC_PINDEX)] = o[2];
    R[rec_off(e, REC_TFORCE)] = o[3];
    S[ST_FLAGS * P] = o[4] & ~FRESH_BIT;
    S[ST_KF * P] = o[5];
    R[rec_off(e, REC_LAMBDA)] = o[6];
    const float lam = __uint_as_float(o[6]);
    R[rec_off(e, REC_INVLAM)] = __float_as_uint(lam > 0.f ? 1.0f / lam : 0.f);
    R[rec_off(e, REC_MASS)] = o[7];
    for (int j = 0; j < N_ACT; ++j) {
        R[rec_off(e, rec_dneg(j))] = o[8 + j];
        R[rec_off(e, rec_dpos(j))] = o[28 + j];
        R[rec_off(e, rec_cact(j))] = o[48 + j];
    }
    for (int i = 0; i < 22; ++i) R[rec_off(e, REC_OFFTIP + i)] = o[68 + i];
    for (int i = 0; i < ST_FLAGS; ++i) S[i * P] = o[90 + i];
    for (int i = 0; i < 3; ++i) S[(ST_FTRIG + i) * P] = o[145 + i];
    for (int i = 0; i < N_ACT; ++i) S[(ST_EMA + i) * P] = o[148 + i];
}

// Physics rows of envs [lo, hi) from their (imported) episode index: a warp per env, as in the reset.
constexpr int IMPORT_PHYS_THREADS = 256;
__global__ void __launch_bounds__(IMPORT_PHYS_THREADS) import_phys_kernel(DevPtrs p, uint32_t lo, uint32_t hi) {
    __shared__ float4 s_pd[MAX_PHYS];
    __shared__ __align__(16) uint32_t s_src[MAX_PHYS];
    __shared__ __align__(16) float s_dr[IMPORT_PHYS_THREADS / 32][RH_DRAW];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    stage_phys_tables(p, s_pd, s_src, tid, IMPORT_PHYS_THREADS);
    if (lane == 0) s_dr[wid][RS_OFF_ZERO] = 0.f;
    __syncthreads();
    const bool phys_on = (c_dc.layer_mask & B_PHYS) != 0;
    const int nub = phys_on ? (c_dc.n_phys_u + 3) / 4 : 0;
    const int nnb = phys_on ? (c_dc.n_phys_n + 3) / 4 : 0;
    const uint32_t e = lo + blockIdx.x * (IMPORT_PHYS_THREADS / 32) + wid;
    if (e >= hi) return;
    reset_phys_warp(p, e, p.rec[rec_index(e) + rec_off(e, REC_EPISODE)], lane, s_dr[wid], s_pd, s_src, nub, nnb);
}

__global__ void debug_philox_kernel(uint32_t n_env, uint32_t dom, uint32_t ch, uint32_t blk, uint4* __restrict__ out) {
    const uint32_t e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e < n_env) out[e] = philox(c_dc.env_offset + e, dom, ch, blk);
}

// Keyed test hook: the same round function on arbitrary (counter, key) pairs, round keys built in
// registers from the key (the key schedule dr_api.cu precomputes for a context).
__global__ void debug_philox_keyed_kernel(const uint4* __restrict__ ctr, const uint2* __restrict__ key,
                                          uint4* __restrict__ out, unsigned long long n) {
    const unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint4 c = ctr[i];
    const uint2 k = key[i];
    PhiloxKeys rk;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        rk.rk0[r] = k.x + (uint32_t)r * 0x9E3779B9u;
        rk.rk1[r] = k.y + (uint32_t)r * 0xBB67AE85u;
    }
    out[i] = philox_rounds(c.x, c.y, c.z, c.w, rk);
}

// =====================================================================================
// launchers
// =====================================================================================
cudaError_t upload_const(const DevConst& c, cudaStream_t s) {
    return cudaMemcpyToSymbolAsync(c_dc, &c, sizeof(DevConst), 0, cudaMemcpyHostToDevice, s);
}

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

cudaError_t launch_reset(const DevPtrs& p, const uint8_t* mask, bool first, uint32_t n_env, int grid,
                         cudaStream_t s, bool early_scan) {
    return launch_k(reset_kernel, grid, RH_THREADS, 0, s, p, mask, first ? 1 : 0, n_env, early_scan ? 1 : 0);
}

int reset_grid_for(uint32_t n_env, int sm_count) {
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, reset_kernel, RH_THREADS, 0) != cudaSuccess || n < 1) n = 1;
    const long long ranges = (n_env + 31) / 32;   // 32-env mask chunks
    return (int)std::max<long long>(1, std::min<long long>(ranges, (long long)sm_count * n));
}

static constexpr uint32_t MASK_FULL = 0xFFu;  // PHYS does not affect the step
static constexpr uint32_t MASK_CFG2 = B_TIMING | B_ACT_NOISE | B_BACKLASH | B_OBS_NOISE;

typedef void (*StepFn)(const DevPtrs, const float*, const float*, float*, float*, float*, float*, float*, uint32_t, int);

static StepFn step_fn_warp(uint32_t m) {
    if (m == MASK_FULL) return step_kernel_warp<MASK_FULL>;
    if (m == MASK_CFG2) return step_kernel_warp<MASK_CFG2>;
    return step_kernel_warp<RUNTIME_MASK>;
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
    return g_step_mode == 1 ? step_fn_lat(m) : step_fn_warp(m);
}

static size_t step_dyn_smem() { return g_step_mode == 1 ? 0 : STEP_DYN_SMEM; }
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

cudaError_t launch_step(const DevPtrs& p, uint32_t layer_mask, const float* actions, const float* raw_obs,
                        float* out_actions, float* out_obs, float* out_dt, float* out_force, float* out_sub,
                        uint32_t n_env, int grid, int chain, cudaStream_t s) {
    return launch_k(step_fn(layer_mask), grid, step_threads(), step_dyn_smem(), s, p, actions, raw_obs, out_actions,
                    out_obs, out_dt, out_force, out_sub, n_env, chain);
}

__global__ void sync_init_kernel(DevPtrs p, unsigned long long t, uint32_t grid, uint32_t max_ctas) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    // the slot of step t starts cleared and empty (as if step t - 1 had prepared it); every other
    // slot's previous owner counts as done
    if (i < N_STAT_SLOTS) p.done[i] = (i == (uint32_t)(t % N_STAT_SLOTS)) ? 0u : grid;
    if (i < max_ctas) p.cta_done[i] = p.cta_ready[i] = (uint32_t)t;     // steps < t finished
    if (i == 0) {
        p.ctl[0] = t;
        p.ctl[4] = t * grid;   // the first ticket of step t
    }
}

cudaError_t launch_sync_init(const DevPtrs& p, uint64_t t, int grid, int max_ctas, cudaStream_t s) {
    const uint32_t n = std::max<uint32_t>((uint32_t)max_ctas, (uint32_t)N_STAT_SLOTS);
    sync_init_kernel<<<(n + 255) / 256, 256, 0, s>>>(p, (unsigned long long)t, (uint32_t)grid, (uint32_t)max_ctas);
    return cudaGetLastError();
}

cudaError_t launch_debug_philox(uint32_t n_env, uint32_t dom, uint32_t ch, uint32_t blk, uint32_t* out, cudaStream_t s) {
    debug_philox_kernel<<<(n_env + 127) / 128, 128, 0, s>>>(n_env, dom, ch, blk, reinterpret_cast<uint4*>(out));
    return cudaGetLastError();
}

cudaError_t launch_debug_philox_keyed(const uint32_t* ctr, const uint32_t* key, uint32_t* out, unsigned long long n,
                                      cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    debug_philox_keyed_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(
        reinterpret_cast<const uint4*>(ctr), reinterpret_cast<const uint2*>(key), reinterpret_cast<uint4*>(out), n);
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
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    constexpr uint32_t W = IMPORT_PHYS_THREADS / 32;
    import_phys_kernel<<<(n + W - 1) / W, IMPORT_PHYS_THREADS, 0, s>>>(p, lo, hi);
    return cudaGetLastError();
}

}  // namespace dr

#ifdef DR_PROBE_TIMING
// A/B probe only: read (or, reset_min != 0, re-arm) the reset kernel's per-CTA stamps.
extern "C" int dr_debug_probe_read(void* dst, size_t bytes, int reset_min) {
    if (reset_min) {   // slot 5 (first warp done) collects a minimum
        static unsigned long long init[4096][8];
        for (auto& r : init) {
            for (auto& v : r) v = 0ull;
            r[5] = ~0ull;
        }
        return (int)cudaMemcpyToSymbol(dr::g_probe_reset, init, sizeof(init));
    }
    return (int)cudaMemcpyFromSymbol(dst, dr::g_probe_reset, bytes < sizeof(dr::g_probe_reset) ? bytes : sizeof(dr::g_probe_reset));
}
#endif
