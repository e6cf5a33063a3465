// dr_kernels.cu -- sm_100a kernels of the domain-randomization pipeline.
//
//  reset_kernel : episode-reset sampling.
//                 Warp-cooperative: a warp ballots 32 mask bytes, then serves each resetting env
//                 with all 32 lanes (Philox blocks spread over lanes into shared memory, then one
//                 lane per field; the [n_phys] parameter row is written as coalesced 128-B lines).
//  step_kernel  : the fused per-env-step transform.  Persistent CTAs, one thread
//                 per env, TILE envs per CTA tile: the row-major I/O tiles are staged through
//                 shared memory with 128-bit coalesced loads/stores, the SoA record/state planes are
//                 read/written directly (coalesced: 32 lanes = one 128-B line per plane), so every
//                 byte of state makes exactly one HBM round trip per step.  Per-CTA stats partials
//                 are reduced by the last CTA in a fixed order (deterministic fp64 sums).
#include <cuda_runtime.h>

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
    B_PHYS = 1u << 8
};

// =====================================================================================
// Reset
// =====================================================================================
// Philox block slots per env (fixed offsets; blocks of disabled layers are skipped).
enum : int {
    SL_PHYS_U = 0,       // up to 64 blocks (256 uniform-kind params)
    SL_PHYS_N = 64,      // up to 64 blocks (256 normal-kind params)
    SL_DELAY = 128,      // 5
    SL_BACKLASH = 133,   // 10 (40 normals)
    SL_LAMBDA = 143,     // 1
    SL_FORCE_P = 144,    // 1
    SL_CORR_ACT = 145,   // 5
    SL_CORR_TIP = 150,   // 4
    SL_MARKER_TIP = 154, // 4
    SL_MARKER_BASE = 158,// 1
    SL_CORR_OBJ = 159,   // 1
    SL_CORR_ROT = 160,   // 1
    SL_COUNT = 161
};

__device__ __forceinline__ bool slot_channel(int i, uint32_t lm, uint32_t& ch, uint32_t& blk) {
    const int nbu = (c_dc.n_phys_u + 3) >> 2, nbn = (c_dc.n_phys_n + 3) >> 2;
    if (i < SL_PHYS_N) { ch = CH_PHYS_U; blk = i; return (lm & B_PHYS) && i < nbu; }
    if (i < SL_DELAY) { ch = CH_PHYS_N; blk = i - SL_PHYS_N; return (lm & B_PHYS) && (int)blk < nbn; }
    if (i < SL_BACKLASH) { ch = CH_DELAY; blk = i - SL_DELAY; return lm & B_DELAY; }
    if (i < SL_LAMBDA) { ch = CH_BACKLASH; blk = i - SL_BACKLASH; return lm & B_BACKLASH; }
    if (i < SL_FORCE_P) { ch = CH_LAMBDA; blk = 0; return lm & B_TIMING; }
    if (i < SL_CORR_ACT) { ch = CH_FORCE_P; blk = 0; return lm & B_FORCE; }
    if (i < SL_CORR_TIP) { ch = CH_CORR_ACT; blk = i - SL_CORR_ACT; return lm & B_ACT_NOISE; }
    if (i < SL_MARKER_TIP) { ch = CH_CORR_TIP; blk = i - SL_CORR_TIP; return lm & B_OBS_NOISE; }
    if (i < SL_MARKER_BASE) { ch = CH_MARKER_TIP; blk = i - SL_MARKER_TIP; return lm & B_OBS_NOISE; }
    if (i < SL_CORR_OBJ) { ch = CH_MARKER_BASE; blk = 0; return lm & B_OBS_NOISE; }
    if (i < SL_CORR_ROT) { ch = CH_CORR_OBJ; blk = 0; return lm & B_OBS_NOISE; }
    ch = CH_CORR_ROT; blk = 0; return lm & B_OBS_NOISE;
}

// normal n of the channel whose blocks start at slot `base`
__device__ __forceinline__ float slot_normal(const uint4* w, int base, int n) {
    const uint4 b = w[base + (n >> 2)];
    float z0, z1;
    if ((n & 3) < 2) box_muller(b.x, b.y, z0, z1);
    else box_muller(b.z, b.w, z0, z1);
    return (n & 1) ? z1 : z0;
}

__device__ __forceinline__ void reset_one(const DevPtrs& p, uint32_t e, bool first, int lane, uint4* w) {
    const uint32_t lm = c_dc.layer_mask;
    constexpr size_t P = PLANE;
    uint32_t* R = p.rec + rec_index(e);
    uint32_t* S = p.st + st_index(e);
    const uint32_t g = c_dc.env_offset + e;
    const uint32_t k = first ? 0u : R[REC_EPISODE * P] + 1u;
    __syncwarp();
    // 1. Philox blocks of every enabled reset channel, spread over the lanes
    for (int i = lane; i < SL_COUNT; i += 32) {
        uint32_t ch, blk;
        if (slot_channel(i, lm, ch, blk)) w[i] = philox(g, k, ch, blk);
    }
    __syncwarp();
    // 2. physical parameters (schema SPEC.md:126): one lane per parameter,
    //    coalesced row writes of phys[e][*]
    const int np = c_dc.n_phys;
    float* prow = p.phys + (size_t)e * np;
    for (int q = lane; q < np; q += 32) {
        const uint32_t kr = __ldg(p.pd_kind_rank + q);
        const uint32_t kind = kr & 0xFFu, rank = kr >> 8;
        const float base = __ldg(p.pd_base + q);
        float v = base;
        if (lm & B_PHYS) {
            const float a = __ldg(p.pd_a + q), b = __ldg(p.pd_b + q);
            if (kind == 1u || kind == 2u) {
                const float u = uni(word_of(w[SL_PHYS_U + (rank >> 2)], rank & 3));
                v = (kind == 1u) ? base * (a + b * u) : base * expf(a + b * u);
            } else if (kind == 3u || kind == 4u) {
                const float z = slot_normal(w, SL_PHYS_N, (int)rank);
                v = (kind == 3u) ? base + a * z : base * expf(a * z);
            }
        }
        prow[q] = v;
        if (q == c_dc.mass_index) R[REC_MASS * P] = __float_as_uint(v);  // object mass [Q18]
    }
    // 3. per-actuator record: delay flag, backlash widths,
    //    correlated action noise (Table action-noise)
    {
        const int j = lane;
        bool dflag = false;
        if (j < N_ACT) {
            if (lm & B_DELAY) dflag = (unsigned long long)word_of(w[SL_DELAY + (j >> 2)], j & 3) < c_dc.t_delay;
            float dn = 0.f, dp = 0.f;
            if (lm & B_BACKLASH) {
                dn = fmaxf(0.f, c_dc.dcal_neg[j] + c_dc.jitter * slot_normal(w, SL_BACKLASH, j));
                dp = fmaxf(0.f, c_dc.dcal_pos[j] + c_dc.jitter * slot_normal(w, SL_BACKLASH, N_ACT + j));
            }
            R[(REC_DNEG + j) * P] = __float_as_uint(dn);
            R[(REC_DPOS + j) * P] = __float_as_uint(dp);
            const float ca = (lm & B_ACT_NOISE) ? c_dc.sc * slot_normal(w, SL_CORR_ACT, j) : 0.f;
            R[(REC_CACT + j) * P] = __float_as_uint(ca);
        }
        const uint32_t bits = __ballot_sync(0xFFFFFFFFu, dflag);
        if (lane == 0) R[REC_DELAY * P] = bits & 0xFFFFFu;
    }
    // 4. correlated observation offsets + marker misplacement [Q14]
    if (lane < 15) {
        float v = 0.f;
        if (lm & B_OBS_NOISE) {
            const float zc = slot_normal(w, SL_CORR_TIP, lane);
            const float zm = slot_normal(w, SL_MARKER_TIP, lane);
            v = c_dc.tip_corr * zc + c_dc.tip_marker * zm;
            if (c_dc.base_to_tips) v = v - c_dc.base_marker * slot_normal(w, SL_MARKER_BASE, lane % 3);
        }
        R[(REC_OFFTIP + lane) * P] = __float_as_uint(v);
    } else if (lane < 18) {
        const int c = lane - 15;
        const float v = (lm & B_OBS_NOISE) ? c_dc.obj_corr * slot_normal(w, SL_CORR_OBJ, c) : 0.f;
        R[(REC_COBJ + c) * P] = __float_as_uint(v);
    } else if (lane == 18) {
        float q[4] = {1.f, 0.f, 0.f, 0.f};
        if (lm & B_OBS_NOISE) rotation(c_dc.rot_corr, w[SL_CORR_ROT], q);
        for (int c = 0; c < 4; ++c) R[(REC_QC + c) * P] = __float_as_uint(q[c]);
    } else if (lane == 19) {
        // timing coefficient lambda ~ U[1250, 10000]
        float lam = 0.f, il = 0.f;
        if (lm & B_TIMING) {
            lam = c_dc.lam_lo + c_dc.lam_range * uni(w[SL_LAMBDA].x);
            il = 1.0f / lam;
        }
        R[REC_LAMBDA * P] = __float_as_uint(lam);
        R[REC_INVLAM * P] = __float_as_uint(il);
    } else if (lane == 20) {
        // loguniform force probability [Q19]: index + exact integer threshold
        uint32_t j = 0, tf = 0;
        if (lm & B_FORCE) {
            j = w[SL_FORCE_P].x >> 16;
            tf = __ldg(p.t_tab + j);
        }
        R[REC_PINDEX * P] = j;
        R[REC_TFORCE * P] = tf;
    } else if (lane == 21) {
        R[REC_EPISODE * P] = k;
    }
    // 5. state: slack 0, prev 0, last 0, timers/has_last 0, force 0
    for (int q = lane; q < ST_PLANES; q += 32) S[q * P] = 0u;
    __syncwarp();
}

__global__ void __launch_bounds__(RESET_THREADS) reset_kernel(DevPtrs p, const uint8_t* __restrict__ mask,
                                                              int first, uint32_t n_env) {
    __shared__ uint4 s_w[RESET_THREADS / 32][SL_COUNT];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const uint32_t n_chunks = (n_env + 31u) >> 5;
    const uint32_t nw = gridDim.x * (RESET_THREADS / 32);
    uint32_t applied = 0;
    for (uint32_t c = blockIdx.x * (RESET_THREADS / 32) + wib; c < n_chunks; c += nw) {
        const uint32_t e = (c << 5) + lane;
        const bool m = e < n_env && (mask == nullptr || mask[e] != 0);
        uint32_t bal = __ballot_sync(0xFFFFFFFFu, m);
        applied += __popc(bal);
        while (bal) {
            const int b = __ffs(bal) - 1;
            bal &= bal - 1;
            reset_one(p, (c << 5) + b, first != 0, lane, s_w[wib]);
        }
    }
    if (!first && lane == 0 && applied) atomicAdd(&p.ctl[2], (unsigned long long)applied);
}

#include "dr_step.cuh"

// =====================================================================================
// Export / import (dr_env_state, 148 words per env)
// =====================================================================================
constexpr int EXP_WORDS = 148;

__global__ void export_kernel(DevPtrs p, uint32_t* __restrict__ dst, uint32_t lo, uint32_t hi) {
    const uint32_t e = lo + blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= hi) return;
    constexpr size_t P = PLANE;
    const uint32_t* R = p.rec + rec_index(e);
    const uint32_t* S = p.st + st_index(e);
    uint32_t* o = dst + (size_t)(e - lo) * EXP_WORDS;
    o[0] = R[REC_EPISODE * P];
    o[1] = R[REC_DELAY * P];
    o[2] = R[REC_PINDEX * P];
    o[3] = R[REC_TFORCE * P];
    o[4] = S[ST_FLAGS * P];
    o[5] = S[ST_KF * P];
    o[6] = R[REC_LAMBDA * P];
    o[7] = R[REC_MASS * P];
    for (int i = 0; i < REC_STEP_PLANES - REC_DNEG; ++i) o[8 + i] = R[(REC_DNEG + i) * P];   // 82 words
    for (int i = 0; i < ST_FLAGS; ++i) o[90 + i] = S[i * P];                                  // 55 words
    for (int i = 0; i < 3; ++i) o[145 + i] = S[(ST_FTRIG + i) * P];
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
    S[ST_FLAGS * P] = o[4];
    S[ST_KF * P] = o[5];
    R[REC_LAMBDA * P] = o[6];
    const float lam = __uint_as_float(o[6]);
    R[REC_INVLAM * P] = __float_as_uint(lam > 0.f ? 1.0f / lam : 0.f);
    R[REC_MASS * P] = o[7];
    for (int i = 0; i < REC_STEP_PLANES - REC_DNEG; ++i) R[(REC_DNEG + i) * P] = o[8 + i];
    for (int i = 0; i < ST_FLAGS; ++i) S[i * P] = o[90 + i];
    for (int i = 0; i < 3; ++i) S[(ST_FTRIG + i) * P] = o[145 + i];
}

// =====================================================================================
// launchers
// =====================================================================================
cudaError_t upload_const(const DevConst& c, cudaStream_t s) {
    return cudaMemcpyToSymbolAsync(c_dc, &c, sizeof(DevConst), 0, cudaMemcpyHostToDevice, s);
}

cudaError_t launch_reset(const DevPtrs& p, const uint8_t* mask, bool first, uint32_t n_env, int grid,
                         cudaStream_t s) {
    reset_kernel<<<grid, RESET_THREADS, 0, s>>>(p, mask, first ? 1 : 0, n_env);
    return cudaGetLastError();
}

static constexpr uint32_t MASK_FULL = 0xFFu;  // PHYS does not affect the step
static constexpr uint32_t MASK_CFG2 = B_TIMING | B_ACT_NOISE | B_BACKLASH | B_OBS_NOISE;

typedef void (*StepFn)(const DevPtrs, const float*, const float*, float*, float*, float*, float*, uint32_t);

// L2 bulk-prefetch policy of the step kernel (DR_PREFETCH=0/1/2).  Measured on B200 at 1M envs
// (profiles/round1_notes.md): 0 = none 2.48e9 env-steps/s, 1 = current tile 2.10e9,
// 2 = next tile 1.92e9 -- the batched per-phase loads already keep enough lines in flight, and
// the prefetched lines compete with the in-flight state for L2.
static int g_prefetch = 0;

void set_step_prefetch(int mode) { g_prefetch = (mode < 0 || mode > 2) ? 0 : mode; }

template <int PF>
static StepFn step_fn_pf(uint32_t m) {
    if (m == MASK_FULL) return step_kernel<MASK_FULL, PF>;
    if (m == MASK_CFG2) return step_kernel<MASK_CFG2, PF>;
    return step_kernel<RUNTIME_MASK, PF>;
}

static StepFn step_fn(uint32_t layer_mask) {
    const uint32_t m = layer_mask & 0xFFu;
    if (g_prefetch == 0) return step_fn_pf<0>(m);
    if (g_prefetch == 2) return step_fn_pf<2>(m);
    return step_fn_pf<1>(m);
}

// the phase ring is dynamic shared memory (static + dynamic > 48 KB needs the opt-in attribute)
static StepFn step_fn_ready(uint32_t layer_mask) {
    StepFn f = step_fn(layer_mask);
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)STEP_DYN_SMEM);
    return f;
}

int step_max_ctas_per_sm(uint32_t layer_mask) {
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, step_fn_ready(layer_mask), STEP_THREADS, STEP_DYN_SMEM) != cudaSuccess)
        return 1;
    return n > 0 ? n : 1;
}

int reset_max_ctas_per_sm() {
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, reset_kernel, RESET_THREADS, 0) != cudaSuccess) return 1;
    return n > 0 ? n : 1;
}

cudaError_t launch_step(const DevPtrs& p, uint32_t layer_mask, const float* actions, const float* raw_obs,
                        float* out_actions, float* out_obs, float* out_dt, float* out_force, uint32_t n_env,
                        int grid, cudaStream_t s) {
    step_fn(layer_mask)<<<grid, STEP_THREADS, STEP_DYN_SMEM, s>>>(p, actions, raw_obs, out_actions, out_obs, out_dt,
                                                      out_force, n_env);
    return cudaGetLastError();
}

__global__ void debug_philox_kernel(uint32_t n_env, uint32_t dom, uint32_t ch, uint32_t blk, uint4* __restrict__ out) {
    const uint32_t e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e < n_env) out[e] = philox(c_dc.env_offset + e, dom, ch, blk);
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
