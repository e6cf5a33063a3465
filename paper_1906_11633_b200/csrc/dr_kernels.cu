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
    const size_t P = c_dc.pitch;
    uint32_t* R = p.rec + e;
    uint32_t* S = p.st + e;
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

// =====================================================================================
// Step
// =====================================================================================
struct Acc {
    uint32_t n[12];
    double m[8];
};

template <uint32_t L>
__device__ __forceinline__ void env_step(const DevPtrs& p, uint32_t e, uint32_t t, int tid,
                                         float* s_act, const float* s_obs, float* s_oobs, float* s_dt,
                                         float* s_frc, const double* s_dec, Acc& acc) {
    const size_t P = c_dc.pitch;
    const uint32_t* __restrict__ R = p.rec + e;
    uint32_t* __restrict__ S = p.st + e;
    const uint32_t g = c_dc.env_offset + e;
    acc.n[0] += 1;

    // ---- 1. timing: 10 substeps of 8 ms + Exp(lambda); dt_env = sum [Q2] ----
    float dt_env;
    {
        float dts[N_SUB];
        if (on<L>(B_TIMING)) {
            const float il = __uint_as_float(R[REC_INVLAM * P]);
#pragma unroll
            for (int b = 0; b < 3; ++b) {
                const uint4 w = philox(g, t, CH_TIMING, b);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int k = 4 * b + q;
                    if (k < N_SUB) dts[k] = c_dc.dt_base + (-logf(uni(word_of(w, q)))) * il;
                }
            }
        } else {
#pragma unroll
            for (int k = 0; k < N_SUB; ++k) dts[k] = c_dc.dt_base;
        }
        dt_env = dts[0];
#pragma unroll
        for (int k = 1; k < N_SUB; ++k) dt_env = dt_env + dts[k];
        float2* d2 = reinterpret_cast<float2*>(s_dt + tid * N_SUB);
#pragma unroll
        for (int k = 0; k < N_SUB / 2; ++k) d2[k] = make_float2(dts[2 * k], dts[2 * k + 1]);
        acc.m[0] += (double)dt_env;
        acc.m[1] += (double)dt_env * (double)dt_env;
    }

    // ---- 2-4. actions: delay -> noise -> clamp -> backlash [Q1] ----
    {
        const uint32_t dbits = on<L>(B_DELAY) ? R[REC_DELAY * P] : 0u;
        acc.n[1] += __popc(dbits);
        float s_da = 0.f, s_da2 = 0.f, s_bl = 0.f, s_zu2 = 0.f;
        float4* a4p = reinterpret_cast<float4*>(s_act + tid * N_ACT);
#pragma unroll
        for (int b = 0; b < 5; ++b) {
            float zu[4], zm[4];
            if (on<L>(B_ACT_NOISE)) {
                normals4(philox(g, t, CH_ACT_UADD, b), zu);
                normals4(philox(g, t, CH_ACT_MULT, b), zm);
            }
            const float4 a4 = a4p[b];
            const float av[4] = {a4.x, a4.y, a4.z, a4.w};
            float ov[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int j = 4 * b + q;
                const float a = av[q];
                float ad = a;
                if (on<L>(B_DELAY)) {
                    // one-step delay of flagged actuators [Q9]
                    const float pv = __uint_as_float(S[(ST_PREV + j) * P]);
                    if ((dbits >> j) & 1u) ad = pv;
                    S[(ST_PREV + j) * P] = __float_as_uint(a);
                }
                float an = ad;
                if (on<L>(B_ACT_NOISE)) {
                    // Table action-noise [Q8]
                    an = ad + ad * (c_dc.sm * zm[q]);
                    an = an + c_dc.su * zu[q];
                    an = an + __uint_as_float(R[(REC_CACT + j) * P]);
                    acc.n[11] += (an > 1.f || an < -1.f) ? 1u : 0u;
                    an = fminf(fmaxf(an, -1.f), 1.f);
                    s_zu2 += zu[q] * zu[q];
                }
                const float da = an - ad;
                s_da += da;
                s_da2 += da * da;
                float out = an;
                if (on<L>(B_BACKLASH)) {
                    // backlash, verbatim [Q4], sgn(0) = 0 [Q3]
                    const float s = __uint_as_float(S[(ST_SLACK + j) * P]);
                    const float sg = (an > 0.f) ? 1.f : ((an < 0.f) ? -1.f : 0.f);
                    const float d = (an > 0.f) ? __uint_as_float(R[(REC_DPOS + j) * P])
                                  : ((an < 0.f) ? __uint_as_float(R[(REC_DNEG + j) * P]) : 0.f);
                    const float sp = fminf(fmaxf(s + an * d * dt_env, -1.f), 1.f);
                    const float ratio = fminf(fmaxf(fabsf(sg - s) / (fabsf(sp - s) + c_dc.eps), 0.f), 1.f);
                    const float al = 1.f - ratio;
                    out = al * an;
                    acc.n[7] += (sg != 0.f && fabsf(sp) == 1.f && sp != s) ? 1u : 0u;
                    acc.n[8] += (al == 1.f) ? 1u : 0u;
                    acc.n[9] += (al == 1.f) ? 0u : 1u;
                    S[(ST_SLACK + j) * P] = __float_as_uint(sp);
                }
                s_bl += fabsf(out - an);
                ov[q] = out;
            }
            a4p[b] = make_float4(ov[0], ov[1], ov[2], ov[3]);
        }
        acc.m[2] += (double)s_da;
        acc.m[3] += (double)s_da2;
        acc.m[4] += (double)s_bl;
        acc.m[5] += (double)s_zu2;
    }

    // ---- 5-8. fingertip markers and object position ----
    const float* ro = s_obs + tid * OBS_IN;
    float* oo = s_oobs + tid * OBS_OUT;
    {
        float tip[15];
#pragma unroll
        for (int c = 0; c < 15; ++c) tip[c] = ro[c];
        float obj[3] = {ro[15], ro[16], ro[17]};
        constexpr bool kHoldPossible = true;
        const bool hold_layers = on<L>(B_DROPOUT) || on<L>(B_OCCLUSION);
        uint32_t occ = 0;
        if (on<L>(B_OCCLUSION) && c_dc.occl_on) {
            // occlusion: another tip or the object centre strictly closer than r
            // [Q13], exactly rounded fp64, ((dx*dx + dy*dy) + dz*dz), no FMA contraction
            const double r2 = c_dc.occl_r2;
#pragma unroll
            for (int i = 0; i < N_TIPS; ++i) {
#pragma unroll
                for (int j = i + 1; j < N_TIPS; ++j) {
                    const double dx = __dsub_rn((double)tip[3 * i], (double)tip[3 * j]);
                    const double dy = __dsub_rn((double)tip[3 * i + 1], (double)tip[3 * j + 1]);
                    const double dz = __dsub_rn((double)tip[3 * i + 2], (double)tip[3 * j + 2]);
                    const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
                    if (d2 < r2) occ |= (1u << i) | (1u << j);
                }
                const double dx = __dsub_rn((double)tip[3 * i], (double)obj[0]);
                const double dy = __dsub_rn((double)tip[3 * i + 1], (double)obj[1]);
                const double dz = __dsub_rn((double)tip[3 * i + 2], (double)obj[2]);
                const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
                if (d2 < r2) occ |= (1u << i);
            }
            acc.n[4] += __popc(occ);
        }
        uint32_t masked = 0, flags = 0, nflags = 0;
        if (hold_layers) {
            flags = S[ST_FLAGS * P];
            if (on<L>(B_DROPOUT)) {
                // dropout: start a 13-step mask with probability 1 - exp(-0.2 * 0.08) per step,
                // retrigger restarts it [Q11]
                const uint4 w0 = philox(g, t, CH_DROPOUT, 0);
                const uint4 w1 = philox(g, t, CH_DROPOUT, 1);
#pragma unroll
                for (int i = 0; i < N_TIPS; ++i) {
                    const uint32_t x = (i < 4) ? word_of(w0, i) : w1.x;
                    uint32_t tm = (flags >> (4 * i)) & 0xFu;
                    if ((unsigned long long)x < c_dc.t_drop) { tm = c_dc.hold_steps; acc.n[2] += 1; }
                    if (tm > 0u) { masked |= 1u << i; tm -= 1u; }
                    nflags |= tm << (4 * i);
                }
                acc.n[3] += __popc(masked);
            }
            nflags |= HAS_LAST_BIT;
            S[ST_FLAGS * P] = nflags;
        }
        const uint32_t hold = ((flags & HAS_LAST_BIT) ? (masked | occ) : 0u);
        acc.n[5] += __popc(hold);
        (void)kHoldPossible;
        // fingertip noise: + (correlated + misplacement offset) + 2 mm uncorrelated; held tips
        // return their last available reading [Q12]
        float s_zt = 0.f;
        if (on<L>(B_OBS_NOISE)) {
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                float z[4];
                normals4(philox(g, t, CH_TIP_NOISE, b), z);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int n = 4 * b + q;
                    if (n < 15) {
                        tip[n] = (tip[n] + __uint_as_float(R[(REC_OFFTIP + n) * P])) + c_dc.tip_uncorr * z[q];
                        s_zt += z[q] * z[q];
                    }
                }
            }
        }
        acc.m[6] += (double)s_zt;
#pragma unroll
        for (int i = 0; i < N_TIPS; ++i) {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                float v = tip[3 * i + c];
                if (hold_layers) {
                    if ((hold >> i) & 1u) v = __uint_as_float(S[(ST_LAST + 3 * i + c) * P]);
                    S[(ST_LAST + 3 * i + c) * P] = __float_as_uint(v);
                }
                oo[4 + 3 * i + c] = v;
            }
        }
        // object position: + 5 mm correlated + 1 mm uncorrelated
        if (on<L>(B_OBS_NOISE)) {
            float z[4];
            normals4(philox(g, t, CH_OBJ_NOISE, 0), z);
#pragma unroll
            for (int c = 0; c < 3; ++c)
                obj[c] = (obj[c] + __uint_as_float(R[(REC_COBJ + c) * P])) + c_dc.obj_uncorr * z[c];
        }
        oo[19] = obj[0];
        oo[20] = obj[1];
        oo[21] = obj[2];
    }

    // ---- 9. orientation noise -> noisy relative goal [Q15, Q16] ----
    {
        float qo[4] = {ro[18], ro[19], ro[20], ro[21]};
        const float goal[4] = {ro[22], ro[23], ro[24], ro[25]};
        float qn[4];
        if (on<L>(B_OBS_NOISE)) {
            float qu[4], qc[4], tmp[4];
            rotation(c_dc.rot_uncorr, philox(g, t, CH_ROT_NOISE, 0), qu);
#pragma unroll
            for (int c = 0; c < 4; ++c) qc[c] = __uint_as_float(R[(REC_QC + c) * P]);
            qmul(qc, qo, tmp);
            qmul(qu, tmp, qn);
        } else {
#pragma unroll
            for (int c = 0; c < 4; ++c) qn[c] = qo[c];
        }
        const float cj[4] = {qn[0], -qn[1], -qn[2], -qn[3]};
        float rel[4];
        qmul(goal, cj, rel);
        const float sgn = (rel[0] < 0.f) ? -1.f : 1.f;
#pragma unroll
        for (int c = 0; c < 4; ++c) oo[c] = sgn * rel[c];
    }

    // ---- 10. random force: replace on trigger, decay 0.99 per step in closed form
    //           [Q17, Q18] ----
    {
        float f[3] = {0.f, 0.f, 0.f};
        if (on<L>(B_FORCE)) {
            const uint32_t x = philox(g, t, CH_FORCE, 0).x;
            const uint32_t tf = R[REC_TFORCE * P];
            uint32_t kf = S[ST_KF * P];
            float ft[3];
            if (x < tf) {
                const uint4 w = philox(g, t, CH_FORCE, 1);
                float z0, z1, z2, z3;
                box_muller(w.x, w.y, z0, z1);
                box_muller(w.z, w.w, z2, z3);
                const float ms = __uint_as_float(R[REC_MASS * P]) * c_dc.accel_std;
                ft[0] = ms * z0;
                ft[1] = ms * z1;
                ft[2] = ms * z2;
#pragma unroll
                for (int c = 0; c < 3; ++c) S[(ST_FTRIG + c) * P] = __float_as_uint(ft[c]);
                kf = 0;
                acc.n[6] += 1;
            } else {
#pragma unroll
                for (int c = 0; c < 3; ++c) ft[c] = __uint_as_float(S[(ST_FTRIG + c) * P]);
                kf = (kf < 65535u) ? kf + 1u : 65535u;
            }
            S[ST_KF * P] = kf;
            const double dec = s_dec[kf & 255u] * s_dec[256u + (kf >> 8)];
#pragma unroll
            for (int c = 0; c < 3; ++c) f[c] = (float)((double)ft[c] * dec);
        }
        s_frc[tid * 3 + 0] = f[0];
        s_frc[tid * 3 + 1] = f[1];
        s_frc[tid * 3 + 2] = f[2];
        acc.m[7] += (double)f[0] * f[0] + (double)f[1] * f[1] + (double)f[2] * f[2];
    }
}

// copy `n` floats global->shared (src/dst 16-B aligned when vec)
__device__ __forceinline__ void tile_load(float* dst, const float* __restrict__ src, uint32_t n, bool vec) {
    if (vec) {
        const float4* s4 = reinterpret_cast<const float4*>(src);
        float4* d4 = reinterpret_cast<float4*>(dst);
        for (uint32_t i = threadIdx.x; i < n / 4; i += blockDim.x) d4[i] = __ldcs(s4 + i);
    } else {
        for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) dst[i] = __ldcs(src + i);
    }
}
__device__ __forceinline__ void tile_store(float* dst, const float* src, uint32_t n, bool vec) {
    if (vec) {
        const float4* s4 = reinterpret_cast<const float4*>(src);
        float4* d4 = reinterpret_cast<float4*>(dst);
        for (uint32_t i = threadIdx.x; i < n / 4; i += blockDim.x) __stcs(d4 + i, s4[i]);
    } else {
        for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) __stcs(dst + i, src[i]);
    }
}

template <uint32_t L>
__global__ void __launch_bounds__(STEP_THREADS) step_kernel(const DevPtrs p, const float* __restrict__ actions,
                                                            const float* __restrict__ raw_obs,
                                                            float* __restrict__ out_actions,
                                                            float* __restrict__ out_obs,
                                                            float* __restrict__ out_dt,
                                                            float* __restrict__ out_force, uint32_t n_env) {
    __shared__ __align__(16) float s_act[TILE * N_ACT];
    __shared__ __align__(16) float s_obs[TILE * OBS_IN];
    __shared__ __align__(16) float s_oobs[TILE * OBS_OUT];
    __shared__ __align__(16) float s_dt[TILE * N_SUB];
    __shared__ __align__(16) float s_frc[TILE * 3];
    __shared__ double s_dec[512];
    __shared__ double s_red[STEP_THREADS / 32][N_STATS];
    __shared__ int s_last;

    const int tid = threadIdx.x;
    const uint32_t t = (uint32_t)p.ctl[0];
    if (on<L>(B_FORCE))
        for (int i = tid; i < 512; i += STEP_THREADS) s_dec[i] = p.dec_tab[i];

    Acc acc;
#pragma unroll
    for (int i = 0; i < 12; ++i) acc.n[i] = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) acc.m[i] = 0.0;

    const uint32_t n_tiles = (n_env + TILE - 1) / TILE;
    for (uint32_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const uint32_t e0 = tile * TILE;
        const uint32_t cnt = min((uint32_t)TILE, n_env - e0);
        const bool full = cnt == (uint32_t)TILE;
        __syncthreads();
        tile_load(s_act, actions + (size_t)e0 * N_ACT, cnt * N_ACT, full);
        tile_load(s_obs, raw_obs + (size_t)e0 * OBS_IN, cnt * OBS_IN, full);
        __syncthreads();
        if ((uint32_t)tid < cnt) env_step<L>(p, e0 + tid, t, tid, s_act, s_obs, s_oobs, s_dt, s_frc, s_dec, acc);
        __syncthreads();
        tile_store(out_actions + (size_t)e0 * N_ACT, s_act, cnt * N_ACT, full);
        tile_store(out_obs + (size_t)e0 * OBS_OUT, s_oobs, cnt * OBS_OUT, full);
        tile_store(out_dt + (size_t)e0 * N_SUB, s_dt, cnt * N_SUB, full);
        tile_store(out_force + (size_t)e0 * 3, s_frc, cnt * 3, full);
    }

    // ---- 12. stats: warp shuffle -> per-CTA partial -> last CTA reduces in a fixed order ----
    const int lane = tid & 31, wid = tid >> 5;
    double v[N_STATS];
#pragma unroll
    for (int i = 0; i < N_STATS; ++i) v[i] = 0.0;
#pragma unroll
    for (int i = 0; i < 12; ++i) v[i] = (double)acc.n[i];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[16 + i] = acc.m[i];
#pragma unroll
    for (int i = 0; i < 24; ++i) {
        if (i >= 12 && i < 16) continue;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[i] += __shfl_xor_sync(0xFFFFFFFFu, v[i], o);
    }
    if (lane == 0) {
#pragma unroll
        for (int i = 0; i < N_STATS; ++i) s_red[wid][i] = v[i];
    }
    __syncthreads();
    if (tid < N_STATS) {
        double sum = 0.0;
#pragma unroll
        for (int w = 0; w < STEP_THREADS / 32; ++w) sum += s_red[w][tid];
        p.partials[(size_t)blockIdx.x * N_STATS + tid] = sum;
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) {
        const unsigned long long prev = atomicAdd(&p.ctl[1], 1ull);
        s_last = (prev == (unsigned long long)gridDim.x - 1ull);
    }
    __syncthreads();
    if (s_last) {
        __threadfence();
        const uint32_t slot = t & 1u;
        for (int s = wid; s < N_STATS; s += STEP_THREADS / 32) {
            double sum = 0.0;
            for (uint32_t b = lane; b < gridDim.x; b += 32) sum += __ldcg(p.partials + (size_t)b * N_STATS + s);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xFFFFFFFFu, sum, o);
            if (lane == 0) p.stats[slot * N_STATS + s] = sum;
        }
        __syncthreads();
        if (tid == 0) {
            const unsigned long long res = atomicExch(&p.ctl[2], 0ull);
            p.stats[slot * N_STATS + 10] = (double)res;
            p.ctl[1] = 0ull;
            p.ctl[0] = (unsigned long long)t + 1ull;
            __threadfence();
        }
    }
}

// =====================================================================================
// Export / import (dr_env_state, 148 words per env)
// =====================================================================================
constexpr int EXP_WORDS = 148;

__global__ void export_kernel(DevPtrs p, uint32_t* __restrict__ dst, uint32_t lo, uint32_t hi) {
    const uint32_t e = lo + blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= hi) return;
    const size_t P = c_dc.pitch;
    const uint32_t* R = p.rec + e;
    const uint32_t* S = p.st + e;
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
    const size_t P = c_dc.pitch;
    uint32_t* R = p.rec + e;
    uint32_t* S = p.st + e;
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

static StepFn step_fn(uint32_t layer_mask) {
    const uint32_t m = layer_mask & 0xFFu;
    if (m == MASK_FULL) return step_kernel<MASK_FULL>;
    if (m == MASK_CFG2) return step_kernel<MASK_CFG2>;
    return step_kernel<RUNTIME_MASK>;
}

int step_max_ctas_per_sm(uint32_t layer_mask) {
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, step_fn(layer_mask), STEP_THREADS, 0) != cudaSuccess) return 1;
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
    step_fn(layer_mask)<<<grid, STEP_THREADS, 0, s>>>(p, actions, raw_obs, out_actions, out_obs, out_dt,
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
