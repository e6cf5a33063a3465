// dr_reset.cuh -- episode-reset sampling (PAPER.md:7-8, 13, 15-18, 36-41, 77-78, 87-88, 100-101,
// 113), included by dr_kernels.cu inside namespace dr.
//
// A warp ballots 32 mask bytes, then serves each resetting env with all 32 lanes in four
// warp-uniform phases driven by host-built task tables (dr_internal.h), so no lane runs a
// different transcendental code path:
//   A. the Philox blocks of every enabled reset channel, one block per lane, into shared memory;
//   B. every Box-Muller pair the episode needs (physics normals + record normals), one pair per
//      lane, into a per-warp z buffer;
//   C. the n_phys physical parameters, one lane per parameter: v = C0 + C1 * f(A + B x) with
//      x a uniform or a normal and f = exp or identity by descriptor -- written as coalesced
//      128-byte lines of the row phys[e][*];
//   D. the episode record fields (cheap arithmetic on the staged draws), one lane per field.
// The 60 state planes are not zeroed here: one word (FRESH_BIT in the flags plane) marks the env
// and the step kernel reads a fresh env's state as zero (dr_internal.h).
#pragma once

__device__ __forceinline__ void reset_one(const DevPtrs& p, uint32_t e, uint32_t k, int lane, uint4* w, float* zb,
                                          const uint32_t* s_ph, const uint32_t* s_pr, const float4* s_pd,
                                          const uint32_t* s_src) {
    const uint32_t lm = c_dc.layer_mask;
    constexpr size_t P = PLANE;
    uint32_t* R = p.rec + rec_index(e);
    uint32_t* S = p.st + st_index(e);
    const uint32_t g = c_dc.env_offset + e;
    __syncwarp();
    // A. Philox blocks, one per lane (k = this env's new episode index, loaded per chunk)
    for (int i = lane; i < c_dc.n_rs_philox; i += 32) {
        const uint32_t task = s_ph[i];
        w[task & 0xFFu] = philox(g, k, task >> 16, (task >> 8) & 0xFFu);
    }
    __syncwarp();
    // the force threshold gather is issued now and consumed in D2 (latency off the critical path)
    const uint32_t tf_pre = (lane == 20 && (lm & B_FORCE)) ? __ldg(p.t_tab + (w[SL_FORCE_P].x >> 16)) : 0u;
    // B. Box-Muller pairs, one per lane: pair q of a channel uses block q / 2, words (x, y) for
    //    even q and (z, w) for odd q, giving normals 2q (cos) and 2q + 1 (sin)
    for (int i = lane; i < c_dc.n_rs_pairs; i += 32) {
        const uint32_t task = s_pr[i];
        const uint32_t q = (task >> 8) & 0xFFu, base = task >> 16;
        const uint4 b = w[(task & 0xFFu) + (q >> 1)];
        float z0, z1;
        box_muller((q & 1u) ? b.z : b.x, (q & 1u) ? b.w : b.y, z0, z1);
        zb[base + 2 * q] = z0;
        zb[base + 2 * q + 1] = z1;
    }
    __syncwarp();
    // C. physical parameters (descriptor schema SPEC.md:126) [Q20]
    const int np = c_dc.n_phys;
    float* prow = p.phys + (size_t)e * np;
    const uint32_t* w32 = reinterpret_cast<const uint32_t*>(w);
    for (int q = lane; q < np; q += 32) {
        const float4 d = s_pd[q];   // (A, B, C0, C1)
        const uint32_t src = s_src[q];
        // (with PHYS off, or a FIXED descriptor, the host table is A = B = C1 = 0, C0 = base)
        const uint32_t idx = src & RS_SRC_IDX;
        const float x = (src & RS_SRC_NORMAL) ? zb[idx] : uni(w32[idx]);
        const float tv = fmaf(d.y, x, d.x);
        const float v = fmaf(d.w, (src & RS_SRC_EXP) ? expf(tv) : tv, d.z);
        prow[q] = v;
        if (q == c_dc.mass_index) R[REC_MASS * P] = __float_as_uint(v);   // the object mass [Q18]
    }
    // D1. per actuator: delay flag, backlash widths [Q7],
    //     correlated action noise (Table action-noise)
    {
        const int j = lane;
        bool dflag = false;
        if (j < N_ACT) {
            if (lm & B_DELAY) dflag = (unsigned long long)w32[SL_DELAY * 4 + j] < c_dc.t_delay;
            float dn = 0.f, dp = 0.f, ca = 0.f;
            if (lm & B_BACKLASH) {
                dn = fmaxf(0.f, c_dc.dcal_neg[j] + c_dc.jitter * zb[ZB_BL + j]);
                dp = fmaxf(0.f, c_dc.dcal_pos[j] + c_dc.jitter * zb[ZB_BL + N_ACT + j]);
            }
            if (lm & B_ACT_NOISE) ca = c_dc.sc * zb[ZB_CA + j];
            R[(REC_DNEG + j) * P] = __float_as_uint(dn);
            R[(REC_DPOS + j) * P] = __float_as_uint(dp);
            R[(REC_CACT + j) * P] = __float_as_uint(ca);
        }
        const uint32_t bits = __ballot_sync(0xFFFFFFFFu, dflag);
        if (lane == 0) R[REC_DELAY * P] = bits & 0xFFFFFu;
    }
    // D2. observation offsets [Q14, Q15], timing, force, episode, state
    if (lane < 15) {
        float v = 0.f;
        if (lm & B_OBS_NOISE) {
            v = c_dc.tip_corr * zb[ZB_CT + lane] + c_dc.tip_marker * zb[ZB_MT + lane];
            if (c_dc.base_to_tips) v = v - c_dc.base_marker * zb[ZB_MB + lane % 3];
        }
        R[(REC_OFFTIP + lane) * P] = __float_as_uint(v);
    } else if (lane < 18) {
        const int c = lane - 15;
        R[(REC_COBJ + c) * P] = __float_as_uint((lm & B_OBS_NOISE) ? c_dc.obj_corr * zb[ZB_CO + c] : 0.f);
    } else if (lane == 18) {
        float q[4] = {1.f, 0.f, 0.f, 0.f};
        if (lm & B_OBS_NOISE) rotation(c_dc.rot_corr, w[SL_CORR_ROT], q);
#pragma unroll
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
        const uint32_t j = (lm & B_FORCE) ? (w[SL_FORCE_P].x >> 16) : 0u;
        R[REC_PINDEX * P] = j;
        R[REC_TFORCE * P] = tf_pre;
    } else if (lane == 21) {
        R[REC_EPISODE * P] = k;
    } else if (lane == 22) {
        S[ST_FLAGS * P] = FRESH_BIT;   // state reads as zero at the next step [Q6, Q9]
    }
    __syncwarp();
}

constexpr int RESET_WARPS = RESET_THREADS / 32;

__global__ void __launch_bounds__(RESET_THREADS) reset_kernel(DevPtrs p, const uint8_t* __restrict__ mask,
                                                              int first, uint32_t n_env) {
    __shared__ uint4 s_w[RESET_WARPS][SL_COUNT];
    __shared__ float s_zb[RESET_WARPS][ZB_COUNT];
    __shared__ float4 s_pd[MAX_PHYS];
    __shared__ uint32_t s_src[MAX_PHYS];
    __shared__ uint32_t s_ph[RS_MAX_PHILOX];
    __shared__ uint32_t s_pr[RS_MAX_PAIRS];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < c_dc.n_phys; i += RESET_THREADS) {
        s_pd[i] = p.rs_phys[i];
        s_src[i] = p.rs_src[i];
    }
    for (int i = threadIdx.x; i < c_dc.n_rs_philox; i += RESET_THREADS) s_ph[i] = p.rs_philox[i];
    for (int i = threadIdx.x; i < c_dc.n_rs_pairs; i += RESET_THREADS) s_pr[i] = p.rs_pairs[i];
    __syncthreads();
    const uint32_t n_chunks = (n_env + 31u) >> 5;
    const uint32_t nw = gridDim.x * RESET_WARPS;
    uint32_t applied = 0;
    // one coalesced load of 32 mask bytes and 32 episode counters per chunk, prefetched a chunk ahead
    auto load_chunk = [&](uint32_t c, uint32_t& m, uint32_t& ep) {
        const uint32_t e = (c << 5) + lane;
        m = 0u;
        ep = 0u;
        if (c < n_chunks && e < n_env) {
            m = (mask == nullptr) ? 1u : (uint32_t)mask[e];
            if (!first) ep = p.rec[rec_index(e) + REC_EPISODE * PLANE];
        }
    };
    uint32_t c = blockIdx.x * RESET_WARPS + wib;
    uint32_t m_cur, ep_cur;
    load_chunk(c, m_cur, ep_cur);
    for (; c < n_chunks; c += nw) {
        uint32_t m_nxt, ep_nxt;
        load_chunk(c + nw, m_nxt, ep_nxt);
        uint32_t bal = __ballot_sync(0xFFFFFFFFu, m_cur != 0u);
        applied += __popc(bal);
        while (bal) {
            const int b = __ffs(bal) - 1;
            bal &= bal - 1;
            const uint32_t k = first ? 0u : __shfl_sync(0xFFFFFFFFu, ep_cur, b) + 1u;
            reset_one(p, (c << 5) + b, k, lane, s_w[wib], s_zb[wib], s_ph, s_pr, s_pd, s_src);
        }
        m_cur = m_nxt;
        ep_cur = ep_nxt;
    }
    if (!first && lane == 0 && applied) atomicAdd(&p.ctl[2], (unsigned long long)applied);
}
