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
// reset_kernel_t (the default) instead compacts the resetting envs of a 2,048-env
// range into a shared-memory list and runs one thread per resetting env over that list: every
// lane does useful work whatever the mask density, with the same draws and arithmetic.
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
        // exp kinds carry log2(e) in A and B (host table), so the exponential is one MUFU.EX2
        // (relative error ~2^-22, inside the 1e-6 budget of the |base| floor)
        const float tv = fmaf(d.y, x, d.x);
        const float v = fmaf(d.w, (src & RS_SRC_EXP) ? ex2_approx(tv) : tv, d.z);
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
    pdl_wait();   // before any global access (dr_device.cuh)
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
    pdl_trigger();
    if (!first && lane == 0 && applied) atomicAdd(&p.ctl[2], (unsigned long long)applied);
}

// =====================================================================================
// Thread-per-resetting-env reset (default): per-CTA compaction of the mask, then one thread per
// env runs the whole episode draw -- physics parameters streamed in descriptor order (a Philox
// block is drawn when the first parameter of its 4-word group comes up; all lanes are at the same
// parameter, so the branches are warp-uniform), then the record fields.  Same channels, words and
// transforms as reset_one / the oracle.
// =====================================================================================
constexpr int RT_THREADS = 256;
constexpr uint32_t RT_RANGE = 2048;   // envs scanned per CTA pass (~205 resetting at 10 %)

__device__ __forceinline__ float sel4(const float z[4], uint32_t r) {
    return r == 0u ? z[0] : (r == 1u ? z[1] : (r == 2u ? z[2] : z[3]));
}
__device__ __forceinline__ uint32_t selw(const uint4 w, uint32_t r) {
    return r == 0u ? w.x : (r == 1u ? w.y : (r == 2u ? w.z : w.w));
}

// kPhys = false: the record part only (reset_kernel_h writes the physics rows warp-cooperatively).
template <bool kPhys = true>
__device__ void reset_env_thread(const DevPtrs& p, uint32_t e, uint32_t k, const float4* s_pd,
                                 const uint32_t* s_src) {
    const uint32_t lm = c_dc.layer_mask;
    constexpr size_t P = PLANE;
    uint32_t* R = p.rec + rec_index(e);
    uint32_t* S = p.st + st_index(e);
    const uint32_t g = c_dc.env_offset + e;
    // ---- physics [Q20]: v = C0 + C1 f(A + B x) ----
    if constexpr (kPhys) {
        const int np = c_dc.n_phys;
        float* prow = p.phys + (size_t)e * np;
        const bool vec = (np & 3) == 0;   // rows are 16-byte aligned: float4 stores
        uint4 wu = make_uint4(0u, 0u, 0u, 0u);
        float zn[4] = {0.f, 0.f, 0.f, 0.f};
        for (int q0 = 0; q0 < np; q0 += 4) {
            float v4[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int q = q0 + r;
                float v = 0.f;
                if (q < np) {
                    const float4 d = s_pd[q];
                    const uint32_t src = s_src[q];
                    float x = 0.f;
                    if (src & RS_SRC_DRAW) {   // warp-uniform: every lane is at parameter q
                        if (src & RS_SRC_NORMAL) {
                            const uint32_t n = (src & RS_SRC_IDX) - ZB_PHYS;
                            if ((n & 3u) == 0u) {
                                const uint4 w = philox(g, k, CH_PHYS_N, n >> 2);
                                box_muller(w.x, w.y, zn[0], zn[1]);
                                box_muller(w.z, w.w, zn[2], zn[3]);
                            }
                            x = sel4(zn, n & 3u);
                        } else {
                            const uint32_t u = (src & RS_SRC_IDX) - SL_PHYS_U * 4;
                            if ((u & 3u) == 0u) wu = philox(g, k, CH_PHYS_U, u >> 2);
                            x = uni(selw(wu, u & 3u));
                        }
                    }
                    const float tv = fmaf(d.y, x, d.x);
                    v = fmaf(d.w, (src & RS_SRC_EXP) ? ex2_approx(tv) : tv, d.z);
                    if (q == c_dc.mass_index) R[REC_MASS * P] = __float_as_uint(v);   // the object mass [Q18]
                    if (!vec) prow[q] = v;
                }
                v4[r] = v;
            }
            if (vec) reinterpret_cast<float4*>(prow)[q0 >> 2] = make_float4(v4[0], v4[1], v4[2], v4[3]);
        }
    }
    // ---- delay flags ----
    uint32_t bits = 0u;
    if (lm & B_DELAY) {
#pragma unroll
        for (int b = 0; b < 5; ++b) {
            const uint4 w = philox(g, k, CH_DELAY, b);
            const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) bits |= ((unsigned long long)ws[q] < c_dc.t_delay ? 1u : 0u) << (4 * b + q);
        }
    }
    R[REC_DELAY * P] = bits;
    // ---- backlash widths [Q7]: normal j -> delta-1_j, 20 + j -> delta+1_j ----
#pragma unroll 1
    for (int b = 0; b < 10; ++b) {
        float z[4] = {0.f, 0.f, 0.f, 0.f};
        if (lm & B_BACKLASH) {
            const uint4 w = philox(g, k, CH_BACKLASH, b);
            box_muller(w.x, w.y, z[0], z[1]);
            box_muller(w.z, w.w, z[2], z[3]);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int n = 4 * b + q;
            const int j = n < N_ACT ? n : n - N_ACT;
            const float cal = n < N_ACT ? c_dc.dcal_neg[j] : c_dc.dcal_pos[j];
            const float dv = (lm & B_BACKLASH) ? fmaxf(0.f, cal + c_dc.jitter * z[q]) : 0.f;
            R[((n < N_ACT ? REC_DNEG : REC_DPOS) + j) * P] = __float_as_uint(dv);
        }
    }
    // ---- correlated action offset (Table action-noise) ----
#pragma unroll 1
    for (int b = 0; b < 5; ++b) {
        float z[4] = {0.f, 0.f, 0.f, 0.f};
        if (lm & B_ACT_NOISE) {
            const uint4 w = philox(g, k, CH_CORR_ACT, b);
            box_muller(w.x, w.y, z[0], z[1]);
            box_muller(w.z, w.w, z[2], z[3]);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) R[(REC_CACT + 4 * b + q) * P] = __float_as_uint(c_dc.sc * z[q]);
    }
    // ---- observation offsets [Q14, Q15] ----
    if (lm & B_OBS_NOISE) {
        float mb[4];
        {
            const uint4 w = philox(g, k, CH_MARKER_BASE, 0);
            box_muller(w.x, w.y, mb[0], mb[1]);
            box_muller(w.z, w.w, mb[2], mb[3]);
        }
#pragma unroll 1
        for (int b = 0; b < 4; ++b) {
            float zc[4], zm[4];
            const uint4 wc = philox(g, k, CH_CORR_TIP, b);
            const uint4 wm = philox(g, k, CH_MARKER_TIP, b);
            box_muller(wc.x, wc.y, zc[0], zc[1]);
            box_muller(wc.z, wc.w, zc[2], zc[3]);
            box_muller(wm.x, wm.y, zm[0], zm[1]);
            box_muller(wm.z, wm.w, zm[2], zm[3]);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int n = 4 * b + q;
                if (n < 15) {
                    float v = c_dc.tip_corr * zc[q] + c_dc.tip_marker * zm[q];
                    if (c_dc.base_to_tips) v = v - c_dc.base_marker * sel4(mb, (uint32_t)(n % 3));
                    R[(REC_OFFTIP + n) * P] = __float_as_uint(v);
                }
            }
        }
        float zo[4];
        const uint4 wo = philox(g, k, CH_CORR_OBJ, 0);
        box_muller(wo.x, wo.y, zo[0], zo[1]);
        box_muller(wo.z, wo.w, zo[2], zo[3]);
#pragma unroll
        for (int c = 0; c < 3; ++c) R[(REC_COBJ + c) * P] = __float_as_uint(c_dc.obj_corr * zo[c]);
        float q[4];
        rotation(c_dc.rot_corr, philox(g, k, CH_CORR_ROT, 0), q);
#pragma unroll
        for (int c = 0; c < 4; ++c) R[(REC_QC + c) * P] = __float_as_uint(q[c]);
    } else {
#pragma unroll
        for (int n = 0; n < 18; ++n) R[(REC_OFFTIP + n) * P] = 0u;   // tips 15 + object 3
        const float q[4] = {1.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int c = 0; c < 4; ++c) R[(REC_QC + c) * P] = __float_as_uint(q[c]);
    }
    // ---- timing coefficient lambda ~ U[1250, 10000] ----
    {
        float lam = 0.f, il = 0.f;
        if (lm & B_TIMING) {
            lam = c_dc.lam_lo + c_dc.lam_range * uni(philox(g, k, CH_LAMBDA, 0).x);
            il = 1.0f / lam;
        }
        R[REC_LAMBDA * P] = __float_as_uint(lam);
        R[REC_INVLAM * P] = __float_as_uint(il);
    }
    // ---- loguniform force probability [Q19]: index + exact integer threshold ----
    {
        const uint32_t j = (lm & B_FORCE) ? (philox(g, k, CH_FORCE_P, 0).x >> 16) : 0u;
        R[REC_PINDEX * P] = j;
        R[REC_TFORCE * P] = (lm & B_FORCE) ? __ldg(p.t_tab + j) : 0u;
    }
    R[REC_EPISODE * P] = k;
    S[ST_FLAGS * P] = FRESH_BIT;   // state reads as zero at the next step [Q6, Q9]
}

__global__ void __launch_bounds__(RT_THREADS) reset_kernel_t(DevPtrs p, const uint8_t* __restrict__ mask, int first,
                                                             uint32_t n_env) {
    __shared__ float4 s_pd[MAX_PHYS];
    __shared__ uint32_t s_src[MAX_PHYS];
    __shared__ uint32_t s_env[RT_RANGE];
    __shared__ uint32_t s_kk[RT_RANGE];
    __shared__ uint32_t s_n;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    pdl_wait();   // before any global access (dr_device.cuh)
    constexpr int NWR = RT_THREADS / 32;
    for (int i = tid; i < c_dc.n_phys; i += RT_THREADS) {
        s_pd[i] = p.rs_phys[i];
        s_src[i] = p.rs_src[i];
    }
    uint32_t applied = 0;
    for (uint32_t base = blockIdx.x * RT_RANGE; base < n_env; base += gridDim.x * RT_RANGE) {
        if (tid == 0) s_n = 0u;
        __syncthreads();
        // compaction: one coalesced load of 32 mask bytes (and, for the masked lanes, episode
        // counters) per chunk; warp-aggregated append to the CTA list
        for (uint32_t c = wid; c < RT_RANGE / 32; c += NWR) {
            const uint32_t e = base + c * 32u + lane;
            const bool m = e < n_env && (mask == nullptr || mask[e] != 0);
            const uint32_t bal = __ballot_sync(0xFFFFFFFFu, m);
            if (!bal) continue;
            uint32_t pos0 = 0;
            if (lane == 0) pos0 = atomicAdd(&s_n, (uint32_t)__popc(bal));
            pos0 = __shfl_sync(0xFFFFFFFFu, pos0, 0);
            if (m) {
                const uint32_t idx = pos0 + __popc(bal & ((1u << lane) - 1u));
                s_env[idx] = e;
                s_kk[idx] = first ? 0u : p.rec[rec_index(e) + REC_EPISODE * PLANE] + 1u;
            }
            applied += (lane == 0) ? (uint32_t)__popc(bal) : 0u;
        }
        __syncthreads();
        const uint32_t n = s_n;
        for (uint32_t i = tid; i < n; i += RT_THREADS) reset_env_thread(p, s_env[i], s_kk[i], s_pd, s_src);
        __syncthreads();
    }
    pdl_trigger();
    if (!first && applied) atomicAdd(&p.ctl[2], (unsigned long long)applied);
}

// =====================================================================================
// Hybrid reset (v6, DR_RESET=6): v3's compaction and thread-per-env record chain, but the physics
// rows -- two thirds of v3's per-thread chain (64 of ~97 Philox blocks, 64 of ~114 Box-Muller
// pairs, a 256-step descriptor walk with data-dependent block draws) -- are written by a warp per
// env: lanes draw the env's physics blocks (uniform blocks -> 4 uniforms, normal blocks -> 4
// normals) into a per-warp shared-memory buffer, then lanes walk the parameters (lane q, q + 32,
// ...), so every store is one coalesced 128-byte line of phys[e][*] and the work has lane- and
// parameter-level parallelism instead of one serial chain.  Same channels, words, transforms and
// operation order as reset_env_thread (bit-identical results).
// =====================================================================================
// per-warp draw buffer: uniforms at [0, 256), normals at [256, 512), a constant 0 at 512 (the x of
// draw-free descriptors).  s_src holds, per parameter, the buffer offset of its x | RH_EXP.
constexpr int RH_DRAW = 2 * MAX_PHYS + 4;
// CTA shape of reset_kernel_h (A/B: DR_RH_THREADS / DR_RH_RANGE): threads, envs scanned per pass.
// Config 5 (1M envs, 10 % resets), reset ms per launch, three runs each: 256/2048 0.202,
// 256/1024 0.168, 128/1024 0.193, 128/512 0.165-0.170, 512/1024 0.158, 512/512 0.167,
// 256/512 0.151-0.152, 128/256 0.151, 256/256 0.163, 128/128 0.153, 64/256 0.169, 64/128 0.188.
// Small ranges (~51 resetting envs per CTA at 10 %) give thousands of short CTAs whose record
// chains and physics warps from different CTAs overlap on each SM, with a small tail.
#ifndef DR_RH_THREADS
#define DR_RH_THREADS 256
#endif
#ifndef DR_RH_RANGE
#define DR_RH_RANGE 512
#endif
#ifndef DR_RH_MINB
#define DR_RH_MINB 1   // __launch_bounds__ min CTAs per SM (A/B, reset ms: 1 (56 regs) 0.156, 5 0.165, 6 0.165, 8 0.169)
#endif
constexpr int RH_THREADS = DR_RH_THREADS;
constexpr uint32_t RH_RANGE = DR_RH_RANGE;
constexpr uint32_t RH_EXP = 1u << 31;

__device__ __forceinline__ void reset_phys_warp(const DevPtrs& p, uint32_t e, uint32_t k, int lane, float* dr,
                                                const float4* s_pd, const uint32_t* s_src, int nub, int nnb) {
    const uint32_t g = c_dc.env_offset + e;
    __syncwarp();
    for (int b = lane; b < nub + nnb; b += 32) {
        if (b < nub) {   // uniform-kind parameter u uses word u % 4 of block u / 4 (channel PHYS_U)
            const uint4 w = philox(g, k, CH_PHYS_U, (uint32_t)b);
            reinterpret_cast<float4*>(dr)[b] = make_float4(uni(w.x), uni(w.y), uni(w.z), uni(w.w));
        } else {         // normal-kind parameter n uses normal n % 4 of block n / 4 (channel PHYS_N)
            const int bn = b - nub;
            const uint4 w = philox(g, k, CH_PHYS_N, (uint32_t)bn);
            float4 z;
            box_muller(w.x, w.y, z.x, z.y);
            box_muller(w.z, w.w, z.z, z.w);
            reinterpret_cast<float4*>(dr + MAX_PHYS)[bn] = z;
        }
    }
    __syncwarp();
    const int np = c_dc.n_phys, mi = c_dc.mass_index;
    float* prow = p.phys + (size_t)e * np;
    float vm = 0.f;
#pragma unroll
    for (int i = 0; i < MAX_PHYS / 32; ++i) {
        const int q = lane + 32 * i;
        if (q < np) {
            const float4 d = s_pd[q];   // (A, B, C0, C1)
            const uint32_t o = s_src[q];
            const float x = dr[o & ~RH_EXP];
            const float tv = fmaf(d.y, x, d.x);
            const float v = fmaf(d.w, (o & RH_EXP) ? ex2_approx(tv) : tv, d.z);
            prow[q] = v;
            if (i == (mi >> 5)) vm = v;
        }
    }
    if (lane == (mi & 31)) p.rec[rec_index(e) + REC_MASS * PLANE] = __float_as_uint(vm);   // the object mass [Q18]
}

__global__ void __launch_bounds__(RH_THREADS, DR_RH_MINB) reset_kernel_h(DevPtrs p, const uint8_t* __restrict__ mask, int first,
                                                             uint32_t n_env) {
    __shared__ float4 s_pd[MAX_PHYS];
    __shared__ uint32_t s_src[MAX_PHYS];
    __shared__ uint32_t s_env[RH_RANGE];
    __shared__ uint32_t s_kk[RH_RANGE];
    __shared__ __align__(16) float s_dr[RH_THREADS / 32][RH_DRAW];
    __shared__ uint32_t s_n;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    pdl_wait();   // before any global access (dr_device.cuh)
    constexpr int NWR = RH_THREADS / 32;
    for (int i = tid; i < c_dc.n_phys; i += RH_THREADS) {
        s_pd[i] = p.rs_phys[i];
        const uint32_t src = p.rs_src[i];   // -> draw-buffer offset of x | RH_EXP (the record part does not read it)
        const uint32_t off = (src & RS_SRC_DRAW) ? (src & RS_SRC_IDX) + ((src & RS_SRC_NORMAL) ? MAX_PHYS : 0) : 2 * MAX_PHYS;
        s_src[i] = off | ((src & RS_SRC_EXP) ? RH_EXP : 0u);
    }
    if (lane == 0) s_dr[wid][2 * MAX_PHYS] = 0.f;
    const bool phys_on = (c_dc.layer_mask & B_PHYS) != 0;
    const int nub = phys_on ? (c_dc.n_phys_u + 3) / 4 : 0;
    const int nnb = phys_on ? (c_dc.n_phys_n + 3) / 4 : 0;
    uint32_t applied = 0;
    for (uint32_t base = blockIdx.x * RH_RANGE; base < n_env; base += gridDim.x * RH_RANGE) {
        if (tid == 0) s_n = 0u;
        __syncthreads();
        for (uint32_t c = wid; c < RH_RANGE / 32; c += NWR) {
            const uint32_t e = base + c * 32u + lane;
            const bool m = e < n_env && (mask == nullptr || mask[e] != 0);
            const uint32_t bal = __ballot_sync(0xFFFFFFFFu, m);
            if (!bal) continue;
            uint32_t pos0 = 0;
            if (lane == 0) pos0 = atomicAdd(&s_n, (uint32_t)__popc(bal));
            pos0 = __shfl_sync(0xFFFFFFFFu, pos0, 0);
            if (m) {
                const uint32_t idx = pos0 + __popc(bal & ((1u << lane) - 1u));
                s_env[idx] = e;
                s_kk[idx] = first ? 0u : p.rec[rec_index(e) + REC_EPISODE * PLANE] + 1u;
            }
            applied += (lane == 0) ? (uint32_t)__popc(bal) : 0u;
        }
        __syncthreads();
        const uint32_t n = s_n;
        // the record chains first (latency-bound), then the lane-parallel physics rows fill the issue slots
        for (uint32_t i = tid; i < n; i += RH_THREADS) reset_env_thread<false>(p, s_env[i], s_kk[i], s_pd, s_src);
        for (uint32_t i = wid; i < n; i += NWR) reset_phys_warp(p, s_env[i], s_kk[i], lane, s_dr[wid], s_pd, s_src, nub, nnb);
        __syncthreads();
    }
    pdl_trigger();
    if (!first && applied) atomicAdd(&p.ctl[2], (unsigned long long)applied);
}

// =====================================================================================
// Task-split reset (v5, A/B variant DR_RESET=5; v3 stays the default): the v3 thread-per-env chain (~11k dependent instructions) left
// the SMs latency-bound with ~22 resident warps of work per SM.  Here each resetting env's work
// is cut into independent tasks -- ceil(n_phys / 32) physics chunks of 32 parameters plus four
// record tasks of 7-10 Philox blocks each -- and a CTA's threads walk (task, env) items with the
// env index fastest, so a warp runs one task kind over 32 envs (warp-uniform descriptor walk).
// Capped at 40 registers (6 CTAs per SM); the host sizes the per-CTA env range so the grid is one
// resident wave (1M envs: 888 CTAs of 1,184 envs).
// Same channels, words and transforms as reset_env_thread / the oracle.
// Measured (B200, 1M envs, 10 % resets): 0.470 ms per reset+step vs v3's 0.458; ncu: 68 % warps
// active (v3 ~24 %) but 98 M warp-instructions and the stalls move to the scattered stores
// (mio / lg throttle, long scoreboard on store operands) -- more resident chains do not pay.
// =====================================================================================
constexpr int R5_THREADS = 256;
constexpr uint32_t R5_RANGE = 2048;   // max envs per CTA pass (shared-memory list size)
constexpr int R5_REC_TASKS = 4;

__device__ __forceinline__ void r5_phys_chunk(const DevPtrs& p, uint32_t e, uint32_t k, uint32_t g, int c,
                                              const float4* s_pd, const uint32_t* s_src) {
    const int np = c_dc.n_phys;
    const int q_lo = c * 32, q_hi = min(np, q_lo + 32);
    float* prow = p.phys + (size_t)e * np;
    const bool vec = (np & 3) == 0;
    uint32_t cur_n = 0xFFFFFFFFu, cur_u = 0xFFFFFFFFu;
    uint4 wu = make_uint4(0u, 0u, 0u, 0u);
    float zn[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 1
    for (int q0 = q_lo; q0 < q_hi; q0 += 4) {
        float v4[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int q = q0 + r;
            float v = 0.f;
            if (q < q_hi) {
                const float4 d = s_pd[q];
                const uint32_t src = s_src[q];
                float x = 0.f;
                if (src & RS_SRC_DRAW) {
                    if (src & RS_SRC_NORMAL) {
                        const uint32_t n = (src & RS_SRC_IDX) - ZB_PHYS;
                        if ((n >> 2) != cur_n) {
                            cur_n = n >> 2;
                            const uint4 w = philox(g, k, CH_PHYS_N, cur_n);
                            box_muller(w.x, w.y, zn[0], zn[1]);
                            box_muller(w.z, w.w, zn[2], zn[3]);
                        }
                        x = sel4(zn, n & 3u);
                    } else {
                        const uint32_t u = (src & RS_SRC_IDX) - SL_PHYS_U * 4;
                        if ((u >> 2) != cur_u) {
                            cur_u = u >> 2;
                            wu = philox(g, k, CH_PHYS_U, cur_u);
                        }
                        x = uni(selw(wu, u & 3u));
                    }
                }
                const float tv = fmaf(d.y, x, d.x);
                v = fmaf(d.w, (src & RS_SRC_EXP) ? ex2_approx(tv) : tv, d.z);
                if (q == c_dc.mass_index) p.rec[rec_index(e) + REC_MASS * PLANE] = __float_as_uint(v);   // [Q18]
                if (!vec) prow[q] = v;
            }
            v4[r] = v;
        }
        if (vec) reinterpret_cast<float4*>(prow)[q0 >> 2] = make_float4(v4[0], v4[1], v4[2], v4[3]);
    }
}

__device__ __forceinline__ void r5_record_task(const DevPtrs& p, uint32_t e, uint32_t k, uint32_t g, int t) {
    const uint32_t lm = c_dc.layer_mask;
    constexpr size_t P = PLANE;
    uint32_t* R = p.rec + rec_index(e);
    if (t == 0) {
        // delay flags, timing lambda, force probability [Q19]
        uint32_t bits = 0u;
        if (lm & B_DELAY) {
#pragma unroll
            for (int b = 0; b < 5; ++b) {
                const uint4 w = philox(g, k, CH_DELAY, b);
                const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    bits |= ((unsigned long long)ws[q] < c_dc.t_delay ? 1u : 0u) << (4 * b + q);
            }
        }
        R[REC_DELAY * P] = bits;
        float lam = 0.f, il = 0.f;
        if (lm & B_TIMING) {
            lam = c_dc.lam_lo + c_dc.lam_range * uni(philox(g, k, CH_LAMBDA, 0).x);
            il = 1.0f / lam;
        }
        R[REC_LAMBDA * P] = __float_as_uint(lam);
        R[REC_INVLAM * P] = __float_as_uint(il);
        const uint32_t j = (lm & B_FORCE) ? (philox(g, k, CH_FORCE_P, 0).x >> 16) : 0u;
        R[REC_PINDEX * P] = j;
        R[REC_TFORCE * P] = (lm & B_FORCE) ? __ldg(p.t_tab + j) : 0u;
        R[REC_EPISODE * P] = k;
        p.st[st_index(e) + ST_FLAGS * P] = FRESH_BIT;   // state reads as zero next step [Q6, Q9]
    } else if (t == 1) {
        // backlash widths [Q7]: normal j -> delta-1_j, 20 + j -> delta+1_j
#pragma unroll 1
        for (int b = 0; b < 10; ++b) {
            float z[4] = {0.f, 0.f, 0.f, 0.f};
            if (lm & B_BACKLASH) {
                const uint4 w = philox(g, k, CH_BACKLASH, b);
                box_muller(w.x, w.y, z[0], z[1]);
                box_muller(w.z, w.w, z[2], z[3]);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int n = 4 * b + q;
                const int j = n < N_ACT ? n : n - N_ACT;
                const float cal = n < N_ACT ? c_dc.dcal_neg[j] : c_dc.dcal_pos[j];
                const float dv = (lm & B_BACKLASH) ? fmaxf(0.f, cal + c_dc.jitter * z[q]) : 0.f;
                R[((n < N_ACT ? REC_DNEG : REC_DPOS) + j) * P] = __float_as_uint(dv);
            }
        }
    } else if (t == 2) {
        // correlated action offset (Table action-noise); object offset and rotation
#pragma unroll 1
        for (int b = 0; b < 5; ++b) {
            float z[4] = {0.f, 0.f, 0.f, 0.f};
            if (lm & B_ACT_NOISE) {
                const uint4 w = philox(g, k, CH_CORR_ACT, b);
                box_muller(w.x, w.y, z[0], z[1]);
                box_muller(w.z, w.w, z[2], z[3]);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) R[(REC_CACT + 4 * b + q) * P] = __float_as_uint(c_dc.sc * z[q]);
        }
        float zo[4] = {0.f, 0.f, 0.f, 0.f};
        float q[4] = {1.f, 0.f, 0.f, 0.f};
        if (lm & B_OBS_NOISE) {
            const uint4 wo = philox(g, k, CH_CORR_OBJ, 0);
            box_muller(wo.x, wo.y, zo[0], zo[1]);
            box_muller(wo.z, wo.w, zo[2], zo[3]);
            rotation(c_dc.rot_corr, philox(g, k, CH_CORR_ROT, 0), q);
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) R[(REC_COBJ + c) * P] = __float_as_uint(c_dc.obj_corr * zo[c]);
#pragma unroll
        for (int c = 0; c < 4; ++c) R[(REC_QC + c) * P] = __float_as_uint(q[c]);
    } else {
        // fingertip offsets [Q14, Q15]
        if (lm & B_OBS_NOISE) {
            float mb[4];
            {
                const uint4 w = philox(g, k, CH_MARKER_BASE, 0);
                box_muller(w.x, w.y, mb[0], mb[1]);
                box_muller(w.z, w.w, mb[2], mb[3]);
            }
#pragma unroll 1
            for (int b = 0; b < 4; ++b) {
                float zc[4], zm[4];
                const uint4 wc = philox(g, k, CH_CORR_TIP, b);
                const uint4 wm = philox(g, k, CH_MARKER_TIP, b);
                box_muller(wc.x, wc.y, zc[0], zc[1]);
                box_muller(wc.z, wc.w, zc[2], zc[3]);
                box_muller(wm.x, wm.y, zm[0], zm[1]);
                box_muller(wm.z, wm.w, zm[2], zm[3]);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int n = 4 * b + q;
                    if (n < 15) {
                        float v = c_dc.tip_corr * zc[q] + c_dc.tip_marker * zm[q];
                        if (c_dc.base_to_tips) v = v - c_dc.base_marker * sel4(mb, (uint32_t)(n % 3));
                        R[(REC_OFFTIP + n) * P] = __float_as_uint(v);
                    }
                }
            }
        } else {
#pragma unroll
            for (int n = 0; n < 15; ++n) R[(REC_OFFTIP + n) * P] = 0u;
        }
    }
}

__global__ void __launch_bounds__(R5_THREADS, 6) reset_kernel_v5(DevPtrs p, const uint8_t* __restrict__ mask,
                                                                 int first, uint32_t n_env, uint32_t range) {
    __shared__ float4 s_pd[MAX_PHYS];
    __shared__ uint32_t s_src[MAX_PHYS];
    __shared__ uint32_t s_env[R5_RANGE];
    __shared__ uint32_t s_kk[R5_RANGE];
    __shared__ uint32_t s_n;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    pdl_wait();   // before any global access (dr_device.cuh)
    constexpr int NWR = R5_THREADS / 32;
    const int np = c_dc.n_phys;
    for (int i = tid; i < np; i += R5_THREADS) {
        s_pd[i] = p.rs_phys[i];
        s_src[i] = p.rs_src[i];
    }
    const int n_pt = (np + 31) >> 5;   // physics chunks
    const uint32_t n_tasks = (uint32_t)(n_pt + R5_REC_TASKS);
    uint32_t applied = 0;
    for (uint32_t base = blockIdx.x * range; base < n_env; base += gridDim.x * range) {
        if (tid == 0) s_n = 0u;
        __syncthreads();
        for (uint32_t c = wid; c < range / 32; c += NWR) {
            const uint32_t e = base + c * 32u + lane;
            const bool m = e < n_env && (mask == nullptr || mask[e] != 0);
            const uint32_t bal = __ballot_sync(0xFFFFFFFFu, m);
            if (!bal) continue;
            uint32_t pos0 = 0;
            if (lane == 0) pos0 = atomicAdd(&s_n, (uint32_t)__popc(bal));
            pos0 = __shfl_sync(0xFFFFFFFFu, pos0, 0);
            if (m) {
                const uint32_t idx = pos0 + __popc(bal & ((1u << lane) - 1u));
                s_env[idx] = e;
                s_kk[idx] = first ? 0u : p.rec[rec_index(e) + REC_EPISODE * PLANE] + 1u;
            }
            applied += (lane == 0) ? (uint32_t)__popc(bal) : 0u;
        }
        __syncthreads();
        const uint32_t n = s_n;
        const uint32_t n32 = (n + 31u) & ~31u;   // each task's segment padded to whole warps: no warp
        const uint32_t total = n32 * n_tasks;    // straddles two task kinds (no divergent task code)
        // the record tasks (longer) first, so the tail is made of short physics chunks
        for (uint32_t j = tid; j < total; j += R5_THREADS) {
            const uint32_t t = j / n32, i = j - t * n32;
            if (i >= n) continue;
            const uint32_t e = s_env[i], k = s_kk[i];
            const uint32_t g = c_dc.env_offset + e;
            if (t < (uint32_t)R5_REC_TASKS) r5_record_task(p, e, k, g, (int)t);
            else r5_phys_chunk(p, e, k, g, (int)t - R5_REC_TASKS, s_pd, s_src);
        }
        __syncthreads();
    }
    pdl_trigger();
    if (!first && applied) atomicAdd(&p.ctl[2], (unsigned long long)applied);
}
