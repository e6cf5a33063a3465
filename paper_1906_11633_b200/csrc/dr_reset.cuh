// dr_reset.cuh -- episode-reset sampling (PAPER.md:7-8, 13, 15-18, 36-41, 77-78, 87-88, 100-101,
// 113), included by dr_kernels.cu inside namespace dr.
//
// A warp ballots 32 mask bytes, then serves each resetting env with all 32 lanes in four
// warp-uniform phases (no lane-divergent transcendental code):
//   A. the Philox blocks of every enabled reset channel, one block per lane, into shared memory;
//   B. every Box-Muller pair the episode needs (physics normals + record normals), one pair per
//      lane, into a per-warp z buffer;
//   C. the n_phys physical parameters, one lane per parameter, branch-light (expf evaluated for
//      every kind, then selected), written as coalesced 128-byte lines of the row phys[e][*];
//   D. the episode record fields (cheap arithmetic on the staged draws), one lane per field.
// The 60 state planes are not zeroed here: one word (FRESH_BIT in the flags plane) marks the env,
// and the step kernel treats a fresh env's state as zero (dr_internal.h).
#pragma once

// Philox block slots per env (fixed offsets; blocks of disabled layers are skipped).
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

// z buffer (per warp): normal n of a channel at its base + n
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

// Box-Muller pair task t -> (first slot of the channel, pair index, z-buffer base).
// Pair p of a channel uses block p / 2, words (x, y) for even p and (z, w) for odd p, and yields
// normals 2p (cos) and 2p + 1 (sin) -- the same indexing as the oracle's draw_normal.
__device__ __forceinline__ void pair_task(int t, int np_phys, uint32_t lm, int& slot, int& pair, int& zb) {
    if (t < np_phys) { slot = SL_PHYS_N; pair = t; zb = ZB_PHYS; return; }
    t -= np_phys;
    if (lm & B_BACKLASH) { if (t < 20) { slot = SL_BACKLASH; pair = t; zb = ZB_BL; return; } t -= 20; }
    if (lm & B_ACT_NOISE) { if (t < 10) { slot = SL_CORR_ACT; pair = t; zb = ZB_CA; return; } t -= 10; }
    // OBS_NOISE: 8 + 8 + 2 + 2
    if (t < 8) { slot = SL_CORR_TIP; pair = t; zb = ZB_CT; return; }
    t -= 8;
    if (t < 8) { slot = SL_MARKER_TIP; pair = t; zb = ZB_MT; return; }
    t -= 8;
    if (t < 2) { slot = SL_MARKER_BASE; pair = t; zb = ZB_MB; return; }
    t -= 2;
    slot = SL_CORR_OBJ; pair = t; zb = ZB_CO;
}

__device__ __forceinline__ void reset_one(const DevPtrs& p, uint32_t e, bool first, int lane, uint4* w, float* zb,
                                          const float4* s_pd) {
    const uint32_t lm = c_dc.layer_mask;
    constexpr size_t P = PLANE;
    uint32_t* R = p.rec + rec_index(e);
    uint32_t* S = p.st + st_index(e);
    const uint32_t g = c_dc.env_offset + e;
    const uint32_t k = first ? 0u : R[REC_EPISODE * P] + 1u;
    __syncwarp();
    // A. Philox blocks of every enabled reset channel, spread over the lanes
    for (int i = lane; i < SL_COUNT; i += 32) {
        uint32_t ch, blk;
        if (slot_channel(i, lm, ch, blk)) w[i] = philox(g, k, ch, blk);
    }
    __syncwarp();
    // B. every Box-Muller pair, one per lane (warp-uniform code; only the operands differ)
    {
        const int np_phys = (lm & B_PHYS) ? (c_dc.n_phys_n + 1) / 2 : 0;
        const int n_tasks = np_phys + ((lm & B_BACKLASH) ? 20 : 0) + ((lm & B_ACT_NOISE) ? 10 : 0) +
                            ((lm & B_OBS_NOISE) ? 20 : 0);
        for (int t = lane; t < n_tasks; t += 32) {
            int slot, pr, base;
            pair_task(t, np_phys, lm, slot, pr, base);
            const uint4 b = w[slot + (pr >> 1)];
            float z0, z1;
            box_muller((pr & 1) ? b.z : b.x, (pr & 1) ? b.w : b.y, z0, z1);
            zb[base + 2 * pr] = z0;
            zb[base + 2 * pr + 1] = z1;
        }
    }
    __syncwarp();
    // C. physical parameters (descriptor schema SPEC.md:126) [Q20]
    const int np = c_dc.n_phys;
    float* prow = p.phys + (size_t)e * np;
    for (int q = lane; q < np; q += 32) {
        const float4 d = s_pd[q];                       // (a', b', base, kind | rank << 8)
        const uint32_t kr = __float_as_uint(d.w);
        const uint32_t kind = kr & 0xFFu, rank = kr >> 8;
        float v = d.z;
        if (lm & B_PHYS) {
            float tv = 0.f;
            if (kind == 1u || kind == 2u) tv = d.x + d.y * uni(word_of(w[SL_PHYS_U + (rank >> 2)], rank & 3));
            else if (kind == 3u || kind == 4u) tv = d.x * zb[ZB_PHYS + rank];
            const float ex = expf(tv);
            v = (kind == 1u) ? d.z * tv : (kind == 3u) ? d.z + tv : (kind == 2u || kind == 4u) ? d.z * ex : d.z;
        }
        prow[q] = v;
        if (q == c_dc.mass_index) R[REC_MASS * P] = __float_as_uint(v);   // the object mass [Q18]
    }
    // D1. per actuator: delay flag, backlash widths [Q7],
    //     correlated action noise (Table action-noise)
    {
        const int j = lane;
        bool dflag = false;
        if (j < N_ACT) {
            if (lm & B_DELAY) dflag = (unsigned long long)word_of(w[SL_DELAY + (j >> 2)], j & 3) < c_dc.t_delay;
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
        uint32_t j = 0, tf = 0;
        if (lm & B_FORCE) {
            j = w[SL_FORCE_P].x >> 16;
            tf = __ldg(p.t_tab + j);
        }
        R[REC_PINDEX * P] = j;
        R[REC_TFORCE * P] = tf;
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
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < c_dc.n_phys; i += RESET_THREADS)
        s_pd[i] = make_float4(__ldg(p.pd_a + i), __ldg(p.pd_b + i), __ldg(p.pd_base + i),
                              __uint_as_float(__ldg(p.pd_kind_rank + i)));
    __syncthreads();
    const uint32_t n_chunks = (n_env + 31u) >> 5;
    const uint32_t nw = gridDim.x * RESET_WARPS;
    uint32_t applied = 0;
    for (uint32_t c = blockIdx.x * RESET_WARPS + wib; c < n_chunks; c += nw) {
        const uint32_t e = (c << 5) + lane;
        const bool m = e < n_env && (mask == nullptr || mask[e] != 0);
        uint32_t bal = __ballot_sync(0xFFFFFFFFu, m);
        applied += __popc(bal);
        while (bal) {
            const int b = __ffs(bal) - 1;
            bal &= bal - 1;
            reset_one(p, (c << 5) + b, first != 0, lane, s_w[wib], s_zb[wib], s_pd);
        }
    }
    if (!first && lane == 0 && applied) atomicAdd(&p.ctl[2], (unsigned long long)applied);
}
