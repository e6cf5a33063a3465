// dr_step.cuh -- the fused per-env-step kernel, included by dr_kernels.cu
// inside namespace dr (after on<L>() and the B_* layer bits).
//
// Mapping: persistent CTAs of TILE (=128) threads, one thread per env, static round-robin tiles.
//
// Data movement (every byte of state makes one HBM round trip per step):
//   * Row-major I/O tiles ([n][20] actions, [n][26] raw_obs) are staged into shared memory with
//     16-byte cp.async (LDGSTS, no register round trip); outputs are written in place over the
//     input rows (out_actions over actions, out_obs + out_force over raw_obs) and stored with
//     coalesced 128/64-bit stores.
//   * The SoA record/state planes (one 128-B line per warp per plane) are software-pipelined
//     through a per-thread two-slot shared-memory ring with 4-byte cp.async: while the thread
//     computes phase k from one slot, the copies of phase k+1 are in flight into the other.
//     Phases: S0 (scalars), A0..A4 (4 actuators each), OB (observation offsets).  In-flight data
//     occupies shared memory, not registers, which is what lets the SM keep enough bytes in
//     flight to approach the HBM roofline with a register-heavy (Philox + Box-Muller) thread.
//   * Held fingertip readings ("last") are fetched with cp.async into the thread's raw-tip slots
//     (already consumed) while the fingertip noise is computed.
//   * stats: per-thread register accumulators -> CTA reduction in shared memory -> per-CTA
//     partials reduced by the last CTA in a fixed order (deterministic fp64 sums).
#pragma once

enum : int { K_DELAYED = 0, K_DROP_INIT, K_MASKED, K_OCCLUDED, K_HELD, K_TRIG, K_RAIL, K_ALPHA1, K_CLAMPS, K_COUNT };

struct Acc {
    uint32_t n[K_COUNT];
    float m[8];   // a thread sums only its ~n/(grid*TILE) envs in fp32; CTA and grid sums are fp64
};

// ---- cp.async (LDGSTS) helpers ------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp_async4(void* sdst, const void* gsrc) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(sdst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sdst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void l2_prefetch(const void* ptr, uint32_t bytes) {
    if (bytes >= 16u)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(ptr), "r"(bytes & ~15u) : "memory");
}

// Optional TMA bulk L2 prefetch of every plane chunk + input row range of a tile (DR_PREFETCH).
template <uint32_t L>
__device__ __forceinline__ void prefetch_tile(const DevPtrs& p, const float* actions, const float* raw_obs,
                                              uint32_t tile, uint32_t n_env) {
    const uint32_t e0 = tile * TILE;
    if (e0 >= n_env) return;
    const uint32_t cnt = min((uint32_t)TILE, n_env - e0);
    // AoSoA: the tile's record planes and state planes are two contiguous blocks
    for (int item = threadIdx.x; item < 4; item += blockDim.x) {
        if (item == 0) {
            l2_prefetch(p.rec + rec_index(e0), REC_STEP_PLANES * TILE * 4u);
        } else if (item == 1) {
            l2_prefetch(p.st + st_index(e0), ST_PLANES * TILE * 4u);
        } else if (item == 2) {
            l2_prefetch(actions + (size_t)e0 * N_ACT, cnt * N_ACT * 4u);
        } else {
            l2_prefetch(raw_obs + (size_t)e0 * OBS_IN, cnt * OBS_IN * 4u);   // rounded down: in bounds
        }
    }
}

// ---- phase ring ----------------------------------------------------------------------------
// slot word w of thread tid lives at ring[(slot * RING_W + w) * TILE + tid]: the 32 lanes of a
// warp touch 32 consecutive words (conflict-free LDS, coalesced LDGSTS).
constexpr int RING_W = 22;
constexpr size_t STEP_DYN_SMEM = 2 * RING_W * TILE * sizeof(uint32_t);
enum : int { S0_INVLAM = 0, S0_DELAY, S0_FLAGS, S0_TFORCE, S0_MASS, S0_KF, S0_FTRIG };   // FTRIG: 3 words

template <uint32_t L>
__device__ __forceinline__ void issue_s0(uint32_t* slot, const uint32_t* R, const uint32_t* S, size_t P) {
    if (on<L>(B_TIMING)) cp_async4(slot + S0_INVLAM * TILE, R + REC_INVLAM * P);
    if (on<L>(B_DELAY)) cp_async4(slot + S0_DELAY * TILE, R + REC_DELAY * P);
    if (on<L>(B_STATEFUL)) cp_async4(slot + S0_FLAGS * TILE, S + ST_FLAGS * P);   // timers, has_last, FRESH
    if (on<L>(B_FORCE)) {
        cp_async4(slot + S0_TFORCE * TILE, R + REC_TFORCE * P);
        cp_async4(slot + S0_MASS * TILE, R + REC_MASS * P);
        cp_async4(slot + S0_KF * TILE, S + ST_KF * P);
#pragma unroll
        for (int c = 0; c < 3; ++c) cp_async4(slot + (S0_FTRIG + c) * TILE, S + (ST_FTRIG + c) * P);
    }
}

// actuator block b: words [prev 4 | slack 4 | dneg 4 | dpos 4 | cact 4]
template <uint32_t L>
__device__ __forceinline__ void issue_act(uint32_t* slot, const uint32_t* R, const uint32_t* S, size_t P, int b) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int j = 4 * b + q;
        if (on<L>(B_DELAY)) cp_async4(slot + (0 + q) * TILE, S + (ST_PREV + j) * P);
        if (on<L>(B_BACKLASH)) {
            cp_async4(slot + (4 + q) * TILE, S + (ST_SLACK + j) * P);
            cp_async4(slot + (8 + q) * TILE, R + (REC_DNEG + j) * P);
            cp_async4(slot + (12 + q) * TILE, R + (REC_DPOS + j) * P);
        }
        if (on<L>(B_ACT_NOISE)) cp_async4(slot + (16 + q) * TILE, R + (REC_CACT + j) * P);
    }
}

// observation offsets: words [offtip 15 | c_obj 3 | q_c 4]  (REC_OFFTIP..REC_QC are contiguous planes)
template <uint32_t L>
__device__ __forceinline__ void issue_obs(uint32_t* slot, const uint32_t* R, size_t P) {
    if (on<L>(B_OBS_NOISE)) {
#pragma unroll
        for (int w = 0; w < 22; ++w) cp_async4(slot + w * TILE, R + (REC_OFFTIP + w) * P);
    }
}

__device__ __forceinline__ float ringf(const uint32_t* slot, int w) { return __uint_as_float(slot[w * TILE]); }

template <uint32_t L>
__device__ __forceinline__ void env_step(const DevPtrs& p, uint32_t e, uint32_t t, int tid, float* s_act,
                                         float* s_obs, float* s_dt, uint32_t* ring, Acc& acc) {
    constexpr size_t P = PLANE;
    const uint32_t* R = p.rec + rec_index(e);
    uint32_t* S = p.st + st_index(e);
    const uint32_t g = c_dc.env_offset + e;
    constexpr bool kHold = (L == RUNTIME_MASK) || (L & (B_DROPOUT | B_OCCLUSION));
    const bool hold_layers = on<L>(B_DROPOUT) || on<L>(B_OCCLUSION);
    uint32_t* slot0 = ring + tid;
    uint32_t* slot1 = ring + RING_W * TILE + tid;

    // ---- S0 (slot0) has landed (the tile loop waited for it); A0 is in flight into slot1 ----
    const float il = on<L>(B_TIMING) ? ringf(slot0, S0_INVLAM) : 0.f;
    const uint32_t dbits = on<L>(B_DELAY) ? slot0[S0_DELAY * TILE] : 0u;
    // a FRESH env (reset since its last step) has all-zero state: slack 0, prev 0, no reading,
    // timers 0, force 0 -- the reset kernel does not write the state planes
    const uint32_t flags_raw = on<L>(B_STATEFUL) ? slot0[S0_FLAGS * TILE] : 0u;
    const bool fresh = (flags_raw & FRESH_BIT) != 0u;
    const uint32_t flags = (kHold && hold_layers && !fresh) ? flags_raw : 0u;
    uint32_t tf = 0, kf = 0;
    float mass = 0.f, ft[3] = {0.f, 0.f, 0.f};
    if (on<L>(B_FORCE)) {
        tf = slot0[S0_TFORCE * TILE];
        mass = ringf(slot0, S0_MASS);
        if (!fresh) {
            kf = slot0[S0_KF * TILE];
#pragma unroll
            for (int c = 0; c < 3; ++c) ft[c] = ringf(slot0, S0_FTRIG + c);
        }
    }
    issue_act<L>(slot0, R, S, P, 1);   // A1 -> slot0
    cp_commit();

    // ---- 1. timing: 10 substeps of 8 ms + Exp(lambda); dt_env = sum [Q2] ----
    float dt_env;
    {
        float d[N_SUB];
        if (on<L>(B_TIMING)) {
#pragma unroll
            for (int b = 0; b < 3; ++b) {
                const uint4 w = philox(g, t, CH_TIMING, b);
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (4 * b + q < N_SUB)
                        d[4 * b + q] = c_dc.dt_base + (-(kSfuNormals ? ln_unit_sfu(uni(word_of(w, q))) : ln_unit(uni(word_of(w, q))))) * il;
            }
        } else {
#pragma unroll
            for (int k = 0; k < N_SUB; ++k) d[k] = c_dc.dt_base;
        }
        dt_env = d[0];
#pragma unroll
        for (int k = 1; k < N_SUB; ++k) dt_env = dt_env + d[k];
        float2* d2 = reinterpret_cast<float2*>(s_dt + tid * N_SUB);
#pragma unroll
        for (int k = 0; k < N_SUB / 2; ++k) d2[k] = make_float2(d[2 * k], d[2 * k + 1]);
        acc.m[0] += dt_env;
        acc.m[1] += dt_env * dt_env;
    }

    // ---- 2-4. actions: delay -> noise -> clamp -> backlash [Q1] ----
    acc.n[K_DELAYED] += __popc(dbits);
    float s_da = 0.f, s_da2 = 0.f, s_bl = 0.f, s_zu2 = 0.f;
    float4* a4p = reinterpret_cast<float4*>(s_act + tid * N_ACT);
#pragma unroll 1
    for (int b = 0; b < 5; ++b) {   // rolled: keeps the kernel inside the instruction cache
        cp_wait<1>();                // A_b has landed
        uint32_t* sl = (b & 1) ? slot0 : slot1;
        float prev[4], slack[4], dneg[4], dpos[4], cact[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            prev[q] = (on<L>(B_DELAY) && !fresh) ? ringf(sl, q) : 0.f;
            slack[q] = (on<L>(B_BACKLASH) && !fresh) ? ringf(sl, 4 + q) : 0.f;
            dneg[q] = on<L>(B_BACKLASH) ? ringf(sl, 8 + q) : 0.f;
            dpos[q] = on<L>(B_BACKLASH) ? ringf(sl, 12 + q) : 0.f;
            cact[q] = on<L>(B_ACT_NOISE) ? ringf(sl, 16 + q) : 0.f;
        }
        // refill the slot just consumed: A_{b+2}, then the observation offsets
        if (b + 2 < 5) issue_act<L>(sl, R, S, P, b + 2);
        else if (b + 2 == 5) issue_obs<L>(sl, R, P);
        cp_commit();

        float zu[4], zm[4];
        if (on<L>(B_ACT_NOISE)) {
            normals4_t<kSfuNormals>(philox(g, t, CH_ACT_UADD, b), zu);
            normals4_t<kSfuNormals>(philox(g, t, CH_ACT_MULT, b), zm);
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
                if ((dbits >> j) & 1u) ad = prev[q];
                S[(ST_PREV + j) * P] = __float_as_uint(a);
            }
            float an = ad;
            if (on<L>(B_ACT_NOISE)) {
                // Table action-noise [Q8]
                an = ad + ad * (c_dc.sm * zm[q]);
                an = an + c_dc.su * zu[q];
                an = an + cact[q];
                acc.n[K_CLAMPS] += (an > 1.f || an < -1.f) ? 1u : 0u;
                an = fminf(fmaxf(an, -1.f), 1.f);
                s_zu2 += zu[q] * zu[q];
            }
            const float da = an - ad;
            s_da += da;
            s_da2 += da * da;
            float out = an;
            if (on<L>(B_BACKLASH)) {
                // backlash, verbatim [Q4], sgn(0) = 0 [Q3]:
                // alpha = 1 - clamp(|sgn - s| / (|s' - s| + eps), 0, 1).  The ratio is >= 1 (alpha 0)
                // unless s sits on the rail sgn already (num == 0: alpha 1) or s' lands on the
                // rail within eps of it (num < den: the one case that needs the division).
                const float s = slack[q];
                const float sg = (an > 0.f) ? 1.f : ((an < 0.f) ? -1.f : 0.f);
                const float d = (an > 0.f) ? dpos[q] : ((an < 0.f) ? dneg[q] : 0.f);
                const float sp = fminf(fmaxf(s + an * d * dt_env, -1.f), 1.f);
                const float num = fabsf(sg - s), den = fabsf(sp - s) + c_dc.eps;
                // num < den only when num < ~1.7e-5 (else num + eps rounds to num in fp32); there
                // alpha = 1 - num/den is a cancellation whose absolute error (<= 2 ulp of 1 with the
                // fast divide) is far inside the 1e-6 budget of alpha * a_n -- so no branch.
                const float al = (num == 0.f) ? 1.f : ((num < den) ? 1.f - __fdividef(num, den) : 0.f);
                out = al * an;
                acc.n[K_RAIL] += (sg != 0.f && fabsf(sp) == 1.f && sp != s) ? 1u : 0u;
                acc.n[K_ALPHA1] += (al == 1.f) ? 1u : 0u;
                S[(ST_SLACK + j) * P] = __float_as_uint(sp);
            }
            s_bl += fabsf(out - an);
            ov[q] = out;
        }
        a4p[b] = make_float4(ov[0], ov[1], ov[2], ov[3]);
    }
    acc.m[2] += s_da;
    acc.m[3] += s_da2;
    acc.m[4] += s_bl;
    acc.m[5] += s_zu2;

    // ---- 5-8. fingertip markers and object position ----
    float* ro = s_obs + tid * OBS_IN;   // raw row in; out_obs (22) + out_force (3) written in place
    float tip[15], obj[3];
    {
        const float2* r2 = reinterpret_cast<const float2*>(ro);
#pragma unroll
        for (int k = 0; k < 9; ++k) {
            const float2 v = r2[k];
            const float x[2] = {v.x, v.y};
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int c = 2 * k + h;
                if (c < 15) tip[c] = x[h];
                else obj[c - 15] = x[h];
            }
        }
    }
    uint32_t occ = 0;
    if (on<L>(B_OCCLUSION) && c_dc.occl_on) {
        // occlusion: another tip or the object centre strictly closer than r [Q13].
        // The decision is the exactly rounded fp64 ((dx*dx + dy*dy) + dz*dz) < r^2 of the oracle.
        // Fast path: every fp32 op is correctly rounded, so the fp32 sum is within a few ulp
        // (relative) of the exact one; only pairs inside a 1e-5 relative band around r^2 (never,
        // in practice) are decided by the exact fp64 evaluation.
        const float lo = c_dc.occl_r2_lo, hi = c_dc.occl_r2_hi;
        uint32_t amb = 0;   // ambiguous pairs, bit 6 i + (j - i - 1)
#pragma unroll
        for (int i = 0; i < N_TIPS; ++i) {
#pragma unroll
            for (int j = i + 1; j <= N_TIPS; ++j) {
                const float* o = (j < N_TIPS) ? &tip[3 * j] : obj;
                const float dx = tip[3 * i] - o[0], dy = tip[3 * i + 1] - o[1], dz = tip[3 * i + 2] - o[2];
                const float d2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
                const uint32_t pair = (1u << i) | ((j < N_TIPS) ? (1u << j) : 0u);
                if (d2 < lo) occ |= pair;
                else if (!(d2 > hi)) amb |= 1u << (6 * i + (j - i - 1));
            }
        }
        if (amb | c_dc.occl_exact_only) {
            const double r2 = c_dc.occl_r2;
            for (int i = 0; i < N_TIPS; ++i) {
                for (int j = i + 1; j <= N_TIPS; ++j) {
                    if (!c_dc.occl_exact_only && !((amb >> (6 * i + (j - i - 1))) & 1u)) continue;
                    const float* o = (j < N_TIPS) ? &tip[3 * j] : obj;
                    const double dx = __dsub_rn((double)tip[3 * i], (double)o[0]);
                    const double dy = __dsub_rn((double)tip[3 * i + 1], (double)o[1]);
                    const double dz = __dsub_rn((double)tip[3 * i + 2], (double)o[2]);
                    const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
                    if (d2 < r2) occ |= (1u << i) | ((j < N_TIPS) ? (1u << j) : 0u);
                }
            }
        }
        acc.n[K_OCCLUDED] += __popc(occ);
    }
    uint32_t masked = 0;
    if (kHold && hold_layers) {
        uint32_t nflags = 0;
        if (on<L>(B_DROPOUT)) {
            // dropout: a 13-step mask starts with probability 1 - exp(-0.2 * 0.08) per step;
            // a retrigger restarts it [Q11]
            const uint4 w0 = philox(g, t, CH_DROPOUT, 0);
            const uint32_t x4 = philox(g, t, CH_DROPOUT, 1).x;
#pragma unroll
            for (int i = 0; i < N_TIPS; ++i) {
                const uint32_t x = (i < 4) ? word_of(w0, i) : x4;
                uint32_t tm = (flags >> (4 * i)) & 0xFu;
                if ((unsigned long long)x < c_dc.t_drop) { tm = c_dc.hold_steps; acc.n[K_DROP_INIT] += 1; }
                if (tm > 0u) { masked |= 1u << i; tm -= 1u; }
                nflags |= tm << (4 * i);
            }
            acc.n[K_MASKED] += __popc(masked);
        }
        S[ST_FLAGS * P] = nflags | HAS_LAST_BIT;
    } else if (on<L>(B_STATEFUL) && fresh) {
        S[ST_FLAGS * P] = 0u;   // clear FRESH (no hold layers: timers / has_last unused)
    }
    const uint32_t hold = (flags & HAS_LAST_BIT) ? (masked | occ) : 0u;
    acc.n[K_HELD] += __popc(hold);
    // held tips return their last available reading [Q12]: fetch it asynchronously
    // into this thread's raw-tip slots (already consumed) while the noise below is computed.
    if (kHold && hold) {
#pragma unroll
        for (int i = 0; i < N_TIPS; ++i)
            if ((hold >> i) & 1u)
#pragma unroll
                for (int c = 0; c < 3; ++c) cp_async4(ro + 3 * i + c, S + (ST_LAST + 3 * i + c) * P);
    }
    cp_commit();
    cp_wait<1>();   // the observation offsets (issued at b = 3) have landed in slot0
    // fingertips: + (correlated + misplacement offset) + 2 mm uncorrelated
    float s_zt = 0.f;
    if (on<L>(B_OBS_NOISE)) {
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            float z[4];
            normals4_t<kSfuNormals>(philox(g, t, CH_TIP_NOISE, b), z);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int n = 4 * b + q;
                if (n < 15) {
                    tip[n] = (tip[n] + ringf(slot0, n)) + c_dc.tip_uncorr * z[q];
                    s_zt += z[q] * z[q];
                }
            }
        }
    }
    acc.m[6] += s_zt;
    cp_wait<0>();   // held readings
    if (kHold && hold_layers) {
#pragma unroll
        for (int i = 0; i < N_TIPS; ++i) {
            if ((hold >> i) & 1u) {
#pragma unroll
                for (int c = 0; c < 3; ++c) tip[3 * i + c] = ro[3 * i + c];   // unchanged: no store
            } else {
#pragma unroll
                for (int c = 0; c < 3; ++c) S[(ST_LAST + 3 * i + c) * P] = __float_as_uint(tip[3 * i + c]);
            }
        }
    }
    // object position: + 5 mm correlated + 1 mm uncorrelated
    if (on<L>(B_OBS_NOISE)) {
        float z[4];
        normals4_t<kSfuNormals>(philox(g, t, CH_OBJ_NOISE, 0), z);
#pragma unroll
        for (int c = 0; c < 3; ++c) obj[c] = (obj[c] + ringf(slot0, 15 + c)) + c_dc.obj_uncorr * z[c];
    }

    // ---- 9. orientation noise -> noisy relative goal [Q15, Q16] ----
    float rel[4];
    {
        // raw q_obj = ro[18..21], goal = ro[22..25] (rows are 8-byte aligned: float2 reads)
        const float2 qa = reinterpret_cast<const float2*>(ro + 18)[0], qb = reinterpret_cast<const float2*>(ro + 20)[0];
        const float2 ga = reinterpret_cast<const float2*>(ro + 22)[0], gb = reinterpret_cast<const float2*>(ro + 24)[0];
        const float qo[4] = {qa.x, qa.y, qb.x, qb.y};
        const float goal[4] = {ga.x, ga.y, gb.x, gb.y};
        float qn[4];
        if (on<L>(B_OBS_NOISE)) {
            float qu[4], tmp[4];
            const float qc[4] = {ringf(slot0, 18), ringf(slot0, 19), ringf(slot0, 20), ringf(slot0, 21)};
            rotation<kSfuNormals>(c_dc.rot_uncorr, philox(g, t, CH_ROT_NOISE, 0), qu);
            qmul(qc, qo, tmp);
            qmul(qu, tmp, qn);
        } else {
#pragma unroll
            for (int c = 0; c < 4; ++c) qn[c] = qo[c];
        }
        const float cj[4] = {qn[0], -qn[1], -qn[2], -qn[3]};
        qmul(goal, cj, rel);
        const float sgn = (rel[0] < 0.f) ? -1.f : 1.f;
#pragma unroll
        for (int c = 0; c < 4; ++c) rel[c] *= sgn;
    }

    // ---- 10. random force: replace on trigger, decay 0.99 per step in closed form
    //           [Q17, Q18] ----
    float f[3] = {0.f, 0.f, 0.f};
    if (on<L>(B_FORCE)) {
        const uint32_t x = philox(g, t, CH_FORCE, 0).x;
        if (x < tf) {
            const uint4 w = philox(g, t, CH_FORCE, 1);
            float z0, z1, z2, z3;
            box_muller(w.x, w.y, z0, z1);
            box_muller(w.z, w.w, z2, z3);
            const float ms = mass * c_dc.accel_std;
            ft[0] = ms * z0;
            ft[1] = ms * z1;
            ft[2] = ms * z2;
#pragma unroll
            for (int c = 0; c < 3; ++c) S[(ST_FTRIG + c) * P] = __float_as_uint(ft[c]);
            kf = 0;
            acc.n[K_TRIG] += 1;
        } else {
            kf = (kf < 65535u) ? kf + 1u : 65535u;
            if (fresh) {   // materialise the zeroed force of a fresh episode
#pragma unroll
                for (int c = 0; c < 3; ++c) S[(ST_FTRIG + c) * P] = 0u;
            }
        }
        S[ST_KF * P] = kf;
        const double dec = __ldg(p.dec_tab + (kf & 255u)) * __ldg(p.dec_tab + 256u + (kf >> 8));   // L1-resident
#pragma unroll
        for (int c = 0; c < 3; ++c) f[c] = (float)((double)ft[c] * dec);
    }
    acc.m[7] += f[0] * f[0] + f[1] * f[1] + f[2] * f[2];

    // ---- outputs in place over the raw row: [rel 4, tips 15, obj 3 | force 3] ----
    {
        float2* o2 = reinterpret_cast<float2*>(ro);
        o2[0] = make_float2(rel[0], rel[1]);
        o2[1] = make_float2(rel[2], rel[3]);
#pragma unroll
        for (int k = 0; k < 7; ++k) o2[2 + k] = make_float2(tip[2 * k], tip[2 * k + 1]);
        o2[9] = make_float2(tip[14], obj[0]);
        o2[10] = make_float2(obj[1], obj[2]);
        o2[11] = make_float2(f[0], f[1]);
        ro[24] = f[2];
    }
}

// Prefetch policy (DR_PREFETCH env at dr_init): 0 = none, 1 = the current tile at its start,
// 2 = the next tile at the start of the current one (TMA bulk L2 prefetch; A/B experiments).
template <uint32_t L, int PF>
__global__ void __launch_bounds__(STEP_THREADS, STEP_MIN_CTAS)
    step_kernel(const DevPtrs p, const float* __restrict__ actions, const float* __restrict__ raw_obs,
                float* __restrict__ out_actions, float* __restrict__ out_obs, float* __restrict__ out_dt,
                float* __restrict__ out_force, uint32_t n_env) {
    __shared__ __align__(16) float s_act[TILE * N_ACT];   // actions in, out_actions out (in place)
    __shared__ __align__(16) float s_obs[TILE * OBS_IN];  // raw_obs in, out_obs + out_force out (stride 26)
    __shared__ __align__(16) float s_dt[TILE * N_SUB];
    extern __shared__ __align__(16) uint32_t s_ring[];   // [2][RING_W][TILE] (dynamic: > 48 KB total)
    __shared__ int s_last;

    const int tid = threadIdx.x;
    const uint32_t t = (uint32_t)p.ctl[0];
    const uint32_t n_tiles = (n_env + TILE - 1) / TILE;
    constexpr size_t P = PLANE;
    if (PF == 2) prefetch_tile<L>(p, actions, raw_obs, blockIdx.x, n_env);
    Acc acc;
#pragma unroll
    for (int k = 0; k < K_COUNT; ++k) acc.n[k] = 0u;
#pragma unroll
    for (int k = 0; k < 8; ++k) acc.m[k] = 0.f;
    uint32_t my_envs = 0;

    for (uint32_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const uint32_t e0 = tile * TILE;
        const uint32_t cnt = min((uint32_t)TILE, n_env - e0);
        const bool full = cnt == (uint32_t)TILE;
        if (PF == 1) prefetch_tile<L>(p, actions, raw_obs, tile, n_env);
        if (PF == 2) prefetch_tile<L>(p, actions, raw_obs, tile + gridDim.x, n_env);
        __syncthreads();   // previous tile's smem fully stored
        // stage the row-major input tiles (LDGSTS, 16 B per copy for full tiles)
        if (full) {
            const float* a = actions + (size_t)e0 * N_ACT;
            const float* o = raw_obs + (size_t)e0 * OBS_IN;
#pragma unroll
            for (int i = tid; i < TILE * N_ACT / 4; i += STEP_THREADS) cp_async16(s_act + 4 * i, a + 4 * i);
#pragma unroll
            for (int i = tid; i < TILE * OBS_IN / 4; i += STEP_THREADS) cp_async16(s_obs + 4 * i, o + 4 * i);
        } else {
            for (uint32_t i = tid; i < cnt * N_ACT; i += STEP_THREADS) cp_async4(s_act + i, actions + (size_t)e0 * N_ACT + i);
            for (uint32_t i = tid; i < cnt * OBS_IN; i += STEP_THREADS) cp_async4(s_obs + i, raw_obs + (size_t)e0 * OBS_IN + i);
        }
        cp_commit();
        const bool mine = (uint32_t)tid < cnt;
        if (mine) issue_s0<L>(s_ring + tid, p.rec + rec_index(e0 + tid), p.st + st_index(e0 + tid), P);  // S0 -> slot0
        cp_commit();
        if (mine) issue_act<L>(s_ring + RING_W * TILE + tid, p.rec + rec_index(e0 + tid), p.st + st_index(e0 + tid), P, 0);  // A0 -> slot1
        cp_commit();
        cp_wait<1>();      // staging + S0 of this thread
        __syncthreads();   // everyone's staging copies
        if (mine) {
            env_step<L>(p, e0 + tid, t, tid, s_act, s_obs, s_dt, s_ring, acc);
            ++my_envs;
        }
        cp_wait<0>();
        __syncthreads();
        // store the output tiles (coalesced)
        if (full) {
            const float4* s4 = reinterpret_cast<const float4*>(s_act);
            float4* a4 = reinterpret_cast<float4*>(out_actions + (size_t)e0 * N_ACT);
#pragma unroll
            for (int i = tid; i < TILE * N_ACT / 4; i += STEP_THREADS) __stcs(a4 + i, s4[i]);
            const float4* d4s = reinterpret_cast<const float4*>(s_dt);
            float4* d4 = reinterpret_cast<float4*>(out_dt + (size_t)e0 * N_SUB);
#pragma unroll
            for (int i = tid; i < TILE * N_SUB / 4; i += STEP_THREADS) __stcs(d4 + i, d4s[i]);
            // out_obs rows (22 floats = 11 float2) read from stride-26 smem rows
            float2* oo = reinterpret_cast<float2*>(out_obs + (size_t)e0 * OBS_OUT);
            for (int i = tid; i < TILE * 11; i += STEP_THREADS) {
                const int r = i / 11, k = i - r * 11;
                __stcs(oo + i, reinterpret_cast<const float2*>(s_obs + r * OBS_IN)[k]);
            }
            float* of = out_force + (size_t)e0 * 3;
            for (int i = tid; i < TILE * 3; i += STEP_THREADS) {
                const int r = i / 3, k = i - r * 3;
                __stcs(of + i, s_obs[r * OBS_IN + 22 + k]);
            }
        } else {
            for (uint32_t i = tid; i < cnt * N_ACT; i += STEP_THREADS) out_actions[(size_t)e0 * N_ACT + i] = s_act[i];
            for (uint32_t i = tid; i < cnt * N_SUB; i += STEP_THREADS) out_dt[(size_t)e0 * N_SUB + i] = s_dt[i];
            for (uint32_t i = tid; i < cnt * OBS_OUT; i += STEP_THREADS) {
                const uint32_t r = i / OBS_OUT, k = i - r * OBS_OUT;
                out_obs[(size_t)e0 * OBS_OUT + i] = s_obs[r * OBS_IN + k];
            }
            for (uint32_t i = tid; i < cnt * 3; i += STEP_THREADS) {
                const uint32_t r = i / 3, k = i - r * 3;
                out_force[(size_t)e0 * 3 + i] = s_obs[r * OBS_IN + 22 + k];
            }
        }
    }

    // ---- 12. stats: CTA reduction in shared memory, last CTA reduces the partials ----
    __syncthreads();
    double* s_red = reinterpret_cast<double*>(s_obs);   // [N_STATS][STEP_THREADS / 32] (reuses s_obs)
    const int lane = tid & 31, wid = tid >> 5;
    {
        auto red = [&](int i, double x) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xFFFFFFFFu, x, o);
            if (lane == 0) s_red[i * (STEP_THREADS / 32) + wid] = x;
        };
        red(0, (double)my_envs);
        red(1, (double)acc.n[K_DELAYED]);
        red(2, (double)acc.n[K_DROP_INIT]);
        red(3, (double)acc.n[K_MASKED]);
        red(4, (double)acc.n[K_OCCLUDED]);
        red(5, (double)acc.n[K_HELD]);
        red(6, (double)acc.n[K_TRIG]);
        red(7, (double)acc.n[K_RAIL]);
        red(8, (double)acc.n[K_ALPHA1]);
        red(9, on<L>(B_BACKLASH) ? (double)my_envs * N_ACT - (double)acc.n[K_ALPHA1] : 0.0);
        red(10, 0.0);
        red(11, (double)acc.n[K_CLAMPS]);
        red(12, 0.0); red(13, 0.0); red(14, 0.0); red(15, 0.0);
#pragma unroll
        for (int i = 0; i < 8; ++i) red(16 + i, (double)acc.m[i]);
    }
    __syncthreads();
    if (tid < N_STATS) {
        double sum = 0.0;
        if (tid < N_STATS - 8)
#pragma unroll
            for (int w = 0; w < STEP_THREADS / 32; ++w) sum += s_red[tid * (STEP_THREADS / 32) + w];
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
