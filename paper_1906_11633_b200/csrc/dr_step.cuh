// dr_step.cuh -- the fused per-env-step kernel, included by dr_kernels.cu
// inside namespace dr (after on<L>() and the B_* layer bits).
//
// Mapping: persistent CTAs of TILE (= 128) threads, one thread per env, static round-robin tiles
// of 128 envs.  Every byte of state makes one HBM round trip per step.
//
// The per-env record (sector groups, dr_internal.h) and state planes are consumed in seven phases
// -- S0 (scalars), A0..A4 (4 actuators each), OB (observation offsets) -- streamed through a
// two-slot shared-memory ring so that in-flight bytes live in shared memory, not in registers.  A
// warp fills its own 32-env column segment of a slot with 16-byte cp.async.cg (L1 bypass) and
// hands over with __syncwarp, so the four warps of a CTA run their pipelines independently
// (DESIGN.md §8).  Outputs are written in place over the input rows in shared memory (out_actions
// over actions, out_obs + out_force over raw_obs) and stored with coalesced 128/64-bit stores.  Held
// fingertip readings are fetched with per-thread cp.async while the fingertip noise is computed.
// Stats: register accumulators -> CTA shared-memory reduction -> order-free exact fp64 atomics.
#pragma once

// State write-back policy (A/B): 0 = default write-back stores, 1 = streaming (st.global.cs).
#ifndef DR_STATE_CS
#define DR_STATE_CS 0
#endif
__device__ __forceinline__ void st_state(uint32_t* p, uint32_t v) {
#if DR_STATE_CS
    __stcs(p, v);
#else
    *p = v;
#endif
}
// Output store policy (A/B): 1 = streaming (st.global.cs, default), 0 = default write-back.
#ifndef DR_OUT_CS
#define DR_OUT_CS 1
#endif
template <class T>
__device__ __forceinline__ void st_out(T* p, T v) {
#if DR_OUT_CS
    __stcs(p, v);
#else
    *p = v;
#endif
}

enum : int { K_DELAYED = 0, K_DROP_INIT, K_MASKED, K_OCCLUDED, K_HELD, K_TRIG, K_RAIL, K_ALPHA1, K_CLAMPS, K_COUNT };

struct Acc {
    uint32_t n[K_COUNT];
    float m[8];   // a thread sums only its ~n/(grid*TILE) envs in fp32; CTA and grid sums are fp64
};

// ---- phase ring layout ---------------------------------------------------------------------
// A slot is RING_W rows of TILE words, and warp w owns columns 32 w .. 32 w + 31 of every row (the
// four warps of a CTA run their pipelines independently, so no row segment is shared).
//  * A state plane takes one row: thread tid's word at row * TILE + tid (a warp reads 32
//    consecutive words, conflict-free).
//  * A record group (one 32-byte sector per env) takes an 8-row block: env lane l's 8 words sit in
//    row l / 4 of the block at columns 32 w + 8 (l % 4) .. + 7 (group_off), in the order they are
//    stored in HBM, so a sector lands contiguously (one L2 request per sector: a split sector costs
//    a request per half -- measured 4x the L2 read requests and 20 % more step time).  Thread tid
//    reads logical half h with one LDS.128 at chunk h ^ rec_swz (dr_internal.h): within each
//    quarter-warp the eight lanes then hit eight different 16-byte bank groups.
// Record groups are fetched whole (two 16-byte cp.async per env, 512 contiguous bytes per
// instruction); a group whose two halves feed different phases lands in a block that outlives both.
constexpr int RING_W = 24;
constexpr int N_PHASES = 7;   // S0, A0..A4, OB
constexpr size_t STEP_DYN_SMEM = 2 * RING_W * TILE * sizeof(uint32_t);   // 2 slots
// S0 (slot 0): state planes flags (row 0), f_trig (1..3), k_f (4).  Its record words 0..3 (delay
// bits, 1/lambda, force threshold, mass) are half 0 of group 0, which lands in slot 1 block 16 with
// c_act 0..3 (half 1, read by A0).
enum : int { S0_FLAGS = 0, S0_FTRIG = 1, S0_KF = 4 };
// A_b (slot 1 for even b, slot 0 for odd b): rows 0..3 prev, 4..7 slack (state planes), block 8 =
// record group 1 + b (half 0 delta-1, half 1 delta+1 of actuators 4b..4b+3).  c_act quads: A0 slot 1
// block 16 half 1 (group 0); A1 / A2 slot 0 block 16 halves 0 / 1 (group 6, fetched with A1); A3 / A4
// slot 1 block 16 halves 0 / 1 (group 7, fetched with A3).  OB (slot 0): blocks 0, 8, 16 = record
// groups 8, 9, 10 (off_tip 0..14, c_obj 0..2, q_c 0..3, lambda, p-index).
enum : int { A_PREV = 0, A_SLACK = 4, A_BL = 8, BLK16 = 16 };

__device__ __forceinline__ float ringf(const uint32_t* slot, int row, int tid) {
    return __uint_as_float(slot[row * TILE + tid]);
}
// word offset of env lane el's 8-word block inside an 8-row group block (see above)
__device__ __forceinline__ int group_off(int el) { return ((el & 31) >> 2) * TILE + (el & ~31) + 8 * (el & 3); }
// logical half h (0: record words 8g..8g+3, 1: 8g+4..8g+7) of thread tid's env in the group block
__device__ __forceinline__ float4 ringh(const uint32_t* blk, int tid, int h) {
    return *reinterpret_cast<const float4*>(blk + group_off(tid) + 4 * (h ^ (int)(rec_swz((uint32_t)tid) >> 2)));
}
__device__ __forceinline__ float q4(const float4 v, int c) { return c == 0 ? v.x : (c == 1 ? v.y : (c == 2 ? v.z : v.w)); }

__device__ __forceinline__ unsigned ld_acquire_u32(const uint32_t* q) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(q) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u32(uint32_t* q, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(q), "r"(v) : "memory");
}
// Warp-cooperative ring: a warp fills its 32-env column segment of a slot with 16-byte cp.async.cg
// (L1 bypass).  State planes: one instruction moves 4 planes x 128 B (lane l: plane l >> 3, bytes
// 16 (l & 7)).  Record groups: two instructions, each moving the 32-byte groups of 16 envs (512
// contiguous bytes; lane l: env 16 i + l / 2, half l & 1).  Lanes read words other lanes copied, so
// every hand-over is a __syncwarp.  Cross-tile pipelining: the next tile's A0 is issued into slot 1
// once A4 is consumed and its S0 once OB is consumed, so a new tile starts with both phases already
// landed; the input rows are waited for only after the timing section (io_wait).
template <uint32_t L>
struct PipeWarp {
    uint32_t* slot0;   // s_ring (row 0, column 0)
    uint32_t* slot1;
    const uint32_t* Rt;   // record tile block
    const uint32_t* Sw;   // state tile block + this warp's first column
    int tid, lane, wcol;  // wcol = 32 * warp
    const uint32_t* nRt;  // next tile of this CTA (nullptr: none)
    const uint32_t* nSw;
    __device__ __forceinline__ void planes(uint32_t* slot, int row, const uint32_t* src, int n) {
        const int sub = 4 * (lane & 7);
        for (int i = 0; i < n; i += 4) {
            const int pi = i + (lane >> 3);
            if (pi < n) cp_async16(slot + (row + pi) * TILE + wcol + sub, src + pi * TILE + sub);
        }
    }
    // record sector group grp of the warp's 32 envs -> the 8-row block at blk
    __device__ __forceinline__ void group(uint32_t* blk, const uint32_t* R, int grp) {
        const int h = lane & 1;
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const int el = wcol + 16 * i + (lane >> 1);
            cp_async16(blk + group_off(el) + 4 * h, R + (size_t)grp * (TILE * 8) + (size_t)el * 8 + 4 * h);
        }
    }
    __device__ __forceinline__ static uint32_t* row(uint32_t* slot, int r) { return slot + r * TILE; }
    // the group-0 block: S0's record words (half 0) and A0's c_act (half 1)
    __device__ __forceinline__ const uint32_t* g0() const { return slot1 + BLK16 * TILE; }
    // c_act quad of phase b: (block, logical half)
    __device__ __forceinline__ float4 cact(int b) const {
        const uint32_t* blk = (b == 1 || b == 2 ? slot0 : slot1) + BLK16 * TILE;
        return ringh(blk, tid, (b == 1 || b == 3) ? 0 : 1);
    }
    __device__ __forceinline__ void issue_s0_of(const uint32_t* R, const uint32_t* S) {
        if (on<L>(B_TIMING) || on<L>(B_DELAY) || on<L>(B_FORCE) || on<L>(B_ACT_NOISE))
            group(row(slot1, BLK16), R, 0);                                            // S0 quad | c_act 0..3
        if (on<L>(B_FORCE)) planes(slot0, S0_FLAGS, S + ST_FLAGS * TILE, 5);           // state planes 55..59
        else if (on<L>(B_STATEFUL)) planes(slot0, S0_FLAGS, S + ST_FLAGS * TILE, 1);
    }
    __device__ __forceinline__ void issue_act_of(uint32_t* sl, int b, const uint32_t* R, const uint32_t* S) {
        if (on<L>(B_DELAY)) planes(sl, A_PREV, S + (ST_PREV + 4 * b) * TILE, 4);
        if (on<L>(B_BACKLASH)) {
            planes(sl, A_SLACK, S + (ST_SLACK + 4 * b) * TILE, 4);
            group(row(sl, A_BL), R, REC_G_BL + b);
        }
        if (on<L>(B_ACT_NOISE)) {
            if (b == 1) group(row(slot0, BLK16), R, 6);   // c_act 4..7 | 8..11 (A1 | A2)
            if (b == 3) group(row(slot1, BLK16), R, 7);   // c_act 12..15 | 16..19 (A3 | A4)
        }
    }
    __device__ __forceinline__ void issue_s0() { issue_s0_of(Rt, Sw); }
    __device__ __forceinline__ void issue_act(uint32_t* sl, int b) { issue_act_of(sl, b, Rt, Sw); }
    __device__ __forceinline__ void issue_obs(uint32_t* sl) {
        if (on<L>(B_OBS_NOISE)) {
#pragma unroll
            for (int gi = 0; gi < 3; ++gi) group(row(sl, 8 * gi), Rt, REC_OFFTIP / 8 + gi);
        }
    }
    __device__ __forceinline__ const uint32_t* s0() { return slot0; }   // the tile loop waited
    __device__ __forceinline__ void s0_done() {
        __syncwarp();
        issue_act(slot0, 1);
        cp_commit();
    }
    __device__ __forceinline__ void io_wait() {   // the tile's input rows (all but the A1 group just committed)
        cp_wait<1>();
        __syncthreads();
    }
    __device__ __forceinline__ const uint32_t* act(int b) {
        cp_wait<1>();
        __syncwarp();
        return (b & 1) ? slot0 : slot1;
    }
    __device__ __forceinline__ void act_done(int b) {
        uint32_t* sl = (b & 1) ? slot0 : slot1;
        __syncwarp();
        if (b + 2 < 5) issue_act(sl, b + 2);
        else if (b + 2 == 5) issue_obs(sl);
        else if (nRt) issue_act_of(slot1, 0, nRt, nSw);   // b == 4: next tile's A0
        cp_commit();
    }
    // called after the held-reading copies were committed: OB is older than (next A0, held)
    __device__ __forceinline__ const uint32_t* obs() {
        cp_wait<2>();
        __syncwarp();
        return slot0;
    }
    __device__ __forceinline__ void obs_done() {   // next tile's S0 into the slot OB just vacated
        __syncwarp();
        if (nRt) issue_s0_of(nRt, nSw);
        cp_commit();
    }
};

// Backlash gate alpha = 1 - clamp(num / den, 0, 1) with num = |sgn - s|, den = |s' - s| + eps
// (PAPER.md:107).  s' moves from s towards sgn and is clamped on the rail sgn, so |s' - s| <= num:
// the ratio is >= 1 (alpha 0) unless num == 0 (s on the rail already: alpha 1) or s' lands on the
// rail (num < den, den = num + eps): there alpha = 1 - num / (num + eps) = eps / den exactly, which
// costs one MUFU.RCP instead of a full divide.  (fp32 values near +-1 are >= 6e-8 apart, so
// 0 < num < eps, where the identity would not hold, cannot occur.)
__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
// Branch-free (the MUFU.RCP is issued unconditionally; selects instead of divergent branches).
__device__ __forceinline__ float backlash_alpha(float num, float den) {
    const float rail = c_dc.eps * rcp_approx(den);
    const float a = (num < den) ? rail : 0.f;
    return (num == 0.f) ? 1.f : a;
}

// ---- the per-env transform -------------------------------------------------------------------
// valid = false: a lane past n_env in a tail tile (it computes on garbage, stores nothing and
// counts nothing).
template <uint32_t L, class Pipe>
__device__ __forceinline__ void env_step(const DevPtrs& p, uint32_t e, bool valid, uint32_t t, int tid, float* s_act,
                                         float* s_obs, float* s_dt, float* out_sub, Pipe& pipe, Acc& acc) {
    constexpr size_t P = PLANE;
    uint32_t* S = p.st + st_index(e);
    const uint32_t g = c_dc.env_offset + e;
    const uint32_t vm = valid ? 0xFFFFFFFFu : 0u;
    constexpr bool kHold = (L == RUNTIME_MASK) || (L & (B_DROPOUT | B_OCCLUSION));
    const bool hold_layers = on<L>(B_DROPOUT) || on<L>(B_OCCLUSION);

    // simulator occlusion bits: issued first so the byte load overlaps the action phases
    const uint32_t occ_in = (on<L>(B_OCCLUSION) && p.occl_in && valid) ? (uint32_t)__ldg(p.occl_in + e) : 0u;

    // ---- S0: scalars ----
    const uint32_t* s0 = pipe.s0();
    const float4 sq = (on<L>(B_TIMING) || on<L>(B_DELAY) || on<L>(B_FORCE)) ? ringh(pipe.g0(), tid, 0)
                                                                             : make_float4(0.f, 0.f, 0.f, 0.f);
    const float il = on<L>(B_TIMING) ? sq.y : 0.f;
    const uint32_t dbits = on<L>(B_DELAY) ? __float_as_uint(sq.x) : 0u;
    // a FRESH env (reset since its last step) has all-zero state: slack 0, prev 0, no reading,
    // timers 0, force 0 -- the reset kernel does not write the state planes
    const uint32_t flags_raw = on<L>(B_STATEFUL) ? s0[S0_FLAGS * TILE + tid] : 0u;
    const bool fresh = (flags_raw & FRESH_BIT) != 0u;
    const uint32_t flags = (kHold && hold_layers && !fresh) ? flags_raw : 0u;
    uint32_t tf = 0, kf = 0;
    float mass = 0.f, ft[3] = {0.f, 0.f, 0.f};
    if (on<L>(B_FORCE)) {
        tf = __float_as_uint(sq.z);
        mass = sq.w;
        if (!fresh) {
            kf = s0[S0_KF * TILE + tid];
#pragma unroll
            for (int c = 0; c < 3; ++c) ft[c] = ringf(s0, S0_FTRIG + c, tid);
        }
    }
    pipe.s0_done();

    // ---- 1. timing: 10 substeps of 8 ms + Exp(lambda); dt_env = sum [Q2] ----
    // Step-word channel: words 0-9 substeps, 10-14 dropout, 15 force trigger.
    // Block 2 (words 8-11) is shared by timing and dropout; block 3 by dropout and the force.
    float dt_env;
    uint2 w_drop01 = make_uint2(0u, 0u);   // words 10, 11
    {
        float d[N_SUB];
        if (on<L>(B_TIMING)) {
#pragma unroll
            for (int b = 0; b < 3; ++b) {
                const uint4 w = philox(g, t, CH_STEP, b);
                if (b == 2) w_drop01 = make_uint2(w.z, w.w);
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
        acc.m[0] += valid ? dt_env : 0.f;
        acc.m[1] += valid ? dt_env * dt_env : 0.f;
    }

    // ---- 2-4. actions: delay -> noise -> clamp -> backlash [Q1] ----
    acc.n[K_DELAYED] += __popc(dbits) & vm;
    uint32_t n_clamp = 0, n_rail = 0, n_a1 = 0;
    float s_da = 0.f, s_da2 = 0.f, s_bl = 0.f, s_zu2 = 0.f;
    float4* a4p = reinterpret_cast<float4*>(s_act + tid * N_ACT);
    pipe.io_wait();   // the input rows of this tile have landed
#pragma unroll 1
    for (int b = 0; b < 5; ++b) {   // rolled: keeps the kernel inside the instruction cache
        const uint32_t* sl = pipe.act(b);
        float prev[4], slack[4], dneg[4], dpos[4], cact[4];
        const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
        const float4 dn4 = on<L>(B_BACKLASH) ? ringh(sl + A_BL * TILE, tid, 0) : z4;
        const float4 dp4 = on<L>(B_BACKLASH) ? ringh(sl + A_BL * TILE, tid, 1) : z4;
        const float4 ca4 = on<L>(B_ACT_NOISE) ? pipe.cact(b) : z4;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            prev[q] = (on<L>(B_DELAY) && !fresh) ? ringf(sl, A_PREV + q, tid) : 0.f;
            slack[q] = (on<L>(B_BACKLASH) && !fresh) ? ringf(sl, A_SLACK + q, tid) : 0.f;
            dneg[q] = q4(dn4, q);
            dpos[q] = q4(dp4, q);
            cact[q] = q4(ca4, q);
        }
        pipe.act_done(b);

        float ema[4];   // DR_SMOOTH state: direct (coalesced) loads, issued before the normals
        if (on<L>(B_SMOOTH)) {
#pragma unroll
            for (int q = 0; q < 4; ++q) ema[q] = fresh ? 0.f : __uint_as_float(S[(ST_EMA + 4 * b + q) * P]);
        }
        float zu[4], zm[4];
        if (on<L>(B_ACT_NOISE)) {
            normals4_t<kSfuNormals>(philox(g, t, CH_ACT_UADD, b), zu);
            normals4_t<kSfuNormals>(philox(g, t, CH_ACT_MULT, b), zm);
        }
        const float4 a4 = a4p[b];
        const float av[4] = {a4.x, a4.y, a4.z, a4.w};
        float ov[4], anv[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int j = 4 * b + q;
            float a = av[q];
            if (on<L>(B_SMOOTH)) {
                // EMA of the policy action before it is applied [Q25]
                a = c_dc.smooth_keep * ema[q] + c_dc.smooth_c * a;
                if (valid) st_state(&S[(ST_EMA + j) * P], __float_as_uint(a));
            }
            float ad = a;
            if (on<L>(B_DELAY)) {
                // one-step delay of flagged actuators [Q9]
                if ((dbits >> j) & 1u) ad = prev[q];
                if (valid) st_state(&S[(ST_PREV + j) * P], __float_as_uint(a));
            }
            float an = ad;
            if (on<L>(B_ACT_NOISE)) {
                // Table action-noise [Q8]
                an = ad + ad * (c_dc.sm * zm[q]);
                an = an + c_dc.su * zu[q];
                an = an + cact[q];
                n_clamp += (fabsf(an) > 1.f) ? 1u : 0u;
                an = fminf(fmaxf(an, -1.f), 1.f);
                s_zu2 += zu[q] * zu[q];
            }
            const float da = an - ad;
            s_da += da;
            s_da2 += da * da;
            float out = an;
            anv[q] = an;
            if (on<L>(B_BACKLASH) && !on<L>(B_SUBSTEP)) {
                // backlash, verbatim [Q4], sgn(0) = 0 [Q3]:
                // alpha = 1 - clamp(|sgn - s| / (|s' - s| + eps), 0, 1).  The ratio is >= 1 (alpha 0)
                // unless s sits on the rail sgn already (num == 0: alpha 1) or s' lands on the rail
                // within eps of it (num < den, only when num < ~1.7e-5 in fp32): there alpha is a
                // cancellation whose absolute error (<= 2 ulp of 1 with the fast divide) is far
                // inside the 1e-6 budget of alpha * a_n -- so no branch.
                // (an == 0: the product an d dt is 0 whatever d is, so d needs no third case; alpha is 1
                //  exactly when num == 0; a rail hit needs s' != s, which an == 0 cannot give)
                const float s = slack[q];
                const float sg = (an != 0.f) ? copysignf(1.f, an) : 0.f;   // sgn, sgn(0) = 0
                const float d = (an > 0.f) ? dpos[q] : dneg[q];
                const float sp = fminf(fmaxf(s + an * d * dt_env, -1.f), 1.f);
                const float num = fabsf(sg - s), den = fabsf(sp - s) + c_dc.eps;
                const float al = backlash_alpha(num, den);
                out = al * an;
                n_rail += (fabsf(sp) == 1.f && sp != s) ? 1u : 0u;
                n_a1 += (num == 0.f) ? 1u : 0u;
                if (valid) st_state(&S[(ST_SLACK + j) * P], __float_as_uint(sp));
            }
            s_bl += on<L>(B_SUBSTEP) ? 0.f : fabsf(out - an);
            ov[q] = out;
        }
        if (on<L>(B_BACKLASH) && on<L>(B_SUBSTEP)) {
            // per-substep backlash [Q26]: the slack model of PAPER.md:102-109 once per substep k
            // with dt_k, a_n held; out_sub[e][k][4b..4b+3] = alpha_k a_n, out_actions = substep 9
            float sl[4], sg[4], dd[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                sl[q] = slack[q];
                sg[q] = (anv[q] > 0.f) ? 1.f : ((anv[q] < 0.f) ? -1.f : 0.f);
                dd[q] = (anv[q] > 0.f) ? dpos[q] : dneg[q];
            }
            float4* osub = reinterpret_cast<float4*>(out_sub + (size_t)e * (N_SUB * N_ACT) + 4 * b);
#pragma unroll 1
            for (int k = 0; k < N_SUB; ++k) {
                const float dtk = s_dt[tid * N_SUB + k];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const float s0 = sl[q];
                    const float sp = fminf(fmaxf(s0 + anv[q] * dd[q] * dtk, -1.f), 1.f);
                    const float num = fabsf(sg[q] - s0), den = fabsf(sp - s0) + c_dc.eps;
                    const float al = backlash_alpha(num, den);
                    ov[q] = al * anv[q];
                    n_rail += (fabsf(sp) == 1.f && sp != s0) ? 1u : 0u;
                    n_a1 += (num == 0.f) ? 1u : 0u;
                    sl[q] = sp;
                }
                if (valid) __stcs(osub + (size_t)k * (N_ACT / 4), make_float4(ov[0], ov[1], ov[2], ov[3]));
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                s_bl += fabsf(ov[q] - anv[q]);
                if (valid) st_state(&S[(ST_SLACK + 4 * b + q) * P], __float_as_uint(sl[q]));
            }
        }
        a4p[b] = make_float4(ov[0], ov[1], ov[2], ov[3]);
    }
    acc.n[K_CLAMPS] += n_clamp & vm;
    acc.n[K_RAIL] += n_rail & vm;
    acc.n[K_ALPHA1] += n_a1 & vm;
    acc.m[2] += valid ? s_da : 0.f;
    acc.m[3] += valid ? s_da2 : 0.f;
    acc.m[4] += valid ? s_bl : 0.f;
    acc.m[5] += valid ? s_zu2 : 0.f;

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
    if (on<L>(B_OCCLUSION) && p.occl_in) {
        // the simulator's own occlusion bits (its collision-site rule) [Q27]
        occ = occ_in & 0x1Fu;
        acc.n[K_OCCLUDED] += __popc(occ) & vm;
    } else if (on<L>(B_OCCLUSION) && c_dc.occl_on) {
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
                occ |= (d2 < lo) ? pair : 0u;   // selects, no divergent branches
                amb |= (d2 < lo || d2 > hi) ? 0u : 1u << (6 * i + (j - i - 1));
            }
        }
        if (amb | c_dc.occl_exact_only) {
            const double r2 = c_dc.occl_r2;
#pragma unroll
            for (int i = 0; i < N_TIPS; ++i) {
#pragma unroll
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
        acc.n[K_OCCLUDED] += __popc(occ) & vm;
    }
    uint32_t masked = 0;
    uint4 w_step3 = make_uint4(0u, 0u, 0u, 0u);   // step words 12-15 (dropout tips 2-4, force trigger)
    if (kHold && hold_layers) {
        uint32_t nflags = 0, n_init = 0;
        if (on<L>(B_DROPOUT)) {
            // dropout: a 13-step mask starts with probability 1 - exp(-0.2 * 0.08) per step;
            // a retrigger restarts it [Q11]
            if (!on<L>(B_TIMING)) {
                const uint4 w2 = philox(g, t, CH_STEP, 2);
                w_drop01 = make_uint2(w2.z, w2.w);
            }
            w_step3 = philox(g, t, CH_STEP, 3);
            const uint32_t xs[N_TIPS] = {w_drop01.x, w_drop01.y, w_step3.x, w_step3.y, w_step3.z};
#pragma unroll
            for (int i = 0; i < N_TIPS; ++i) {
                const uint32_t x = xs[i];
                uint32_t tm = (flags >> (4 * i)) & 0xFu;
                if ((unsigned long long)x < c_dc.t_drop) { tm = c_dc.hold_steps; ++n_init; }
                if (tm > 0u) { masked |= 1u << i; tm -= 1u; }
                nflags |= tm << (4 * i);
            }
            acc.n[K_MASKED] += __popc(masked) & vm;
            acc.n[K_DROP_INIT] += n_init & vm;
        }
        if (valid) st_state(&S[ST_FLAGS * P], nflags | HAS_LAST_BIT);
    } else if (on<L>(B_STATEFUL) && fresh) {
        if (valid) st_state(&S[ST_FLAGS * P], 0u);   // clear FRESH (no hold layers: timers / has_last unused)
    }
    const uint32_t hold = (flags & HAS_LAST_BIT) ? (masked | occ) : 0u;
    acc.n[K_HELD] += __popc(hold) & vm;
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
    const uint32_t* ob = pipe.obs();   // the observation offsets
    // fingertips: + (correlated + misplacement offset) + 2 mm uncorrelated
    float s_zt = 0.f;
    if (on<L>(B_OBS_NOISE)) {
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            float z[4];
            normals4_t<kSfuNormals>(philox(g, t, CH_TIP_NOISE, b), z);
            const float4 off4 = ringh(ob + 8 * (b >> 1) * TILE, tid, b & 1);   // off_tip 4b..4b+3 (b = 3: 12..14, c_obj 0)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int n = 4 * b + q;
                if (n < 15) {
                    tip[n] = (tip[n] + q4(off4, q)) + c_dc.tip_uncorr * z[q];
                    s_zt += z[q] * z[q];
                }
            }
        }
    }
    acc.m[6] += valid ? s_zt : 0.f;
    cp_wait<0>();   // held readings
    if (kHold && hold_layers) {
#pragma unroll
        for (int i = 0; i < N_TIPS; ++i) {
            if ((hold >> i) & 1u) {
#pragma unroll
                for (int c = 0; c < 3; ++c) tip[3 * i + c] = ro[3 * i + c];   // unchanged: no store
            } else if (valid) {
#pragma unroll
                for (int c = 0; c < 3; ++c) st_state(&S[(ST_LAST + 3 * i + c) * P], __float_as_uint(tip[3 * i + c]));
            }
        }
    }
    // object position: + 5 mm correlated + 1 mm uncorrelated
    if (on<L>(B_OBS_NOISE)) {
        float z[4];
        normals4_t<kSfuNormals>(philox(g, t, CH_OBJ_NOISE, 0), z);
        const float4 c0 = ringh(ob + 8 * TILE, tid, 1), c1 = ringh(ob + 16 * TILE, tid, 0);
        const float co[3] = {c0.w, c1.x, c1.y};
#pragma unroll
        for (int c = 0; c < 3; ++c) obj[c] = (obj[c] + co[c]) + c_dc.obj_uncorr * z[c];
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
            const float4 qa4 = ringh(ob + 16 * TILE, tid, 0), qb4 = ringh(ob + 16 * TILE, tid, 1);   // q_c = words 82..85
            const float qc[4] = {qa4.z, qa4.w, qb4.x, qb4.y};
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
    pipe.obs_done();

    // ---- 10. random force: replace on trigger, decay 0.99 per step in closed form
    //           [Q17, Q18] ----
    float f[3] = {0.f, 0.f, 0.f};
    if (on<L>(B_FORCE)) {
        const uint32_t x = on<L>(B_DROPOUT) ? w_step3.w : philox(g, t, CH_STEP, 3).w;   // step word 15
        if (x < tf) {
            const uint4 w = philox(g, t, CH_FORCE, 1);
            float z0, z1, z2, z3;
            box_muller(w.x, w.y, z0, z1);
            box_muller(w.z, w.w, z2, z3);
            const float ms = mass * c_dc.accel_std;
            ft[0] = ms * z0;
            ft[1] = ms * z1;
            ft[2] = ms * z2;
            if (valid) {
#pragma unroll
                for (int c = 0; c < 3; ++c) st_state(&S[(ST_FTRIG + c) * P], __float_as_uint(ft[c]));
            }
            kf = 0;
            acc.n[K_TRIG] += vm & 1u;
        } else {
            kf = (kf < 65535u) ? kf + 1u : 65535u;
            if (fresh && valid) {   // materialise the zeroed force of a fresh episode
#pragma unroll
                for (int c = 0; c < 3; ++c) st_state(&S[(ST_FTRIG + c) * P], 0u);
            }
        }
        if (valid) st_state(&S[ST_KF * P], kf);
        const double dec = __ldg(p.dec_tab + (kf & 255u)) * __ldg(p.dec_tab + 256u + (kf >> 8));   // L1-resident
#pragma unroll
        for (int c = 0; c < 3; ++c) f[c] = (float)((double)ft[c] * dec);
    }
    acc.m[7] += valid ? f[0] * f[0] + f[1] * f[1] + f[2] * f[2] : 0.f;   // select, not multiply: invalid lanes may hold NaN

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

// ---- tile output store (shared by both kernels) ----
__device__ __forceinline__ void store_tile(uint32_t e0, uint32_t cnt, int tid, const float* s_act, const float* s_obs,
                                           const float* s_dt, float* out_actions, float* out_obs, float* out_dt,
                                           float* out_force) {
    if (cnt == (uint32_t)TILE) {
        const float4* s4 = reinterpret_cast<const float4*>(s_act);
        float4* a4 = reinterpret_cast<float4*>(out_actions + (size_t)e0 * N_ACT);
#pragma unroll
        for (int i = tid; i < TILE * N_ACT / 4; i += STEP_THREADS) st_out(a4 + i, s4[i]);
        const float4* d4s = reinterpret_cast<const float4*>(s_dt);
        float4* d4 = reinterpret_cast<float4*>(out_dt + (size_t)e0 * N_SUB);
#pragma unroll
        for (int i = tid; i < TILE * N_SUB / 4; i += STEP_THREADS) st_out(d4 + i, d4s[i]);
        // out_obs rows (22 floats = 11 float2) read from stride-26 smem rows
        // thread (r0, k) = divmod(tid, 11), tid < 121: each pass stores 11 whole rows (121 float2,
        // contiguous), so the row/column indices only advance -- no division per element
        float2* oo = reinterpret_cast<float2*>(out_obs + (size_t)e0 * OBS_OUT);
        if (tid < 121) {
            const int r0 = tid / 11, k = tid - r0 * 11;
            for (int r = r0; r < TILE; r += 11)
                st_out(oo + r * 11 + k, reinterpret_cast<const float2*>(s_obs + r * OBS_IN)[k]);
        }
        float* of = out_force + (size_t)e0 * 3;
        for (int i = tid; i < TILE * 3; i += STEP_THREADS) {
            const int r = i / 3, k = i - r * 3;
            st_out(of + i, s_obs[r * OBS_IN + 22 + k]);
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

// ---- step index + stats protocol ---------------------------------------------------------
// Every CTA of every step kernel takes a ticket (one atomic on ctl[4]); step t owns the tickets
// [t G, (t + 1) G), G the context's fixed grid, so t = ticket / G.  A CTA takes its ticket before
// it lets the next step launch (griddepcontrol.launch_dependents), and the ticket atomic's result
// is consumed first, so every ticket of step t precedes every ticket of step t + 1 in the atomic's
// coherence order -- no grid-wide barrier and no wait on the previous grid are needed to know t.
// The last CTA of step t publishes t + 1 in ctl[0] (dr_step_index_sync).
// Stats: step t accumulates into slot t % 4.  Its first CTA prepares slot (t + 1) % 4 for step
// t + 1: it waits until every CTA of step t - 3 (the slot's previous owner) has counted itself in
// done[(t + 1) % 4] after its atomics, clears the slot and re-arms the counter, moves the pending
// reset count into slot t % 4, and only then lets the next step launch.  At the end every CTA adds
// its reduced partials into slot t % 4 with fp64 atomics -- counts are small integers and the moment
// sums are rounded per CTA to multiples of a host-chosen power of two, so every partial total is
// exact and the slot does not depend on the order the atomics land in -- then counts itself done.
// chain = 1 (the previous launch on the stream was a step kernel of this context): no
// griddepcontrol.wait -- CTA c works on tiles c, c + G, ... like CTA c of the previous step, so it
// starts as soon as that CTA has finished and published its stores (cta_done[c]), while the
// previous step's other CTAs may still run: consecutive steps overlap at their boundary (a CTA
// that starts early spins in a slot a finished CTA freed); chain = 0 (after a reset, dr_init or
// dr_set_step_index): wait for the previous grid to complete.  Both step kernels chain (the latency
// kernel's CTA c works on 32-env groups c, c + G, ... every step).
#ifdef DR_PROBE_TIMING   // A/B probe only (scripts/probe_timing.py): per-CTA globaltimer stamps over the physics rows
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
    return v;
}
__device__ __forceinline__ unsigned long long* probe_slot(const DevPtrs& p, uint32_t t) {
    return reinterpret_cast<unsigned long long*>(p.phys) + ((size_t)(t % 8u) * gridDim.x + blockIdx.x) * 16;
}
#define DR_PROBE(t, k) probe_slot(p, t)[k] = gtime()
#else
#define DR_PROBE(t, k) (void)0
#endif
#ifndef DR_STEP_EARLY_TRIGGER
#define DR_STEP_EARLY_TRIGGER 0   // A/B knob: unchained steps trigger the next launch after the ticket
#endif
#ifndef DR_POLL_NS
#define DR_POLL_NS 64   // back-off of the chained step's readiness poll (A/B knob; 0 = spin)
#endif
__device__ __forceinline__ uint32_t step_begin(const DevPtrs& p, uint32_t* s_t, int chain) {
#ifdef DR_PROBE_TIMING
    const unsigned long long ts0 = gtime();
#endif
    if (!chain) pdl_wait();   // before any global access (dr_device.cuh)
    if (threadIdx.x == 0) {
        const unsigned long long ticket = atomicAdd(&p.ctl[4], 1ull);
#ifdef DR_PROBE_TIMING
        const unsigned long long ts1 = gtime() + (ticket & 0ull);
#endif
        const uint32_t t = (uint32_t)(ticket / gridDim.x);
        const uint32_t k = (uint32_t)(ticket - (unsigned long long)t * gridDim.x);
        if (k == 0) {
            const uint32_t nslot = (t + 1u) % N_STAT_SLOTS;
            while (ld_acquire_u32(p.done + nslot) != gridDim.x) __nanosleep(128);   // step t - 3 is done with it
            double* nxt = p.stats + nslot * N_STATS;
            for (int i = 0; i < N_STATS; ++i) nxt[i] = 0.0;
            p.done[nslot] = 0u;
            p.stats[(t % N_STAT_SLOTS) * N_STATS + 10] = (double)atomicExch(&p.ctl[2], 0ull);   // resets
            __threadfence();
        }
        if (k == gridDim.x - 1u)
            asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(&p.ctl[0]), "l"((unsigned long long)t + 1ull) : "memory");
        // chained: this CTA works on the same tiles as the same-index CTA of step t - 1 (fixed grid,
        // tile i on CTA i % G); start once that CTA has published its state stores (cta_ready: before
        // its stats atomics, which are not on this step's path)
        if (chain)
            while (ld_acquire_u32(p.cta_ready + blockIdx.x) != t) {
#if DR_POLL_NS > 0
                __nanosleep(DR_POLL_NS);
#endif
            }
        *s_t = t;
#ifdef DR_PROBE_TIMING
        probe_slot(p, t)[0] = ts0;
        probe_slot(p, t)[1] = ts1;
        DR_PROBE(t, 2);
#endif
    }
    __syncthreads();
    if (chain || DR_STEP_EARLY_TRIGGER) pdl_trigger();   // ticket taken (and, for the first CTA, the next slot prepared)
    return *s_t;
}
template <uint32_t L, int NT = STEP_THREADS>
__device__ __forceinline__ void reduce_stats(const DevPtrs& p, const Acc& acc, uint32_t my_envs, uint32_t t,
                                             double* s_red) {
    if (!DR_STEP_EARLY_TRIGGER) pdl_trigger();   // (unchained launches) this CTA's tiles are issued: the next step may launch
    if (threadIdx.x == 0) DR_PROBE(t, 3);
    const int tid = threadIdx.x;
    const int lane = tid & 31, wid = tid >> 5;
    constexpr int NW = NT / 32;
    __syncthreads();
    // every state and output store of this CTA is issued: the same-index CTA of step t + 1 (same
    // tiles) may start now -- the stats atomics below are off its path (their round trip and the
    // fence behind them were ~0.7 us of config 2's 3.9 us step)
    // (st.release.gpu after the CTA barrier: the release is cumulative over the CTA's stores that
    // precede the barrier (PTX memory model), so no extra fence.sc -- measured: the MEMBAR.SC +
    // L1 invalidate it compiled to cost config 2 0.17 us per step)
    if (tid == 0) {
        DR_PROBE(t, 4);
        st_release_u32(p.cta_ready + blockIdx.x, t + 1u);
        DR_PROBE(t, 5);
    }
    {
        // counts: one REDUX.SUM per slot (32-bit integer warp sums, exact); moments: fp64 butterflies
        auto redc = [&](int i, uint32_t x) {
            const uint32_t v = __reduce_add_sync(0xFFFFFFFFu, x);
            if (lane == 0) s_red[i * NW + wid] = (double)v;
            return v;
        };
        auto red = [&](int i, double x) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xFFFFFFFFu, x, o);
            if (lane == 0) s_red[i * NW + wid] = x;
        };
        const uint32_t envs = redc(0, my_envs);
        redc(1, acc.n[K_DELAYED]);
        redc(2, acc.n[K_DROP_INIT]);
        redc(3, acc.n[K_MASKED]);
        redc(4, acc.n[K_OCCLUDED]);
        redc(5, acc.n[K_HELD]);
        redc(6, acc.n[K_TRIG]);
        redc(7, acc.n[K_RAIL]);
        const uint32_t a1 = redc(8, acc.n[K_ALPHA1]);
        if (lane == 0)   // gated actuator-steps (alpha < 1) = actuator-steps - alpha-1 count
            s_red[9 * NW + wid] = on<L>(B_BACKLASH)
                                      ? (double)envs * N_ACT * (on<L>(B_SUBSTEP) ? N_SUB : 1) - (double)a1 : 0.0;
        redc(11, acc.n[K_CLAMPS]);
#pragma unroll
        for (int i = 0; i < 8; ++i) red(16 + i, (double)acc.m[i]);
    }
    __syncthreads();
    if (tid < 24 && tid != 10 && (tid < 12 || tid >= 16)) {
        double sum = 0.0;
#pragma unroll
        for (int w = 0; w < NW; ++w) sum += s_red[tid * NW + w];
        if (tid >= 16) sum = rint(sum * c_dc.mq_scale[tid - 16]) * c_dc.mq_inv[tid - 16];
        if (sum != 0.0) atomicAdd(p.stats + (t % N_STAT_SLOTS) * N_STATS + tid, sum);
    }
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        atomicAdd(p.done + (t % N_STAT_SLOTS), 1u);   // this CTA's atomics into slot t % 4 are in
        // a step never completes before its predecessor (so stream order still means "all done"):
        // this CTA ends only after the same-index CTA of step t - 1 has ended (long since, in practice)
        while (ld_acquire_u32(p.cta_done + blockIdx.x) != t) __nanosleep(64);
        st_release_u32(p.cta_done + blockIdx.x, t + 1u);
        DR_PROBE(t, 6);
    }
}

__device__ __forceinline__ void acc_zero(Acc& acc) {
#pragma unroll
    for (int k = 0; k < K_COUNT; ++k) acc.n[k] = 0u;
#pragma unroll
    for (int k = 0; k < 8; ++k) acc.m[k] = 0.f;
}

// ============================================================================================
// step_kernel_warp: persistent CTAs, the warp-cooperative phase ring, cross-tile pipelining.
// ============================================================================================
template <uint32_t L>
__global__ void __launch_bounds__(STEP_THREADS, STEP_MIN_CTAS)
    step_kernel_warp(const DevPtrs p, const float* __restrict__ actions, const float* __restrict__ raw_obs,
                     float* __restrict__ out_actions, float* __restrict__ out_obs, float* __restrict__ out_dt,
                     float* __restrict__ out_force, float* __restrict__ out_sub, uint32_t n_env, int chain) {
    __shared__ __align__(16) float s_act[TILE * N_ACT];
    __shared__ __align__(16) float s_obs[TILE * OBS_IN];
    __shared__ __align__(16) float s_dt[TILE * N_SUB];
    extern __shared__ __align__(128) uint32_t s_ring[];   // [2][RING_W][TILE]

    const int tid = threadIdx.x, lane = tid & 31, wcol = tid & ~31;
    __shared__ uint32_t s_tstep;
    const uint32_t t = step_begin(p, &s_tstep, chain);
    const uint32_t n_tiles = (n_env + TILE - 1) / TILE;
    Acc acc;
    acc_zero(acc);
    uint32_t my_envs = 0;

    for (uint32_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const uint32_t e0 = tile * TILE;
        const uint32_t cnt = min((uint32_t)TILE, n_env - e0);
        const bool full = cnt == (uint32_t)TILE;
        __syncthreads();   // previous tile's smem fully stored
        const uint32_t ntile = tile + gridDim.x;
        const uint32_t en = ntile * TILE;
        PipeWarp<L> pipe{s_ring, s_ring + RING_W * TILE, p.rec + rec_index(e0), p.st + st_index(e0) + wcol,
                         tid, lane, wcol, ntile < n_tiles ? p.rec + rec_index(en) : nullptr,
                         ntile < n_tiles ? p.st + st_index(en) + wcol : nullptr};
        // S0 / A0 of this tile were issued by the previous tile (on the first tile: here, ahead of
        // the staging group); the staging group is waited for in io_wait(), after timing
        if (tile == blockIdx.x) {
            pipe.issue_s0();
            cp_commit();
            pipe.issue_act(pipe.slot1, 0);
            cp_commit();
        }
        // the row-major input tile -> shared memory (16-byte cp.async)
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
        cp_wait<1>();   // S0 and A0 landed; the staging group may still fly
        __syncwarp();
        const bool mine = (uint32_t)tid < cnt;
        env_step<L>(p, e0 + tid, mine, t, tid, s_act, s_obs, s_dt, out_sub, pipe, acc);
        my_envs += mine ? 1u : 0u;
        cp_wait<1>();   // the next tile's S0 keeps flying through the store
        __syncthreads();
        store_tile(e0, cnt, tid, s_act, s_obs, s_dt, out_actions, out_obs, out_dt, out_force);
    }
    reduce_stats<L>(p, acc, my_envs, t, reinterpret_cast<double*>(s_obs));
}
