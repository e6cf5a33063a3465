// dr_step.cuh -- the fused per-env-step kernel, included by dr_kernels.cu
// inside namespace dr (after on<L>() and the B_* layer bits).
//
// Mapping: persistent CTAs of TILE (= 128) threads, one thread per env, static round-robin tiles
// of 128 envs.  Every byte of state makes one HBM round trip per step.
//
// The per-env record/state planes (AoSoA: a tile's plane is one contiguous 512-B chunk) are
// consumed in seven phases -- S0 (scalars), A0..A4 (4 actuators each), OB (observation offsets)
// -- streamed through a shared-memory ring so that in-flight bytes live in shared memory, not in
// registers.  Two interchangeable pipelines feed the ring:
//   * PipeThread (step_kernel, default): a per-thread 2-slot ring filled with 4-byte cp.async
//     (LDGSTS) -- each thread's pipeline is independent of the other warps'.
//   * PipeTma (step_kernel_tma, DR_PIPE=1): a 3-slot CTA-wide ring filled by TMA bulk copies
//     (cp.async.bulk + mbarrier complete_tx); a slot is refilled two phases ahead by the last
//     warp to release it (smem atomic), so no thread ever blocks to produce; the row-major input
//     tile is also a TMA bulk copy, and the next tile's inputs are issued as soon as the current
//     tile's outputs are stored.  Measured slower (the ring couples the CTA's warps); kept as an
//     A/B alternative and parity-tested.
// Outputs are written in place over the input rows in shared memory (out_actions over actions,
// out_obs + out_force over raw_obs) and stored with coalesced 128/64-bit stores.  Held fingertip
// readings are fetched with per-thread cp.async while the fingertip noise is computed.  Stats:
// register accumulators -> CTA shared-memory reduction -> last-CTA fixed-order fp64 reduction.
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

// ---- mbarrier + TMA bulk-copy helpers (sm_90+ PTX; SASS: SYNCS.* and UBLKCP) --------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(sdst)),
                 "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
// order this thread's generic-proxy shared-memory accesses before subsequent async-proxy (TMA)
// writes to the same buffers (ring / I/O slot reuse)
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

__device__ __forceinline__ void l2_prefetch(const void* ptr, uint32_t bytes) {
    if (bytes >= 16u)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(ptr), "r"(bytes & ~15u) : "memory");
}

// Optional TMA bulk L2 prefetch of a tile's record/state blocks + input rows (DR_PREFETCH; A/B).
// first_item = 2 prefetches only the row-major input rows.
template <uint32_t L>
__device__ __forceinline__ void prefetch_tile(const DevPtrs& p, const float* actions, const float* raw_obs,
                                              uint32_t tile, uint32_t n_env, int first_item = 0) {
    const uint32_t e0 = tile * TILE;
    if (e0 >= n_env) return;
    const uint32_t cnt = min((uint32_t)TILE, n_env - e0);
    for (int item = first_item + (int)threadIdx.x; item < 4; item += blockDim.x) {
        if (item == 0) l2_prefetch(p.rec + rec_index(e0), REC_STEP_PLANES * TILE * 4u);
        else if (item == 1) l2_prefetch(p.st + st_index(e0), (on<L>(B_SMOOTH) ? ST_PLANES : ST_EMA) * TILE * 4u);
        else if (item == 2) l2_prefetch(actions + (size_t)e0 * N_ACT, cnt * N_ACT * 4u);
        else l2_prefetch(raw_obs + (size_t)e0 * OBS_IN, cnt * OBS_IN * 4u);   // rounded down: in bounds
    }
}

// ---- phase ring layout ---------------------------------------------------------------------
// slot row w of thread tid lives at slot[w * TILE + tid]: a warp reads 32 consecutive words
// (conflict-free LDS), and a tile's plane chunk (512 B) maps onto one row.
constexpr int RING_W = 22;
constexpr int N_PHASES = 7;   // S0, A0..A4, OB
constexpr size_t STEP_DYN_SMEM = 2 * RING_W * TILE * sizeof(uint32_t);   // PipeThread: 2 slots
// S0 rows: record planes 0..3 then state planes 55..59 (both contiguous ranges)
enum : int { S0_DELAY = 0, S0_INVLAM = 1, S0_TFORCE = 2, S0_MASS = 3, S0_FLAGS = 4, S0_FTRIG = 5, S0_KF = 8 };
// A_b rows: prev 0..3 | slack 4..7 | dneg 8..11 | dpos 12..15 | cact 16..19 ; OB rows: offtip 0..14 |
// c_obj 15..17 | q_c 18..21 (record planes 64..85)

// -- per-thread 4-byte copies (PipeThread) --
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
template <uint32_t L>
__device__ __forceinline__ void issue_obs(uint32_t* slot, const uint32_t* R, size_t P) {
    if (on<L>(B_OBS_NOISE)) {
#pragma unroll
        for (int w = 0; w < 22; ++w) cp_async4(slot + w * TILE, R + (REC_OFFTIP + w) * P);
    }
}

// -- CTA-wide TMA bulk copies of phase k of a tile (PipeTma): contiguous plane ranges --
template <uint32_t L>
__device__ __forceinline__ uint32_t phase_bytes(int k) {
    constexpr uint32_t C = TILE * 4u;   // one plane chunk
    if (k == 0) {
        uint32_t b = (on<L>(B_TIMING) || on<L>(B_DELAY) || on<L>(B_FORCE)) ? 4 * C : 0u;
        if (on<L>(B_FORCE)) b += 5 * C;
        else if (on<L>(B_STATEFUL)) b += C;
        return b;
    }
    if (k == N_PHASES - 1) return on<L>(B_OBS_NOISE) ? 22 * C : 0u;
    return (on<L>(B_DELAY) ? 4 * C : 0u) + (on<L>(B_BACKLASH) ? 12 * C : 0u) + (on<L>(B_ACT_NOISE) ? 4 * C : 0u);
}
template <uint32_t L>
__device__ __forceinline__ void issue_phase_tma(uint32_t* slot, const uint32_t* Rt, const uint32_t* St, int k,
                                                uint64_t* bar) {
    constexpr uint32_t C = TILE * 4u;
    mbar_arrive_expect_tx(bar, phase_bytes<L>(k));
    if (k == 0) {
        if (on<L>(B_TIMING) || on<L>(B_DELAY) || on<L>(B_FORCE)) tma_load(slot, Rt, 4 * C, bar);   // planes 0..3
        if (on<L>(B_FORCE)) tma_load(slot + S0_FLAGS * TILE, St + ST_FLAGS * TILE, 5 * C, bar);    // 55..59
        else if (on<L>(B_STATEFUL)) tma_load(slot + S0_FLAGS * TILE, St + ST_FLAGS * TILE, C, bar);
    } else if (k == N_PHASES - 1) {
        if (on<L>(B_OBS_NOISE)) tma_load(slot, Rt + REC_OFFTIP * TILE, 22 * C, bar);
    } else {
        const int b = k - 1;
        if (on<L>(B_DELAY)) tma_load(slot, St + (ST_PREV + 4 * b) * TILE, 4 * C, bar);
        if (on<L>(B_BACKLASH)) {
            tma_load(slot + 4 * TILE, St + (ST_SLACK + 4 * b) * TILE, 4 * C, bar);
            tma_load(slot + 8 * TILE, Rt + (REC_DNEG + 4 * b) * TILE, 4 * C, bar);
            tma_load(slot + 12 * TILE, Rt + (REC_DPOS + 4 * b) * TILE, 4 * C, bar);
        }
        if (on<L>(B_ACT_NOISE)) tma_load(slot + 16 * TILE, Rt + (REC_CACT + 4 * b) * TILE, 4 * C, bar);
    }
}

__device__ __forceinline__ float ringf(const uint32_t* slot, int w) { return __uint_as_float(slot[w * TILE]); }

// ---- pipeline policies -----------------------------------------------------------------------
// Per-thread ring (v3-v5): slot0 holds S0, A1, A3, OB; slot1 holds A0, A2, A4.
template <uint32_t L>
struct PipeThread {
    uint32_t* slot0;
    uint32_t* slot1;
    const uint32_t* R;
    const uint32_t* S;
    __device__ __forceinline__ const uint32_t* s0() { return slot0; }   // the tile loop waited for it
    __device__ __forceinline__ void s0_done() {
        issue_act<L>(slot0, R, S, PLANE, 1);
        cp_commit();
    }
    __device__ __forceinline__ void io_wait() {}
    __device__ __forceinline__ const uint32_t* act(int b) {
        cp_wait<1>();
        return (b & 1) ? slot0 : slot1;
    }
    __device__ __forceinline__ void act_done(int b) {
        uint32_t* sl = (b & 1) ? slot0 : slot1;
        if (b + 2 < 5) issue_act<L>(sl, R, S, PLANE, b + 2);
        else if (b + 2 == 5) issue_obs<L>(sl, R, PLANE);
        cp_commit();
    }
    // called after the held-reading copies were committed: wait for everything but them
    __device__ __forceinline__ const uint32_t* obs() {
        cp_wait<1>();
        return slot0;
    }
    __device__ __forceinline__ void obs_done() {}
};

// Warp-cooperative ring (DR_PIPE=2): the same 2-slot layout as PipeThread, but a warp fills its
// 32-env column segment of a slot with 16-byte cp.async.cg (L1 bypass): one instruction moves 4
// planes x 128 B (lane l: plane l >> 3, bytes 16 (l & 7)), i.e. 4x fewer LDGSTS and no L1 lines.
// Lanes read words other lanes copied, so every hand-over is a __syncwarp.
template <uint32_t L, bool XT = false>
struct PipeWarp {
    uint32_t* slot0;   // s_ring (row 0, column 0)
    uint32_t* slot1;
    const uint32_t* Rw;   // record tile block + this warp's first column
    const uint32_t* Sw;   // state tile block + this warp's first column
    int tid, lane, wcol;  // wcol = 32 * warp
    // XT (cross-tile pipelining): the next tile's A0 is issued into slot1 once A4 is consumed and its
    // S0 into slot0 once OB is consumed, so a new tile starts with both phases already landed; the
    // input rows are then waited for only after the timing section (io_wait).
    const uint32_t* nRw;  // next tile of this CTA (nullptr: none)
    const uint32_t* nSw;
    __device__ __forceinline__ void planes(uint32_t* slot, int row, const uint32_t* src, int n) {
        const int sub = 4 * (lane & 7);
        for (int i = 0; i < n; i += 4) {
            const int pi = i + (lane >> 3);
            if (pi < n) cp_async16(slot + (row + pi) * TILE + wcol + sub, src + pi * TILE + sub);
        }
    }
    __device__ __forceinline__ void issue_s0_of(const uint32_t* R, const uint32_t* S) {
        if (on<L>(B_TIMING) || on<L>(B_DELAY) || on<L>(B_FORCE)) planes(slot0, 0, R, 4);   // record planes 0..3
        if (on<L>(B_FORCE)) planes(slot0, S0_FLAGS, S + ST_FLAGS * TILE, 5);                // state planes 55..59
        else if (on<L>(B_STATEFUL)) planes(slot0, S0_FLAGS, S + ST_FLAGS * TILE, 1);
    }
    __device__ __forceinline__ void issue_act_of(uint32_t* sl, int b, const uint32_t* R, const uint32_t* S) {
        if (on<L>(B_DELAY)) planes(sl, 0, S + (ST_PREV + 4 * b) * TILE, 4);
        if (on<L>(B_BACKLASH)) {
            planes(sl, 4, S + (ST_SLACK + 4 * b) * TILE, 4);
            planes(sl, 8, R + (REC_DNEG + 4 * b) * TILE, 4);
            planes(sl, 12, R + (REC_DPOS + 4 * b) * TILE, 4);
        }
        if (on<L>(B_ACT_NOISE)) planes(sl, 16, R + (REC_CACT + 4 * b) * TILE, 4);
    }
    __device__ __forceinline__ void issue_s0() { issue_s0_of(Rw, Sw); }
    __device__ __forceinline__ void issue_act(uint32_t* sl, int b) { issue_act_of(sl, b, Rw, Sw); }
    __device__ __forceinline__ void issue_obs(uint32_t* sl) {
        if (on<L>(B_OBS_NOISE)) planes(sl, 0, Rw + REC_OFFTIP * TILE, 22);
    }
    __device__ __forceinline__ const uint32_t* s0() { return slot0 + tid; }   // the tile loop waited
    __device__ __forceinline__ void s0_done() {
        __syncwarp();
        issue_act(slot0, 1);
        cp_commit();
    }
    __device__ __forceinline__ void io_wait() {
        if constexpr (XT) {   // the tile's input rows (all but the A1 group just committed)
            cp_wait<1>();
            __syncthreads();
        }
    }
    __device__ __forceinline__ const uint32_t* act(int b) {
        cp_wait<1>();
        __syncwarp();
        return ((b & 1) ? slot0 : slot1) + tid;
    }
    __device__ __forceinline__ void act_done(int b) {
        uint32_t* sl = (b & 1) ? slot0 : slot1;
        __syncwarp();
        if (b + 2 < 5) issue_act(sl, b + 2);
        else if (b + 2 == 5) issue_obs(sl);
        else if (XT && nRw) issue_act_of(slot1, 0, nRw, nSw);   // b == 4: next tile's A0
        cp_commit();
    }
    // called after the held-reading copies were committed: OB is older than (next A0, held)
    __device__ __forceinline__ const uint32_t* obs() {
        cp_wait<XT ? 2 : 1>();
        __syncwarp();
        return slot0 + tid;
    }
    __device__ __forceinline__ void obs_done() {
        if constexpr (XT) {   // next tile's S0 into the slot OB just vacated
            __syncwarp();
            if (nRw) issue_s0_of(nRw, nSw);
            cp_commit();
        }
    }
};

// CTA-wide TMA ring: phase ph (counted over this CTA's tiles) lives in slot ph % NS.
constexpr int TMA_SLOTS = 3;
struct TmaShared {
    uint64_t full[TMA_SLOTS];
    uint64_t io_full;
    uint32_t rel[TMA_SLOTS];   // warps that released the slot's current phase
    uint32_t io_rel;
};

template <uint32_t L>
__device__ __forceinline__ void tma_issue_phase(const DevPtrs& p, uint32_t* ring, TmaShared* ts, uint32_t ph,
                                                uint32_t n_my, uint32_t n_tiles) {
    const uint32_t it = ph / N_PHASES, k = ph % N_PHASES;
    if (it >= n_my) return;
    const uint32_t tile = blockIdx.x + it * gridDim.x;
    if (tile >= n_tiles) return;
    const uint32_t e0 = tile * TILE;
    issue_phase_tma<L>(ring + (ph % TMA_SLOTS) * (RING_W * TILE), p.rec + rec_index(e0), p.st + st_index(e0), (int)k,
                       &ts->full[ph % TMA_SLOTS]);
}

template <uint32_t L>
struct PipeTma {
    const DevPtrs* p;
    uint32_t* ring;
    TmaShared* ts;
    uint32_t ph0;   // global phase index of this tile's S0
    uint32_t it;    // tile iteration (I/O parity)
    uint32_t n_my, n_tiles;
    int tid;
    __device__ __forceinline__ const uint32_t* wait(uint32_t ph) {
        mbar_wait(&ts->full[ph % TMA_SLOTS], (ph / TMA_SLOTS) & 1u);
        return ring + (ph % TMA_SLOTS) * (RING_W * TILE) + tid;
    }
    // the last of the 4 warps to release phase ph refills its slot with phase ph + NS
    __device__ __forceinline__ void release(uint32_t ph) {
        __syncwarp();
        if ((tid & 31) == 0) {
            const uint32_t s = ph % TMA_SLOTS;
            if (atomicAdd(&ts->rel[s], 1u) == (uint32_t)(TILE / 32) - 1u) {
                ts->rel[s] = 0u;
                fence_proxy_async();
                tma_issue_phase<L>(*p, ring, ts, ph + TMA_SLOTS, n_my, n_tiles);
            }
        }
    }
    __device__ __forceinline__ const uint32_t* s0() { return wait(ph0); }
    __device__ __forceinline__ void s0_done() { release(ph0); }
    __device__ __forceinline__ void io_wait() { mbar_wait(&ts->io_full, it & 1u); }
    __device__ __forceinline__ const uint32_t* act(int b) { return wait(ph0 + 1 + b); }
    __device__ __forceinline__ void act_done(int b) { release(ph0 + 1 + b); }
    __device__ __forceinline__ const uint32_t* obs() { return wait(ph0 + N_PHASES - 1); }
    __device__ __forceinline__ void obs_done() { release(ph0 + N_PHASES - 1); }
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
// valid = false only for the lanes past n_env in the tail tile of the TMA kernel: they follow the
// same path (the ring protocol is warp-synchronous) but store nothing and count nothing.
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
    const float il = on<L>(B_TIMING) ? ringf(s0, S0_INVLAM) : 0.f;
    const uint32_t dbits = on<L>(B_DELAY) ? s0[S0_DELAY * TILE] : 0u;
    // a FRESH env (reset since its last step) has all-zero state: slack 0, prev 0, no reading,
    // timers 0, force 0 -- the reset kernel does not write the state planes
    const uint32_t flags_raw = on<L>(B_STATEFUL) ? s0[S0_FLAGS * TILE] : 0u;
    const bool fresh = (flags_raw & FRESH_BIT) != 0u;
    const uint32_t flags = (kHold && hold_layers && !fresh) ? flags_raw : 0u;
    uint32_t tf = 0, kf = 0;
    float mass = 0.f, ft[3] = {0.f, 0.f, 0.f};
    if (on<L>(B_FORCE)) {
        tf = s0[S0_TFORCE * TILE];
        mass = ringf(s0, S0_MASS);
        if (!fresh) {
            kf = s0[S0_KF * TILE];
#pragma unroll
            for (int c = 0; c < 3; ++c) ft[c] = ringf(s0, S0_FTRIG + c);
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
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            prev[q] = (on<L>(B_DELAY) && !fresh) ? ringf(sl, q) : 0.f;
            slack[q] = (on<L>(B_BACKLASH) && !fresh) ? ringf(sl, 4 + q) : 0.f;
            dneg[q] = on<L>(B_BACKLASH) ? ringf(sl, 8 + q) : 0.f;
            dpos[q] = on<L>(B_BACKLASH) ? ringf(sl, 12 + q) : 0.f;
            cact[q] = on<L>(B_ACT_NOISE) ? ringf(sl, 16 + q) : 0.f;
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
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int n = 4 * b + q;
                if (n < 15) {
                    tip[n] = (tip[n] + ringf(ob, n)) + c_dc.tip_uncorr * z[q];
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
#pragma unroll
        for (int c = 0; c < 3; ++c) obj[c] = (obj[c] + ringf(ob, 15 + c)) + c_dc.obj_uncorr * z[c];
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
            const float qc[4] = {ringf(ob, 18), ringf(ob, 19), ringf(ob, 20), ringf(ob, 21)};
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

// ---- step index + stats protocol (no grid-wide tail) ----------------------------------------
// step_begin: thread 0 reads the step index t and counts its CTA in with an acq_rel atomic; the
// last CTA to start advances ctl[0] to t + 1 (every CTA read t before counting in) and re-arms the
// counter.  CTA 0 also clears stats slot (t + 1) % 4 for the next step (its all-reduce, from step
// t - 3, finished before this step was enqueued: parallel.StatsReducer) and moves the pending reset
// count into slot t % 4.  At the end every CTA adds its reduced partials into slot t % 4 with fp64
// atomics -- counts are small integers and the moment sums are rounded per CTA to multiples of a
// host-chosen power of two, so every partial total is exact and the slot does not depend on the
// order the atomics land in (deterministic, and identical to a fixed-order sum of the rounded CTA
// sums).  No fence, no last-CTA pass: the kernel ends when its last tile is stored.
__device__ __forceinline__ uint32_t step_begin(const DevPtrs& p, uint32_t* s_t) {
    pdl_wait();   // before any global access (dr_device.cuh)
    if (threadIdx.x == 0) {
        const uint32_t t = (uint32_t)*(volatile unsigned long long*)&p.ctl[0];
        unsigned long long prev;
        asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], 1;" : "=l"(prev) : "l"(&p.ctl[1]) : "memory");
        if (prev == (unsigned long long)gridDim.x - 1ull) {
            p.ctl[1] = 0ull;
            *(volatile unsigned long long*)&p.ctl[0] = (unsigned long long)t + 1ull;
        }
        if (blockIdx.x == 0) {
            double* nxt = p.stats + ((t + 1u) % N_STAT_SLOTS) * N_STATS;
            for (int i = 0; i < N_STATS; ++i) nxt[i] = 0.0;
            p.stats[(t % N_STAT_SLOTS) * N_STATS + 10] = (double)atomicExch(&p.ctl[2], 0ull);   // resets
        }
        *s_t = t;
    }
    __syncthreads();
    return *s_t;
}

template <uint32_t L, int NT = STEP_THREADS>
__device__ __forceinline__ void reduce_stats(const DevPtrs& p, const Acc& acc, uint32_t my_envs, uint32_t t,
                                             double* s_red) {
    pdl_trigger();   // this CTA's tiles are issued: the next step may launch (dr_device.cuh)
    const int tid = threadIdx.x;
    const int lane = tid & 31, wid = tid >> 5;
    constexpr int NW = NT / 32;
    __syncthreads();
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
}

__device__ __forceinline__ void acc_zero(Acc& acc) {
#pragma unroll
    for (int k = 0; k < K_COUNT; ++k) acc.n[k] = 0u;
#pragma unroll
    for (int k = 0; k < 8; ++k) acc.m[k] = 0.f;
}

// ============================================================================================
// Kernel A (PipeThread): per-thread cp.async ring.  Prefetch policy (DR_PREFETCH): 0 = none,
// 1 = TMA L2 prefetch of the current tile, 2 = of the next tile (A/B experiments).
// ============================================================================================
template <uint32_t L, int PF>
__global__ void __launch_bounds__(STEP_THREADS, STEP_MIN_CTAS)
    step_kernel(const DevPtrs p, const float* __restrict__ actions, const float* __restrict__ raw_obs,
                float* __restrict__ out_actions, float* __restrict__ out_obs, float* __restrict__ out_dt,
                float* __restrict__ out_force, float* __restrict__ out_sub, uint32_t n_env) {
    __shared__ __align__(16) float s_act[TILE * N_ACT];   // actions in, out_actions out (in place)
    __shared__ __align__(16) float s_obs[TILE * OBS_IN];  // raw_obs in, out_obs + out_force out (stride 26)
    __shared__ __align__(16) float s_dt[TILE * N_SUB];
    extern __shared__ __align__(128) uint32_t s_ring[];   // [2][RING_W][TILE] (dynamic: > 48 KB total)

    const int tid = threadIdx.x;
    __shared__ uint32_t s_tstep;
    const uint32_t t = step_begin(p, &s_tstep);
    const uint32_t n_tiles = (n_env + TILE - 1) / TILE;
    constexpr size_t P = PLANE;
    if (PF == 2) prefetch_tile<L>(p, actions, raw_obs, blockIdx.x, n_env);
    Acc acc;
    acc_zero(acc);
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
        const uint32_t* R = p.rec + rec_index(e0 + tid);
        const uint32_t* S = p.st + st_index(e0 + tid);
        if (mine) issue_s0<L>(s_ring + tid, R, S, P);                          // S0 -> slot0
        cp_commit();
        if (mine) issue_act<L>(s_ring + RING_W * TILE + tid, R, S, P, 0);      // A0 -> slot1
        cp_commit();
        cp_wait<1>();      // staging + S0 of this thread
        __syncthreads();   // everyone's staging copies
        if (mine) {
            PipeThread<L> pipe{s_ring + tid, s_ring + RING_W * TILE + tid, R, S};
            env_step<L>(p, e0 + tid, true, t, tid, s_act, s_obs, s_dt, out_sub, pipe, acc);
            ++my_envs;
        }
        cp_wait<0>();
        __syncthreads();
        store_tile(e0, cnt, tid, s_act, s_obs, s_dt, out_actions, out_obs, out_dt, out_force);
    }
    reduce_stats<L>(p, acc, my_envs, t, reinterpret_cast<double*>(s_obs));
}

// ============================================================================================
// Kernel B (PipeTma, default): CTA-wide TMA ring of TMA_SLOTS phase slots + TMA input tiles.
// ============================================================================================
constexpr size_t STEP_TMA_DYN_SMEM = (size_t)TMA_SLOTS * RING_W * TILE * sizeof(uint32_t);

template <uint32_t L>
__device__ __forceinline__ void tma_issue_io(const float* actions, const float* raw_obs, float* s_act, float* s_obs,
                                             TmaShared* ts, uint32_t it, uint32_t n_my, uint32_t n_env) {
    if (it >= n_my) return;
    const uint32_t tile = blockIdx.x + it * gridDim.x;
    const uint32_t e0 = tile * TILE;
    const uint32_t cnt = min((uint32_t)TILE, n_env - e0);
    const uint32_t ba = cnt * N_ACT * 4u;             // multiple of 16
    const uint32_t bo = (cnt * OBS_IN * 4u) & ~15u;   // odd tail: the last 8 bytes are loaded by hand
    mbar_arrive_expect_tx(&ts->io_full, ba + bo);
    tma_load(s_act, actions + (size_t)e0 * N_ACT, ba, &ts->io_full);
    tma_load(s_obs, raw_obs + (size_t)e0 * OBS_IN, bo, &ts->io_full);
}

template <uint32_t L>
__global__ void __launch_bounds__(STEP_THREADS, STEP_MIN_CTAS)
    step_kernel_tma(const DevPtrs p, const float* __restrict__ actions, const float* __restrict__ raw_obs,
                    float* __restrict__ out_actions, float* __restrict__ out_obs, float* __restrict__ out_dt,
                    float* __restrict__ out_force, float* __restrict__ out_sub, uint32_t n_env) {
    __shared__ __align__(128) float s_act[TILE * N_ACT];   // TMA destination; out_actions in place
    __shared__ __align__(128) float s_obs[TILE * OBS_IN];  // TMA destination; out_obs + out_force in place
    __shared__ __align__(16) float s_dt[TILE * N_SUB];
    __shared__ TmaShared ts;
    extern __shared__ __align__(128) uint32_t s_ring[];    // [TMA_SLOTS][RING_W][TILE]

    const int tid = threadIdx.x;
    __shared__ uint32_t s_tstep;
    const uint32_t t = step_begin(p, &s_tstep);
    const uint32_t n_tiles = (n_env + TILE - 1) / TILE;
    const uint32_t n_my = (blockIdx.x < n_tiles) ? (n_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0u;
    if (tid == 0) {
#pragma unroll
        for (int s = 0; s < TMA_SLOTS; ++s) {
            mbar_init(&ts.full[s], 1);
            ts.rel[s] = 0u;
        }
        mbar_init(&ts.io_full, 1);
        ts.io_rel = 0u;
        fence_mbar_init();
    }
    __syncthreads();
    if (tid == 0) {
        for (uint32_t ph = 0; ph < (uint32_t)TMA_SLOTS; ++ph) tma_issue_phase<L>(p, s_ring, &ts, ph, n_my, n_tiles);
        tma_issue_io<L>(actions, raw_obs, s_act, s_obs, &ts, 0, n_my, n_env);
    }
    Acc acc;
    acc_zero(acc);
    uint32_t my_envs = 0;

    for (uint32_t it = 0; it < n_my; ++it) {
        const uint32_t tile = blockIdx.x + it * gridDim.x;
        const uint32_t e0 = tile * TILE;
        const uint32_t cnt = min((uint32_t)TILE, n_env - e0);
        const bool mine = (uint32_t)tid < cnt;
        if ((cnt & 1u) && tid == (int)cnt - 1) {
            // odd tail tile: the TMA copy was rounded down to 16 B; this env's last 2 words by hand
            mbar_wait(&ts.io_full, it & 1u);
            const float2 v = *reinterpret_cast<const float2*>(raw_obs + (size_t)(e0 + cnt) * OBS_IN - 2);
            *reinterpret_cast<float2*>(s_obs + cnt * OBS_IN - 2) = v;
        }
        PipeTma<L> pipe{&p, s_ring, &ts, it * N_PHASES, it, n_my, n_tiles, tid};
        env_step<L>(p, e0 + tid, mine, t, tid, s_act, s_obs, s_dt, out_sub, pipe, acc);
        my_envs += mine ? 1u : 0u;
        __syncthreads();   // all output rows are in shared memory
        store_tile(e0, cnt, tid, s_act, s_obs, s_dt, out_actions, out_obs, out_dt, out_force);
        // the last warp done storing issues the next tile's input rows into the same buffers
        __syncwarp();
        if ((tid & 31) == 0 && atomicAdd(&ts.io_rel, 1u) == (uint32_t)(STEP_THREADS / 32) - 1u) {
            ts.io_rel = 0u;
            fence_proxy_async();
            tma_issue_io<L>(actions, raw_obs, s_act, s_obs, &ts, it + 1, n_my, n_env);
        }
    }
    reduce_stats<L>(p, acc, my_envs, t, reinterpret_cast<double*>(s_dt));
}

// ============================================================================================
// Kernel C (PipeWarp, DR_PIPE=2): warp-cooperative 16-byte cp.async.cg ring.
// ============================================================================================
template <uint32_t L, int WPF, bool XT>
__global__ void __launch_bounds__(STEP_THREADS, STEP_MIN_CTAS)
    step_kernel_warp(const DevPtrs p, const float* __restrict__ actions, const float* __restrict__ raw_obs,
                     float* __restrict__ out_actions, float* __restrict__ out_obs, float* __restrict__ out_dt,
                     float* __restrict__ out_force, float* __restrict__ out_sub, uint32_t n_env) {
    __shared__ __align__(16) float s_act[TILE * N_ACT];
    __shared__ __align__(16) float s_obs[TILE * OBS_IN];
    __shared__ __align__(16) float s_dt[TILE * N_SUB];
    extern __shared__ __align__(128) uint32_t s_ring[];   // [2][RING_W][TILE]

    const int tid = threadIdx.x, lane = tid & 31, wcol = tid & ~31;
    __shared__ uint32_t s_tstep;
    const uint32_t t = step_begin(p, &s_tstep);
    const uint32_t n_tiles = (n_env + TILE - 1) / TILE;
    Acc acc;
    acc_zero(acc);
    uint32_t my_envs = 0;

    for (uint32_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const uint32_t e0 = tile * TILE;
        const uint32_t cnt = min((uint32_t)TILE, n_env - e0);
        const bool full = cnt == (uint32_t)TILE;
        // WPF (A/B): TMA L2 prefetch of the next tile's input rows (1) or of everything it reads (2)
        if (WPF) prefetch_tile<L>(p, actions, raw_obs, tile + gridDim.x, n_env, WPF == 1 ? 2 : 0);
        __syncthreads();   // previous tile's smem fully stored
        auto stage = [&]() {   // the row-major input tile -> shared memory (16-byte cp.async)
            if (full) {
                const float* a = actions + (size_t)e0 * N_ACT;
                const float* o = raw_obs + (size_t)e0 * OBS_IN;
#pragma unroll
                for (int i = tid; i < TILE * N_ACT / 4; i += STEP_THREADS) cp_async16(s_act + 4 * i, a + 4 * i);
#pragma unroll
                for (int i = tid; i < TILE * OBS_IN / 4; i += STEP_THREADS) cp_async16(s_obs + 4 * i, o + 4 * i);
            } else {
                for (uint32_t i = tid; i < cnt * N_ACT; i += STEP_THREADS)
                    cp_async4(s_act + i, actions + (size_t)e0 * N_ACT + i);
                for (uint32_t i = tid; i < cnt * OBS_IN; i += STEP_THREADS)
                    cp_async4(s_obs + i, raw_obs + (size_t)e0 * OBS_IN + i);
            }
            cp_commit();
        };
        const uint32_t ntile = tile + gridDim.x;
        const uint32_t en = ntile * TILE;
        PipeWarp<L, XT> pipe{s_ring, s_ring + RING_W * TILE, p.rec + rec_index(e0) + wcol, p.st + st_index(e0) + wcol,
                             tid, lane, wcol, (XT && ntile < n_tiles) ? p.rec + rec_index(en) + wcol : nullptr,
                             (XT && ntile < n_tiles) ? p.st + st_index(en) + wcol : nullptr};
        if (XT) {
            // S0 / A0 of this tile were issued by the previous tile (on the first tile: here, ahead
            // of the staging group); the staging group is waited for in io_wait(), after timing
            if (tile == blockIdx.x) {
                pipe.issue_s0();
                cp_commit();
                pipe.issue_act(pipe.slot1, 0);
                cp_commit();
            }
            stage();
            cp_wait<1>();   // S0 and A0 landed; the staging group may still fly
            __syncwarp();
        } else {
            stage();
            pipe.issue_s0();                   // S0 -> slot0 (this warp's columns)
            cp_commit();
            pipe.issue_act(pipe.slot1, 0);     // A0 -> slot1
            cp_commit();
            cp_wait<1>();      // staging + S0
            __syncthreads();   // everyone's staging copies (and each warp's S0)
        }
        const bool mine = (uint32_t)tid < cnt;
        env_step<L>(p, e0 + tid, mine, t, tid, s_act, s_obs, s_dt, out_sub, pipe, acc);
        my_envs += mine ? 1u : 0u;
        cp_wait<XT ? 1 : 0>();   // XT: the next tile's S0 keeps flying through the store
        __syncthreads();
        store_tile(e0, cnt, tid, s_act, s_obs, s_dt, out_actions, out_obs, out_dt, out_force);
    }
    reduce_stats<L>(p, acc, my_envs, t, reinterpret_cast<double*>(s_obs));
}
