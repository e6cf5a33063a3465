// dr_reset.cuh -- episode-reset sampling (PAPER.md:7-8, 13, 15-18, 36-41, 77-78, 87-88, 100-101,
// 113), included by dr_kernels.cu inside namespace dr.
//
// reset_kernel: each CTA scans its interleaved 32-env chunks of the mask (one coalesced 32-byte
// load and a ballot per warp and chunk), appends the resetting envs (and their next episode index)
// to a shared-memory list, then
//   * three threads per resetting env draw its episode record in three independent parts and write
//     it as 12 whole 32-byte sectors (one 256-bit store per record group, dr_internal.h): the
//     record of an env is written in full, so L2 never read-fills a partially written sector from
//     DRAM (the AoSoA record of round 1 wrote one 4-byte word into each of 89 sectors per reset
//     env: 4.5x the algorithmic DRAM bytes);
//   * one warp per resetting env (pulled from a shared counter) writes its physics row: lane l
//     draws uniform and normal Philox block l together into the warp's draw buffer (draw-major:
//     draw j of block b at word 64 j + b, rs_slot), then evaluates parameters 8 l .. 8 l + 7 and
//     writes them with one 256-bit store (a warp writes its row as 1 KB of contiguous memory).
// The 60 state planes are not zeroed: one word (FRESH_BIT in the flags plane) marks the env and the
// step kernel reads a fresh env's state as zero (dr_internal.h).
#pragma once

// per-warp draw buffer: uniforms at [0, 256), normals at [256, 512) (both draw-major, rs_slot), a
// constant 0 at 512 (the x of draw-free descriptors); rs_src holds, per parameter, the buffer offset
// of its x | RS_EXP.
constexpr int RH_DRAW = 2 * MAX_PHYS + 4;
// CTA shape: 256 threads, <= 64 registers (4 CTAs per SM).  Scan schedule: CTA c owns the 32-env
// mask chunks c, c + G, c + 2 G, ... (G = the grid) and scans up to RH_PASS envs of them into one
// shared-memory list per pass -- at 1M envs one pass of ~1,771 envs per CTA.  Measured against the
// round-1/2 schedule of 512-env ranges handed out grid-stride (3.46 ranges per CTA: four barrier
// rounds and a 4-vs-3.46 tail), config 5 reset ms per launch (three alternating runs): ranges
// 0.0952, passes of 512 / 1,024 / 2,048 envs 0.0949 / 0.0920 / 0.0887 (kept).
#ifndef DR_RH_THREADS
#define DR_RH_THREADS 256
#endif
#ifndef DR_RH_MINB
#define DR_RH_MINB 4   // __launch_bounds__ min CTAs per SM (<= 64 registers)
#endif
constexpr int RH_THREADS = DR_RH_THREADS;
#ifndef DR_RH_PASS
#define DR_RH_PASS 2048
#endif
constexpr uint32_t RH_PASS = DR_RH_PASS;
#ifndef DR_RESET_EARLY_TRIGGER
#define DR_RESET_EARLY_TRIGGER 0   // A/B knob: trigger the next launch at the start, not at the end
#endif   // envs scanned per pass (the shared-memory list's capacity)

__device__ __forceinline__ float sel4(const float z[4], uint32_t r) {
    return r == 0u ? z[0] : (r == 1u ? z[1] : (r == 2u ? z[2] : z[3]));
}
__device__ __forceinline__ uint32_t selw(const uint4 w, uint32_t r) {
    return r == 0u ? w.x : (r == 1u ? w.y : (r == 2u ? w.z : w.w));
}

// One record group (8 words = one DRAM sector of one env) in one 256-bit store, its halves swapped
// for the envs rec_swz says.
__device__ __forceinline__ void st_group(uint32_t* R, uint32_t e, int grp, uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t a4, uint32_t a5, uint32_t a6, uint32_t a7) {
    uint32_t* q = R + (size_t)grp * (TILE * 8);
    // selects instead of a divergent branch (the lanes of a warp hold envs with either swap):
    // reset 0.0840 -> 0.0830 ms
    const bool sw = rec_swz(e) != 0u;
    const uint32_t b0 = sw ? a4 : a0, b1 = sw ? a5 : a1, b2 = sw ? a6 : a2, b3 = sw ? a7 : a3;
    const uint32_t b4 = sw ? a0 : a4, b5 = sw ? a1 : a5, b6 = sw ? a2 : a6, b7 = sw ? a3 : a7;
    asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(q), "r"(b0), "r"(b1), "r"(b2),
                 "r"(b3), "r"(b4), "r"(b5), "r"(b6), "r"(b7)
                 : "memory");
}
__device__ __forceinline__ uint32_t fu(float x) { return __float_as_uint(x); }

// Four normals of block b of a reset channel (normal n = 4 b + (0..3)).  One out-of-line copy
// serves every call site: ~15 inlined copies of the Philox block + two Box-Muller pairs were most
// of the kernel's code (4,360 -> 2,080 SASS instructions; time unchanged).
__device__ __noinline__ float4 normals4_block(uint32_t g, uint32_t k, uint32_t ch, uint32_t b) {
    const uint4 w = philox(g, k, ch, b);
    float4 z;
    box_muller(w.x, w.y, z.x, z.y);
    box_muller(w.z, w.w, z.z, z.w);
    return z;
}
// Eight normals of two blocks (block b1 of channel ch1, block b2 of channel ch2): the two Philox
// chains are independent, so their rounds interleave (twice the ILP of two normals4_block calls).
struct Normals8 {
    float4 a, b;
};
__device__ __noinline__ Normals8 normals8_block(uint32_t g, uint32_t k, uint32_t ch1, uint32_t b1, uint32_t ch2,
                                                uint32_t b2) {
    const uint4 w1 = philox(g, k, ch1, b1);
    const uint4 w2 = philox(g, k, ch2, b2);
    Normals8 z;
    box_muller(w1.x, w1.y, z.a.x, z.a.y);
    box_muller(w1.z, w1.w, z.a.z, z.a.w);
    box_muller(w2.x, w2.y, z.b.x, z.b.y);
    box_muller(w2.z, w2.w, z.b.z, z.b.w);
    return z;
}
// Physics draws of block b: 4 uniforms of PHYS_U block b (a) and 4 normals of PHYS_N block b (b).
__device__ __forceinline__ Normals8 phys_pair_block(uint32_t g, uint32_t k, uint32_t b) {
    const uint4 wu = philox(g, k, CH_PHYS_U, b);
    const uint4 wn = philox(g, k, CH_PHYS_N, b);
    Normals8 z;
    z.a = make_float4(uni(wu.x), uni(wu.y), uni(wu.z), uni(wu.w));
    box_muller(wn.x, wn.y, z.b.x, z.b.y);
    box_muller(wn.z, wn.w, z.b.z, z.b.w);
    return z;
}
__device__ __forceinline__ void reset_normals8(bool on, uint32_t g, uint32_t k, uint32_t ch1, uint32_t b1, uint32_t ch2,
                                               uint32_t b2, float z1[4], float z2[4]) {
#pragma unroll
    for (int q = 0; q < 4; ++q) z1[q] = z2[q] = 0.f;
    if (on) {
        const Normals8 v = normals8_block(g, k, ch1, b1, ch2, b2);
        z1[0] = v.a.x; z1[1] = v.a.y; z1[2] = v.a.z; z1[3] = v.a.w;
        z2[0] = v.b.x; z2[1] = v.b.y; z2[2] = v.b.z; z2[3] = v.b.w;
    }
}
// ... zero when the layer is off.
__device__ __forceinline__ void reset_normals4(bool on, uint32_t g, uint32_t k, uint32_t ch, uint32_t b, float z[4]) {
    z[0] = z[1] = z[2] = z[3] = 0.f;
    if (on) {
        const float4 v = normals4_block(g, k, ch, b);
        z[0] = v.x;
        z[1] = v.y;
        z[2] = v.z;
        z[3] = v.w;
    }
}

// Physics tables in shared memory, transposed for the row evaluation: lane l writes parameters
// 8 l .. 8 l + 7 of a row (one 256-bit store), so parameter q lives at [q % 8][q / 8] (s_pd) and the
// draw sources of lane l's quad h at [h][l] (s_src4): every LDS.128 of a warp is conflict-free.
__device__ __forceinline__ int pd_slot(int q) { return (q & 7) * 32 + (q >> 3); }
__device__ __forceinline__ void stage_phys_tables(const DevPtrs& p, float4* s_pd, uint32_t* s_src, int tid, int nthr) {
    for (int q = tid; q < MAX_PHYS; q += nthr) {   // padded: draw-free zero entries past n_phys
        const bool live = q < c_dc.n_phys;
        s_pd[pd_slot(q)] = live ? p.rs_phys[q] : make_float4(0.f, 0.f, 0.f, 0.f);
        s_src[(((q & 7) >> 2) * 32 + (q >> 3)) * 4 + (q & 3)] = live ? p.rs_src[q] : RS_OFF_ZERO;
    }
}

// The object mass phys[mass_index] [Q18], recomputed by the record thread so that record group 0
// is written whole (same draw, coefficients and operations as reset_phys_warp: bit-identical).
__device__ __forceinline__ float reset_mass(uint32_t g, uint32_t k, const float4* s_pd, const uint32_t* s_src) {
    const int mi = c_dc.mass_index;
    const float4 d = s_pd[pd_slot(mi)];
    const uint32_t o = s_src[(((mi & 7) >> 2) * 32 + (mi >> 3)) * 4 + (mi & 3)], off = o & ~RS_EXP;
    float x = 0.f;
    // buffer slot j * 64 + b (rs_slot) -> draw j of Philox block b
    if (off < RS_OFF_NORMAL) {                       // uniform-kind parameter u: word u % 4 of block u / 4
        x = uni(selw(philox(g, k, CH_PHYS_U, off & 63u), off >> 6));
    } else if (off < RS_OFF_ZERO) {                  // normal-kind parameter n: normal n % 4 of block n / 4
        const uint32_t sl = off - RS_OFF_NORMAL, n = ((sl & 63u) << 2) | (sl >> 6);
        const uint4 w = philox(g, k, CH_PHYS_N, n >> 2);
        float z0, z1;
        if (n & 2u) box_muller(w.z, w.w, z0, z1);
        else box_muller(w.x, w.y, z0, z1);
        x = (n & 1u) ? z1 : z0;
    }
    const float tv = fmaf(d.y, x, d.x);
    return fmaf(d.w, (o & RS_EXP) ? ex2_approx(tv) : tv, d.z);
}

// The episode record of env e for episode k (oracle: reset_env, steps 2-9), in three independent
// parts so three threads share one env's serial chain (each ~a third of the Philox blocks and
// Box-Muller pairs); every part writes whole record groups:
//   part 0: group 0 (delay flags, 1/lambda, force threshold, mass, c_act 0..3), groups 6-7 (c_act
//           4..19), group 11 (episode counter) and the FRESH flag;
//   part 1: groups 1-5 (backlash widths);
//   part 2: groups 8-10 (observation offsets; lambda and p-index, drawn again, ride in group 10).
__device__ void reset_record_part(const DevPtrs& p, uint32_t e, uint32_t k, int part, const float4* s_pd,
                                  const uint32_t* s_src) {
    const uint32_t lm = c_dc.layer_mask;
    uint32_t* R = p.rec + rec_index(e);
    const uint32_t g = c_dc.env_offset + e;
    const float sc = c_dc.sc;   // correlated action noise, Table action-noise
    float lam = 0.f, il = 0.f;   // timing coefficient lambda ~ U[1250, 10000]
    uint32_t jp = 0u;            // loguniform force probability [Q19]: index
    if (part != 1) {
        if (lm & B_TIMING) {
            lam = c_dc.lam_lo + c_dc.lam_range * uni(philox(g, k, CH_LAMBDA, 0).x);
            il = 1.0f / lam;
        }
        jp = (lm & B_FORCE) ? (philox(g, k, CH_FORCE_P, 0).x >> 16) : 0u;
    }
    if (part == 0) {
        uint32_t bits = 0u;   // per-actuator delay flags, Bernoulli(0.5) per episode
        if (lm & B_DELAY) {
#pragma unroll
            for (int b = 0; b < 5; ++b) {
                const uint4 w = philox(g, k, CH_DELAY, b);
                const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                for (int q = 0; q < 4; ++q) bits |= ((unsigned long long)ws[q] < c_dc.t_delay ? 1u : 0u) << (4 * b + q);
            }
        }
        const uint32_t tf = (lm & B_FORCE) ? __ldg(p.t_tab + jp) : 0u;   // exact integer threshold
        const float mass = reset_mass(g, k, s_pd, s_src);
        {
            float z[4];
            reset_normals4(lm & B_ACT_NOISE, g, k, CH_CORR_ACT, 0, z);
            st_group(R, e, 0, bits, fu(il), tf, fu(mass), fu(sc * z[0]), fu(sc * z[1]), fu(sc * z[2]), fu(sc * z[3]));
        }
#pragma unroll 1
        for (int b = 1; b < 5; b += 2) {   // groups 6..7: c_act 4..11, 12..19
            float z0[4], z1[4];
            reset_normals8(lm & B_ACT_NOISE, g, k, CH_CORR_ACT, b, CH_CORR_ACT, b + 1, z0, z1);
            st_group(R, e, 6 + (b >> 1), fu(sc * z0[0]), fu(sc * z0[1]), fu(sc * z0[2]), fu(sc * z0[3]), fu(sc * z1[0]),
                     fu(sc * z1[1]), fu(sc * z1[2]), fu(sc * z1[3]));
        }
        st_group(R, e, 11, k, 0u, 0u, 0u, 0u, 0u, 0u, 0u);
        p.st[st_index(e) + ST_FLAGS * PLANE] = FRESH_BIT;   // state reads as zero at the next step [Q6, Q9]
    } else if (part == 1) {
        // backlash widths of actuators 4b..4b+3 [Q7]: normal j -> delta-1_j
        // (block j / 4), normal 20 + j -> delta+1_j (block 5 + j / 4)
#pragma unroll 1
        for (int b = 0; b < 5; ++b) {
            float zn[4], zp[4], dn[4], dp[4];
            reset_normals8(lm & B_BACKLASH, g, k, CH_BACKLASH, b, CH_BACKLASH, 5 + b, zn, zp);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int j = 4 * b + q;
                dn[q] = (lm & B_BACKLASH) ? fmaxf(0.f, c_dc.dcal_neg[j] + c_dc.jitter * zn[q]) : 0.f;
                dp[q] = (lm & B_BACKLASH) ? fmaxf(0.f, c_dc.dcal_pos[j] + c_dc.jitter * zp[q]) : 0.f;
            }
            st_group(R, e, REC_G_BL + b, fu(dn[0]), fu(dn[1]), fu(dn[2]), fu(dn[3]), fu(dp[0]), fu(dp[1]), fu(dp[2]),
                     fu(dp[3]));
        }
    } else {
        // observation offsets [Q14, Q15]
        float off[16], co[4], qc[4] = {1.f, 0.f, 0.f, 0.f};
        const bool obs = (lm & B_OBS_NOISE) != 0;
        float mb[4];
        reset_normals8(obs, g, k, CH_MARKER_BASE, 0, CH_CORR_OBJ, 0, mb, co);
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            float zc[4], zm[4];
            reset_normals8(obs, g, k, CH_CORR_TIP, b, CH_MARKER_TIP, b, zc, zm);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int n = 4 * b + q;
                float v = c_dc.tip_corr * zc[q] + c_dc.tip_marker * zm[q];
                if (c_dc.base_to_tips) v = v - c_dc.base_marker * mb[n % 3];
                off[n] = obs ? v : 0.f;
            }
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) co[c] = obs ? c_dc.obj_corr * co[c] : 0.f;
        if (obs) rotation(c_dc.rot_corr, philox(g, k, CH_CORR_ROT, 0), qc);
        st_group(R, e, 8, fu(off[0]), fu(off[1]), fu(off[2]), fu(off[3]), fu(off[4]), fu(off[5]), fu(off[6]), fu(off[7]));
        st_group(R, e, 9, fu(off[8]), fu(off[9]), fu(off[10]), fu(off[11]), fu(off[12]), fu(off[13]), fu(off[14]), fu(co[0]));
        st_group(R, e, 10, fu(co[1]), fu(co[2]), fu(qc[0]), fu(qc[1]), fu(qc[2]), fu(qc[3]), fu(lam), jp);
    }
}

// The physics row of env e for episode k [Q20]: v = C0 + C1 f(A + B x),
// f = 2^(.) for the exp kinds (the host folds log2(e) into A and B: one MUFU.EX2).  Lanes draw the
// env's Philox blocks into the warp's draw buffer, then lane l evaluates parameters 8 l .. 8 l + 7
// (tables padded to 256 with draw-free zero entries) and writes them with one 256-bit store.
__device__ __forceinline__ void reset_phys_warp(const DevPtrs& p, uint32_t e, uint32_t k, int lane, float* dr,
                                                const float4* s_pd, const uint32_t* s_src, int nub, int nnb) {
    const uint32_t g = c_dc.env_offset + e;
    __syncwarp();
    // uniform-kind parameter u uses word u % 4 of block u / 4 (channel PHYS_U); normal-kind
    // parameter n uses normal n % 4 of block n / 4 (channel PHYS_N).  Lane l draws uniform block b and
    // normal block b (b = l, l + 32) together: two independent Philox chains interleave.
    // Draw j of block b sits at buffer word rs_slot(4 b + j) = j * 64 + b (dr_internal.h), so the
    // evaluation's reads -- lane l mostly needs draws 4 l .. 4 l + 3 -- hit 32 different banks
    // (the block-contiguous layout made them 4-way bank conflicts).
    const int nb = max(nub, nnb);
    for (int b = lane; b < nb; b += 32) {
        float4 zu = make_float4(0.f, 0.f, 0.f, 0.f), zn = zu;
        if (b < nub && b < nnb) {
            const Normals8 v = phys_pair_block(g, k, (uint32_t)b);
            zu = v.a;
            zn = v.b;
        } else if (b < nub) {
            const uint4 w = philox(g, k, CH_PHYS_U, (uint32_t)b);
            zu = make_float4(uni(w.x), uni(w.y), uni(w.z), uni(w.w));
        } else {
            zn = normals4_block(g, k, CH_PHYS_N, (uint32_t)b);
        }
        if (b < nub) {
            dr[b] = zu.x; dr[64 + b] = zu.y; dr[128 + b] = zu.z; dr[192 + b] = zu.w;
        }
        if (b < nnb) {
            float* q = dr + MAX_PHYS;
            q[b] = zn.x; q[64 + b] = zn.y; q[128 + b] = zn.z; q[192 + b] = zn.w;
        }
    }
    __syncwarp();
    const int np = c_dc.n_phys;
    if (8 * lane >= np) return;
    const uint4* src4 = reinterpret_cast<const uint4*>(s_src);
    float v[8];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const uint4 o4 = src4[h * 32 + lane];
        const uint32_t os[4] = {o4.x, o4.y, o4.z, o4.w};
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const float4 d = s_pd[(4 * h + c) * 32 + lane];   // (A, B, C0, C1)
            const float x = dr[os[c] & ~RS_EXP];
            const float tv = fmaf(d.y, x, d.x);
            v[4 * h + c] = fmaf(d.w, (os[c] & RS_EXP) ? ex2_approx(tv) : tv, d.z);
        }
    }
    float* prow = p.phys + (size_t)e * np + 8 * lane;
    if ((np & 7) == 0) {   // rows 32-byte aligned (np % 8 == 0): one 256-bit store per lane
        asm volatile("st.global.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(prow), "f"(v[0]), "f"(v[1]),
                     "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
                     : "memory");
    } else {
#pragma unroll
        for (int c = 0; c < 8; ++c)
            if (8 * lane + c < np) prow[c] = v[c];
    }
}

#ifdef DR_PROBE_TIMING   // A/B probe only (scripts/probe_reset_timing.py): per-CTA globaltimer stamps and SM id
__device__ unsigned long long g_probe_reset[4096][8];
__device__ __forceinline__ unsigned long long rgtime() {
    unsigned long long v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
    return v;
}
#define RPROBE(k) do { if (threadIdx.x == 0 && blockIdx.x < 4096) g_probe_reset[blockIdx.x][k] = rgtime(); } while (0)
#else
#define RPROBE(k) (void)0
#endif
// early_scan != 0 (the host saw the previous libdr launch on the stream is a step kernel, which
// writes neither masks nor episode counters nor the physics tables): the first pass's table staging
// and mask scan run before griddepcontrol.wait, overlapping the step's tail; every write (records,
// physics rows, FRESH flags) still follows the wait.  Otherwise (e.g. two resets back to back: the
// previous one wrote the episode counters) the wait comes first.
__global__ void __launch_bounds__(RH_THREADS, DR_RH_MINB) reset_kernel(DevPtrs p, const uint8_t* __restrict__ mask, int first,
                                                              uint32_t n_env, int early_scan) {
    __shared__ float4 s_pd[MAX_PHYS];           // transposed: parameter q at pd_slot(q)
    __shared__ __align__(16) uint32_t s_src[MAX_PHYS];   // transposed: lane l's quad h at [(h * 32 + l) * 4]
    __shared__ uint32_t s_env[1][RH_PASS];
    __shared__ uint32_t s_kk[1][RH_PASS];    // episode counter k - 1 (0xFFFFFFFF on the first reset)
    __shared__ __align__(16) float s_dr[RH_THREADS / 32][RH_DRAW];
    __shared__ uint32_t s_n[1], s_next[1];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    RPROBE(0);
#ifdef DR_PROBE_TIMING
    if (threadIdx.x == 0 && blockIdx.x < 4096) {
        uint32_t smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        g_probe_reset[blockIdx.x][6] = smid;
    }
#endif
    bool waited = !early_scan;
    if (DR_RESET_EARLY_TRIGGER) pdl_trigger();
    if (waited) pdl_wait();   // before any global access (dr_device.cuh)
    RPROBE(1);
    constexpr int NWR = RH_THREADS / 32;
    static_assert(RH_PASS % (32 * NWR) == 0, "pass = whole chunks per warp");
    stage_phys_tables(p, s_pd, s_src, tid, RH_THREADS);
    if (lane == 0) s_dr[wid][RS_OFF_ZERO] = 0.f;
    const bool phys_on = (c_dc.layer_mask & B_PHYS) != 0;
    const int nub = phys_on ? (c_dc.n_phys_u + 3) / 4 : 0;
    const int nnb = phys_on ? (c_dc.n_phys_n + 3) / 4 : 0;
    uint32_t applied = 0;
    // the record chains first: part p of env i on thread p * npad + i (whole warps per part, so no
    // warp mixes code paths); then every warp pulls physics rows from a shared counter, so the
    // warps without a record chunk start on them at once and the rows spread over all warps
    auto work = [&](int sl, uint32_t n, uint32_t* next) {
        const uint32_t npad = (n + 31u) & ~31u;
        for (uint32_t ti = tid; ti < 3u * npad; ti += RH_THREADS) {
            const uint32_t part = ti / npad, i = ti - part * npad;
            if (i < n) reset_record_part(p, s_env[sl][i], s_kk[sl][i] + 1u, (int)part, s_pd, s_src);
        }
        for (;;) {
            uint32_t i = 0;
            if (lane == 0) i = atomicAdd(next, 1u);
            i = __shfl_sync(0xFFFFFFFFu, i, 0);
            if (i >= n) break;
            reset_phys_warp(p, s_env[sl][i], s_kk[sl][i] + 1u, lane, s_dr[wid], s_pd, s_src, nub, nnb);
        }
    };
    // interleaved 32-env chunks: CTA c owns chunks c, c + G, c + 2 G, ... (G = gridDim.x), scanned
    // RH_PASS / 32 at a time into one shared-memory list: one barrier round per pass and, for any
    // mask that is uniform at the scale of G chunks, the same number of resets in every CTA
    {
        constexpr uint32_t PASS_CH = RH_PASS / 32;
        constexpr int NCH1 = PASS_CH / NWR;
        const uint32_t nch = (n_env + 31u) / 32u, G = gridDim.x;
        const uint32_t my = (nch > blockIdx.x) ? (nch - blockIdx.x + G - 1u) / G : 0u;
        for (uint32_t j0 = 0; j0 < my; j0 += PASS_CH) {
            if (tid == 0) {
                s_n[0] = 0u;
                s_next[0] = 0u;
            }
            __syncthreads();
            uint32_t mk1[NCH1], ee[NCH1];
#pragma unroll
            for (int jj = 0; jj < NCH1; ++jj) {
                const uint32_t j = j0 + (uint32_t)(wid + NWR * jj);
                ee[jj] = (blockIdx.x + G * j) * 32u + lane;
                mk1[jj] = (j < my && ee[jj] < n_env) ? (mask == nullptr ? 1u : (uint32_t)mask[ee[jj]]) : 0u;
            }
#pragma unroll
            for (int jj = 0; jj < NCH1; ++jj) {
                const bool m = mk1[jj] != 0u;
                const uint32_t bal = __ballot_sync(0xFFFFFFFFu, m);
                if (!bal) continue;
                uint32_t pos0 = 0;
                if (lane == 0) pos0 = atomicAdd(&s_n[0], (uint32_t)__popc(bal));
                pos0 = __shfl_sync(0xFFFFFFFFu, pos0, 0);
                if (m) {
                    const uint32_t idx = pos0 + __popc(bal & ((1u << lane) - 1u));
                    const uint32_t e = ee[jj];
                    s_env[0][idx] = e;
                    if (first) s_kk[0][idx] = 0xFFFFFFFFu;
                    else cp_async4(&s_kk[0][idx], p.rec + rec_index(e) + rec_off(e, REC_EPISODE));
                }
                applied += (lane == 0) ? (uint32_t)__popc(bal) : 0u;
            }
            cp_commit();
            cp_wait<0>();
            __syncthreads();
            if (!waited) {   // the first pass's reads are done: now the previous kernel must be complete
                pdl_wait();
                waited = true;
            }
            RPROBE(2);
            work(0, s_n[0], &s_next[0]);
#ifdef DR_PROBE_TIMING
            if ((threadIdx.x & 31) == 0 && blockIdx.x < 4096) {
                atomicMax(&g_probe_reset[blockIdx.x][4], rgtime());   // last warp done
                atomicMin(&g_probe_reset[blockIdx.x][5], rgtime());   // first warp done
            }
#endif
            __syncthreads();
            RPROBE(3);
        }
    }
    if (!waited) pdl_wait();   // (a CTA without a pass) before the global atomic below
    if (!DR_RESET_EARLY_TRIGGER) pdl_trigger();
    if (!first && applied) atomicAdd(&p.ctl[2], (unsigned long long)applied);
}
