// dr_step_lat.cuh -- latency-mode step kernel, included by dr_kernels.cu after
// dr_step.cuh inside namespace dr.
//
// The throughput kernel (step_kernel_warp) runs one thread per env through the whole ~4k
// instruction transform; with few envs (4,096 - 131,072 per job) a step is then as long as one
// thread's serial chain.  Here one CTA of 8 warps serves 32 envs (one env per lane) and every warp
// runs one part of the transform for all 32:
//   warps 0-4  actuator group b = warp (4 actuators: smoothing, delay, noise, clamp, backlash)
//   warp  5    substep timing and the remaining step words (dropout tips, force trigger)
//   warp  6    fingertips (occlusion, dropout timers, noise, hold-last-reading)
//   warp  7    object position, orientation -> relative goal, random force
// Each warp loads its own state planes straight from HBM/L2 (coalesced 128-byte lines: one env per
// lane) and its record words as 16/32-byte vectors of its env's sector groups (dr_internal.h)
// and the one cross-warp dependency -- dt_env and the step words of warp 5 -- goes through shared
// memory behind a single CTA barrier (role_barrier).  The arithmetic of every output is the same expression,
// in the same order, as env_step's (so the same oracle parity contract holds).
#pragma once

constexpr int LAT_THREADS = 256;
constexpr int LAT_ENVS = 32;
#ifndef DR_LAT_MIN_CTAS
#define DR_LAT_MIN_CTAS 2   // __launch_bounds__ occupancy target (A/B: 3 or 4 spill and run slower)
#endif

// The warp roles meet at one CTA barrier per group, reached from a different call site in each
// role: the non-.aligned barrier.sync (all threads of a warp take the same site; sites differ across
// warps), not __syncthreads (barrier.sync.aligned requires every thread of the CTA at the same
// instruction -- compute-sanitizer synccheck flags it).
__device__ __forceinline__ void role_barrier() { asm volatile("barrier.sync 0;" ::: "memory"); }

template <uint32_t L>
__global__ void __launch_bounds__(LAT_THREADS, DR_LAT_MIN_CTAS) step_kernel_lat(const DevPtrs p, const float* __restrict__ actions,
                                                               const float* __restrict__ raw_obs,
                                                               float* __restrict__ out_actions,
                                                               float* __restrict__ out_obs, float* __restrict__ out_dt,
                                                               float* __restrict__ out_force, float* __restrict__ out_sub,
                                                               uint32_t n_env, int chain) {
    __shared__ float s_dtenv[LAT_ENVS];
    __shared__ float s_dtk[N_SUB][LAT_ENVS];
    __shared__ uint32_t s_wd[6][LAT_ENVS];   // step words 10-15
    __shared__ double s_red[N_STATS * (LAT_THREADS / 32)];

    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    __shared__ uint32_t s_tstep;
    const uint32_t t = step_begin(p, &s_tstep, chain);   // CTA g works on groups g, g + G, ... every step
    constexpr size_t P = PLANE;
    constexpr bool kHold = (L == RUNTIME_MASK) || (L & (B_DROPOUT | B_OCCLUSION));
    const bool hold_layers = on<L>(B_DROPOUT) || on<L>(B_OCCLUSION);
    Acc acc;
    acc_zero(acc);
    uint32_t my_envs = 0;
    const uint32_t n_groups = (n_env + LAT_ENVS - 1) / LAT_ENVS;

    for (uint32_t grp = blockIdx.x; grp < n_groups; grp += gridDim.x) {
        const uint32_t e = grp * LAT_ENVS + (uint32_t)lane;
        const bool valid = e < n_env;
        const uint32_t ec = valid ? e : n_env - 1u;   // tail lanes compute on a real env, store nothing
        const uint32_t* R = p.rec + rec_index(ec);
        uint32_t* S = p.st + st_index(ec);
        const uint32_t g = c_dc.env_offset + ec;
        const uint32_t vm = valid ? 0xFFFFFFFFu : 0u;
        const uint32_t flags_raw = on<L>(B_STATEFUL) ? S[ST_FLAGS * P] : 0u;
        const bool fresh = (flags_raw & FRESH_BIT) != 0u;
        const uint32_t flags = (kHold && hold_layers && !fresh) ? flags_raw : 0u;
        __syncthreads();   // every warp read the flags word before warp 6 may rewrite it; smem reuse

        if (wid < 5) {
            // ================= actuators 4b .. 4b+3 [Q1] =================
            const int b = wid;
            const uint32_t dbits = on<L>(B_DELAY) ? R[rec_off(ec, REC_DELAY)] : 0u;
            float prev[4], slack[4], dneg[4], dpos[4], cact[4], ema[4];
            const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
            const float4* Rq = reinterpret_cast<const float4*>(R);
            const float4 dn4 = on<L>(B_BACKLASH) ? Rq[rec_off(ec, rec_dneg(4 * b)) / 4] : z4;   // record group 1 + b
            const float4 dp4 = on<L>(B_BACKLASH) ? Rq[rec_off(ec, rec_dpos(4 * b)) / 4] : z4;
            const float4 ca4 = on<L>(B_ACT_NOISE) ? Rq[rec_off(ec, rec_cact(4 * b)) / 4] : z4;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int j = 4 * b + q;
                prev[q] = (on<L>(B_DELAY) && !fresh) ? __uint_as_float(S[(ST_PREV + j) * P]) : 0.f;
                slack[q] = (on<L>(B_BACKLASH) && !fresh) ? __uint_as_float(S[(ST_SLACK + j) * P]) : 0.f;
                dneg[q] = q4(dn4, q);
                dpos[q] = q4(dp4, q);
                cact[q] = q4(ca4, q);
                ema[q] = (on<L>(B_SMOOTH) && !fresh) ? __uint_as_float(S[(ST_EMA + j) * P]) : 0.f;
            }
            const float4 a4 = __ldg(reinterpret_cast<const float4*>(actions + (size_t)ec * N_ACT) + b);
            float zu[4], zm[4];
            if (on<L>(B_ACT_NOISE)) {
                normals4_t<kSfuNormals>(philox(g, t, CH_ACT_UADD, b), zu);
                normals4_t<kSfuNormals>(philox(g, t, CH_ACT_MULT, b), zm);
            }
            if (b == 0) acc.n[K_DELAYED] += __popc(dbits) & vm;
            uint32_t n_clamp = 0, n_rail = 0, n_a1 = 0;
            float s_da = 0.f, s_da2 = 0.f, s_bl = 0.f, s_zu2 = 0.f;
            const float av[4] = {a4.x, a4.y, a4.z, a4.w};
            float anv[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int j = 4 * b + q;
                float a = av[q];
                if (on<L>(B_SMOOTH)) {
                    a = c_dc.smooth_keep * ema[q] + c_dc.smooth_c * a;   // [Q25]
                    if (valid) st_state(&S[(ST_EMA + j) * P], __float_as_uint(a));
                }
                float ad = a;
                if (on<L>(B_DELAY)) {
                    if ((dbits >> j) & 1u) ad = prev[q];                 // [Q9]
                    if (valid) st_state(&S[(ST_PREV + j) * P], __float_as_uint(a));
                }
                float an = ad;
                if (on<L>(B_ACT_NOISE)) {                                // [Q8]
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
                anv[q] = an;
            }
            role_barrier();   // dt_env / dt_k of warp 5
            float ov[4];
            if (on<L>(B_BACKLASH) && !on<L>(B_SUBSTEP)) {
                const float dt_env = s_dtenv[lane];
#pragma unroll
                for (int q = 0; q < 4; ++q) {                            // [Q3, Q4]
                    const float an = anv[q], s = slack[q];
                    const float sg = (an != 0.f) ? copysignf(1.f, an) : 0.f;   // sgn, sgn(0) = 0
                    const float d = (an > 0.f) ? dpos[q] : dneg[q];
                    const float sp = fminf(fmaxf(s + an * d * dt_env, -1.f), 1.f);
                    const float num = fabsf(sg - s), den = fabsf(sp - s) + c_dc.eps;
                    const float al = backlash_alpha(num, den);
                    ov[q] = al * an;
                    n_rail += (fabsf(sp) == 1.f && sp != s) ? 1u : 0u;
                    n_a1 += (num == 0.f) ? 1u : 0u;
                    s_bl += fabsf(ov[q] - an);
                    if (valid) st_state(&S[(ST_SLACK + 4 * b + q) * P], __float_as_uint(sp));
                }
            } else if (on<L>(B_BACKLASH)) {                              // per substep [Q26]
                float sl[4], sg[4], dd[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    sl[q] = slack[q];
                    sg[q] = (anv[q] > 0.f) ? 1.f : ((anv[q] < 0.f) ? -1.f : 0.f);
                    dd[q] = (anv[q] > 0.f) ? dpos[q] : dneg[q];
                    ov[q] = anv[q];
                }
                float4* osub = reinterpret_cast<float4*>(out_sub + (size_t)ec * (N_SUB * N_ACT) + 4 * b);
#pragma unroll 1
                for (int k = 0; k < N_SUB; ++k) {
                    const float dtk = s_dtk[k][lane];
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
            } else {
#pragma unroll
                for (int q = 0; q < 4; ++q) ov[q] = anv[q];
            }
            if (valid)
                st_out(reinterpret_cast<float4*>(out_actions + (size_t)e * N_ACT) + b, make_float4(ov[0], ov[1], ov[2], ov[3]));
            acc.n[K_CLAMPS] += n_clamp & vm;
            acc.n[K_RAIL] += n_rail & vm;
            acc.n[K_ALPHA1] += n_a1 & vm;
            acc.m[2] += valid ? s_da : 0.f;
            acc.m[3] += valid ? s_da2 : 0.f;
            acc.m[4] += valid ? s_bl : 0.f;
            acc.m[5] += valid ? s_zu2 : 0.f;
        } else if (wid == 5) {
            // ================= timing + step words [Q2] =================
            const float il = on<L>(B_TIMING) ? __uint_as_float(R[rec_off(ec, REC_INVLAM)]) : 0.f;
            float d[N_SUB];
            uint2 w01 = make_uint2(0u, 0u);
            if (on<L>(B_TIMING)) {
#pragma unroll
                for (int bb = 0; bb < 3; ++bb) {
                    const uint4 w = philox(g, t, CH_STEP, bb);
                    if (bb == 2) w01 = make_uint2(w.z, w.w);
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        if (4 * bb + q < N_SUB)
                            d[4 * bb + q] = c_dc.dt_base + (-(kSfuNormals ? ln_unit_sfu(uni(word_of(w, q))) : ln_unit(uni(word_of(w, q))))) * il;
                }
            } else {
#pragma unroll
                for (int k = 0; k < N_SUB; ++k) d[k] = c_dc.dt_base;
                if (on<L>(B_DROPOUT)) {
                    const uint4 w2 = philox(g, t, CH_STEP, 2);
                    w01 = make_uint2(w2.z, w2.w);
                }
            }
            const uint4 w3 = (on<L>(B_DROPOUT) || on<L>(B_FORCE)) ? philox(g, t, CH_STEP, 3) : make_uint4(0u, 0u, 0u, 0u);
            float dt_env = d[0];
#pragma unroll
            for (int k = 1; k < N_SUB; ++k) dt_env = dt_env + d[k];
            s_dtenv[lane] = dt_env;
#pragma unroll
            for (int k = 0; k < N_SUB; ++k) s_dtk[k][lane] = d[k];
            s_wd[0][lane] = w01.x;
            s_wd[1][lane] = w01.y;
            s_wd[2][lane] = w3.x;
            s_wd[3][lane] = w3.y;
            s_wd[4][lane] = w3.z;
            s_wd[5][lane] = w3.w;
            if (valid) {
                float2* o = reinterpret_cast<float2*>(out_dt + (size_t)e * N_SUB);
#pragma unroll
                for (int k = 0; k < N_SUB / 2; ++k) st_out(o + k, make_float2(d[2 * k], d[2 * k + 1]));
            }
            acc.m[0] += valid ? dt_env : 0.f;
            acc.m[1] += valid ? dt_env * dt_env : 0.f;
            my_envs += valid ? 1u : 0u;
            role_barrier();
        } else if (wid == 6) {
            // ================= fingertips =================
            const float* ro = raw_obs + (size_t)ec * OBS_IN;
            float tip[15], obj[3], off[15], last[15];
            {
                const float2* r2 = reinterpret_cast<const float2*>(ro);
#pragma unroll
                for (int k = 0; k < 9; ++k) {
                    const float2 v = __ldg(r2 + k);
                    const float x[2] = {v.x, v.y};
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int c = 2 * k + h;
                        if (c < 15) tip[c] = x[h];
                        else obj[c - 15] = x[h];
                    }
                }
            }
            if (on<L>(B_OBS_NOISE)) {   // off_tip = record words 64..78 (groups 8, 9)
                const float4* Rq = reinterpret_cast<const float4*>(R);
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    const float4 v = Rq[rec_off(ec, REC_OFFTIP + 4 * h) / 4];
#pragma unroll
                    for (int c = 0; c < 4; ++c)
                        if (4 * h + c < 15) off[4 * h + c] = q4(v, c);
                }
            } else {
#pragma unroll
                for (int n = 0; n < 15; ++n) off[n] = 0.f;
            }
#pragma unroll
            for (int n = 0; n < 15; ++n) last[n] = (kHold && hold_layers && !fresh) ? __uint_as_float(S[(ST_LAST + n) * P]) : 0.f;
            const uint32_t occ_in = (on<L>(B_OCCLUSION) && p.occl_in) ? (uint32_t)__ldg(p.occl_in + ec) : 0u;
            uint32_t occ = 0;
            if (on<L>(B_OCCLUSION) && p.occl_in) {                       // [Q27]
                occ = occ_in & 0x1Fu;
                acc.n[K_OCCLUDED] += __popc(occ) & vm;
            } else if (on<L>(B_OCCLUSION) && c_dc.occl_on) {             // [Q13]
                const float lo = c_dc.occl_r2_lo, hi = c_dc.occl_r2_hi;
                uint32_t amb = 0;
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
            float s_zt = 0.f;
            if (on<L>(B_OBS_NOISE)) {
#pragma unroll
                for (int bb = 0; bb < 4; ++bb) {
                    float z[4];
                    normals4_t<kSfuNormals>(philox(g, t, CH_TIP_NOISE, bb), z);
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int n = 4 * bb + q;
                        if (n < 15) {
                            tip[n] = (tip[n] + off[n]) + c_dc.tip_uncorr * z[q];
                            s_zt += z[q] * z[q];
                        }
                    }
                }
            }
            acc.m[6] += valid ? s_zt : 0.f;
            role_barrier();   // the dropout words of warp 5
            uint32_t masked = 0;
            if (kHold && hold_layers) {
                uint32_t nflags = 0, n_init = 0;
                if (on<L>(B_DROPOUT)) {                                  // [Q11]
#pragma unroll
                    for (int i = 0; i < N_TIPS; ++i) {
                        const uint32_t x = s_wd[i][lane];
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
                if (valid) st_state(&S[ST_FLAGS * P], 0u);
            }
            const uint32_t hold = (flags & HAS_LAST_BIT) ? (masked | occ) : 0u;   // [Q12]
            acc.n[K_HELD] += __popc(hold) & vm;
            if (kHold && hold_layers) {
#pragma unroll
                for (int i = 0; i < N_TIPS; ++i) {
                    if ((hold >> i) & 1u) {
#pragma unroll
                        for (int c = 0; c < 3; ++c) tip[3 * i + c] = last[3 * i + c];
                    } else if (valid) {
#pragma unroll
                        for (int c = 0; c < 3; ++c) st_state(&S[(ST_LAST + 3 * i + c) * P], __float_as_uint(tip[3 * i + c]));
                    }
                }
            }
            if (valid) {
                float* oo = out_obs + (size_t)e * OBS_OUT;
                float2* o2 = reinterpret_cast<float2*>(oo);
#pragma unroll
                for (int k = 0; k < 7; ++k) st_out(o2 + 2 + k, make_float2(tip[2 * k], tip[2 * k + 1]));
                st_out(oo + 18, tip[14]);
            }
        } else {
            // ========== object position, orientation, force ==========
            const float* ro = raw_obs + (size_t)ec * OBS_IN;
            float obj[3];
            obj[0] = __ldg(ro + 15);
            {
                const float2 v = __ldg(reinterpret_cast<const float2*>(ro + 16));
                obj[1] = v.x;
                obj[2] = v.y;
            }
            const float2 qa = __ldg(reinterpret_cast<const float2*>(ro + 18)), qb = __ldg(reinterpret_cast<const float2*>(ro + 20));
            const float2 ga = __ldg(reinterpret_cast<const float2*>(ro + 22)), gb = __ldg(reinterpret_cast<const float2*>(ro + 24));
            float cobj[3] = {0.f, 0.f, 0.f}, qc[4] = {0.f, 0.f, 0.f, 0.f};
            if (on<L>(B_OBS_NOISE)) {   // c_obj, q_c = record words 79..85 (groups 9, 10)
                const float4* Rq = reinterpret_cast<const float4*>(R);
                const float4 v0 = Rq[rec_off(ec, 76) / 4], v1 = Rq[rec_off(ec, 80) / 4], v2 = Rq[rec_off(ec, 84) / 4];
                cobj[0] = v0.w; cobj[1] = v1.x; cobj[2] = v1.y;
                qc[0] = v1.z; qc[1] = v1.w; qc[2] = v2.x; qc[3] = v2.y;
            }
            uint32_t tf = 0, kf = 0;
            float mass = 0.f, ft[3] = {0.f, 0.f, 0.f};
            if (on<L>(B_FORCE)) {
                tf = R[rec_off(ec, REC_TFORCE)];
                mass = __uint_as_float(R[rec_off(ec, REC_MASS)]);
                if (!fresh) {
                    kf = S[ST_KF * P];
#pragma unroll
                    for (int c = 0; c < 3; ++c) ft[c] = __uint_as_float(S[(ST_FTRIG + c) * P]);
                }
            }
            if (on<L>(B_OBS_NOISE)) {                                    // object position
                float z[4];
                normals4_t<kSfuNormals>(philox(g, t, CH_OBJ_NOISE, 0), z);
#pragma unroll
                for (int c = 0; c < 3; ++c) obj[c] = (obj[c] + cobj[c]) + c_dc.obj_uncorr * z[c];
            }
            float rel[4];                                                // [Q15, Q16]
            {
                const float qo[4] = {qa.x, qa.y, qb.x, qb.y};
                const float goal[4] = {ga.x, ga.y, gb.x, gb.y};
                float qn[4];
                if (on<L>(B_OBS_NOISE)) {
                    float qu[4], tmp[4];
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
            if (valid) {
                float* oo = out_obs + (size_t)e * OBS_OUT;
                float2* o2 = reinterpret_cast<float2*>(oo);
                st_out(o2 + 0, make_float2(rel[0], rel[1]));
                st_out(o2 + 1, make_float2(rel[2], rel[3]));
                st_out(oo + 19, obj[0]);
                st_out(o2 + 10, make_float2(obj[1], obj[2]));
            }
            role_barrier();   // the force trigger word of warp 5
            float f[3] = {0.f, 0.f, 0.f};
            if (on<L>(B_FORCE)) {                                        // [Q17, Q18]
                const uint32_t x = s_wd[5][lane];                        // step word 15
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
                    if (fresh && valid) {
#pragma unroll
                        for (int c = 0; c < 3; ++c) st_state(&S[(ST_FTRIG + c) * P], 0u);
                    }
                }
                if (valid) st_state(&S[ST_KF * P], kf);
                const double dec = __ldg(p.dec_tab + (kf & 255u)) * __ldg(p.dec_tab + 256u + (kf >> 8));
#pragma unroll
                for (int c = 0; c < 3; ++c) f[c] = (float)((double)ft[c] * dec);
            }
            acc.m[7] += valid ? f[0] * f[0] + f[1] * f[1] + f[2] * f[2] : 0.f;
            if (valid) {
                float* of = out_force + (size_t)e * 3;
#pragma unroll
                for (int c = 0; c < 3; ++c) st_out(of + c, f[c]);
            }
        }
    }
#ifdef DR_PROBE_TIMING
    if (lane == 0) probe_slot(p, t)[8 + wid] = gtime();   // this warp's role done
#endif
    reduce_stats<L, LAT_THREADS>(p, acc, my_envs, t, s_red);
}
