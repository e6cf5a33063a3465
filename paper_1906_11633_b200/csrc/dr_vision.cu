// dr_vision.cu -- vision randomizations (include/dr_vision.h): appearance draws (Table
// vision-randomization) and the post-render image augmentation
// for sm_100a.
//
// image_augment_kernel: one thread-block cluster of K CTAs per image (K = 1..8, chosen so a
// CTA's slice of the image fits in <= 32 KB of shared memory when it can).  Each CTA
//   1. pulls its slice of the u8 image into shared memory with one TMA bulk copy
//      (cp.async.bulk + mbarrier complete_tx), so the image crosses HBM exactly once;
//   2. reduces exact integer sum / sum of squares (DP4A: 2 instructions per 4 pixels), then the
//      cluster exchanges the K partials through distributed shared memory (mapa +
//      ld.shared::cluster between two cluster barriers) -- every CTA gets the same exact totals;
//   3. writes out = (x - mean) * (f / std) + s * z with streaming float4 stores, one Philox
//      block per 4 elements for the noise.
// HBM traffic per image: E bytes in + 4E bytes out (E = H W C), the algorithmic minimum.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "dr.h"
#include "dr_internal.h"
#include "dr_math.cuh"
#include "dr_vision.h"

namespace dr {

enum : uint32_t { CH_POSE = 0x401, CH_IMG_PARAM = 0x201, CH_IMG_NOISE = 0x202, CH_SCENE_CAM = 0x301, CH_SCENE_MAT = 0x302,
                  CH_SCENE_LIGHT = 0x303 };

#ifndef DR_IMG_THREADS
#define DR_IMG_THREADS 128   // A/B (us per 192-image batch, map v2): 128 35.9, 256 36.7, 512 49.5 (map v1: 41.1, 40.2, 43.3)
#endif
constexpr int IMG_THREADS = DR_IMG_THREADS;
#ifndef DR_IMG_PROBE
#define DR_IMG_PROBE 0   // roofline probes (A/B builds only): 1 = no noise draws, 2 = no output stores
#endif
#ifndef DR_IMG_PRE
#define DR_IMG_PRE 1   // 8-element groups per thread whose noise is drawn while the slice loads
#endif
#ifndef DR_IMG_MID
#define DR_IMG_MID 1   // ... and groups drawn between the cluster barrier's arrive and wait
#endif
constexpr int IMG_PRE = DR_IMG_PRE, IMG_MID = DR_IMG_MID, IMG_EARLY = IMG_PRE + IMG_MID;
constexpr uint32_t IMG_SLICE_MAX = 200 * 1024;


struct ImgArgs {
    const uint8_t* images;
    float* out;
    float* img_stats;
    uint64_t E;          // bytes (= elements) per image
    uint32_t slice;      // bytes per CTA slice (multiple of 16)
    uint32_t aligned;    // TMA + float4 path (E % 16 == 0, pointers 16-byte aligned)
    uint32_t batch;
    uint32_t image_offset;
    uint32_t early_read;    // 1: this call may read its images before the previous kernel of the stream completed
    uint32_t early_write;   // 1: ... and write its outputs
    double contrast_lo, contrast_range, noise_lo, noise_range;   // lo + (hi - lo) U, as the oracle
    double std_floor;
    PhiloxKeys keys;
};

// ---- cluster / DSMEM / TMA helpers (PTX, sm_90+) ------------------------------------------
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t cluster_size() {
    uint32_t n;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(n));
    return n;
}
__device__ __forceinline__ void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
// 64-bit load from CTA `rank`'s copy of the shared variable at local address `a`
__device__ __forceinline__ unsigned long long ld_dsmem_u64(uint32_t a, uint32_t rank) {
    uint32_t ra;
    unsigned long long v;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
    asm volatile("ld.shared::cluster.u64 %0, [%1];" : "=l"(v) : "r"(ra) : "memory");
    return v;
}
__device__ __forceinline__ void mbar_init1(uint64_t* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait0(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "W_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t"
        "@!p bra W_%=;\n}" ::"r"(smem_addr(bar))
        : "memory");
}
__device__ __forceinline__ void tma_bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(dst)),
                 "l"(src), "r"(bytes), "r"(smem_addr(bar))
                 : "memory");
}

// Image-noise normals (vision RNG map v2, V7): one Philox block gives 8 normals -- word w
// is one Box-Muller pair with the radius from its top 20 bits and the angle from its low 12 bits --
// so element e takes normal e % 2 of the pair of word (e % 8) / 2 of block e / 8 (map v1 drew one
// block per 4 elements: Philox was ~40 % of the kernel's instructions).
// nz_raw gives the pair's s r, sin and cos; the noise of the two elements is then
// (-(s r) cos + k, -(s r) sin + k) with the per-image constant k (nz_fold), so the draws -- all of the
// XU work -- need no image moments and start while the slice is still loading:
//   -2 ln U (s^2 folded into the constants): MUFU.LG2 except for 1 - U < 2^-6, where the series
//   v (2 + v (1 + 2v/3)) keeps the tiny radius accurate (the fast pair of dr_math.cuh); U and 1 - U
//   are exact, built from the word's bits; r s from MUFU.SQRT;
//   the angle 2 pi (A - 1/2) in one FFMA from the 12-bit integer, then MUFU.SIN / MUFU.COS
//   (cos(t - pi) = -cos t and sin(t - pi) = -sin t: the sign goes into the FFMA with k).
//   A/B (µs per 192-image batch): a quarter-wave (cos, sin) table in shared memory 41.4 vs 35.9 (the
//   random reads conflict); (sin, cos) as FMA-pipe polynomials 43.0, for half the pairs 38.6.
struct NzConst {
    float s2_lg;    // -2 ln(2) s^2
    float s2_c2, s2_c1, s2_c0;   // s^2 (2/3), s^2, 2 s^2
};
struct NzRaw {
    float rs[4], sn[4], cs[4];   // the four pairs of one 8-element group
};
__device__ __forceinline__ void nz_raw(uint32_t x, const NzConst& c, float& rs, float& sn, float& cs) {
    uint32_t ub;   // (x >> 12) * 8 + 0x3F800004 in one IMAD after the shift (the OR form took two LOP3s)
    asm("mad.lo.u32 %0, %1, 8, 0x3F800004;" : "=r"(ub) : "r"(x >> 12));
    const float u = __uint_as_float(ub) - 1.0f;                                       // (k + 1/2) 2^-20, exact
    const float v = 1.0f - u;   // exact: u has 21 significant bits below 1 (one FADD: 32.8 -> 30.9 us)
    const float series = v * fmaf(fmaf(v, c.s2_c2, c.s2_c1), v, c.s2_c0);
    const float lg = lg2_approx(u) * c.s2_lg;
    rs = sqrt_approx((v < 0.015625f) ? series : lg);                                  // s sqrt(-2 ln u)
    const float ang = fmaf((float)(x & 0xFFFu), 1.53398078788564122e-03f, -3.14082566319585e+00f);
    __sincosf(ang, &sn, &cs);
}
__device__ __forceinline__ void nz_group(const uint4 w, const NzConst& c, NzRaw& q) {
    nz_raw(w.x, c, q.rs[0], q.sn[0], q.cs[0]);
    nz_raw(w.y, c, q.rs[1], q.sn[1], q.cs[1]);
    nz_raw(w.z, c, q.rs[2], q.sn[2], q.cs[2]);
    nz_raw(w.w, c, q.rs[3], q.sn[3], q.cs[3]);
}
__device__ __forceinline__ void nz_fold(const NzRaw& q, float kq, float z[8]) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        z[2 * j] = fmaf(-q.rs[j], q.cs[j], kq);
        z[2 * j + 1] = fmaf(-q.rs[j], q.sn[j], kq);
    }
}

// Programmatic dependent launch (the augment kernel goes out with
// cudaLaunchAttributeProgrammaticStreamSerialization): every CTA lets the next kernel of the stream
// launch at once, so the next batch's clusters take the SM slots this batch's clusters free and
// read their images, reduce their moments and draw their first noise groups while this batch is
// still writing (one batch is one wave of clusters that read all images, then write all outputs).
// A call reads its images before the previous kernel of the stream has completed only when the
// host saw that kernel is the previous augmentation of the same stream and its outputs do not
// overlap these images (a.early_read), and writes (img_stats, out) early only when in addition
// neither call's outputs overlap the other's images or outputs (a.early_write, dr_image_augment);
// otherwise every CTA waits (griddepcontrol.wait) at its start, or before its first write.  Every
// CTA waits before it exits, so no call completes before its predecessor.  Back-to-back batches of 192 images (A/B): 28.7 us per batch
// without PDL, 27.3 with every write behind the wait, 21.5 with early writes.
__device__ __forceinline__ void img_pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void img_pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Register cap: 10 CTAs of 128 threads per SM (48 registers, no spills with one pre-drawn group)
// instead of 7 (72 registers, two pre-drawn groups), so more of the next batch's clusters fit beside
// this batch's and load while it writes.  A/B (us per 192-image batch, three alternating runs,
// bit-identical): 72 registers 21.56; caps of 8 / 10 / 11 / 16 CTAs 20.93 / 20.82 / 21.34 / 21.37
// (11 and 16 spill); DR_IMG_MINB=0 restores the uncapped build.
#ifndef DR_IMG_MINB
#define DR_IMG_MINB (1280 / DR_IMG_THREADS)   // 10 CTAs of 128 threads (48 registers); scales with the CTA size
#endif
#if DR_IMG_MINB > 0
#define DR_IMG_BOUNDS __launch_bounds__(IMG_THREADS, DR_IMG_MINB)
#else
#define DR_IMG_BOUNDS __launch_bounds__(IMG_THREADS)
#endif
__global__ void DR_IMG_BOUNDS image_augment_kernel(const ImgArgs a) {
    img_pdl_trigger();
    if (!a.early_read) img_pdl_wait();   // the previous kernel of the stream may have written the images
    extern __shared__ __align__(128) uint8_t s_img[];
    __shared__ __align__(8) uint64_t s_bar;
    __shared__ unsigned long long s_part[2];
    __shared__ unsigned long long s_warp[2][IMG_THREADS / 32];

    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const uint32_t K = cluster_size(), r = cluster_rank();
    const uint64_t img = blockIdx.x / K;
    const uint64_t E = a.E;
    const uint64_t lo0 = (uint64_t)r * a.slice;
    const uint64_t lo = lo0 < E ? lo0 : E;
    const uint64_t hi = (lo + a.slice) < E ? (lo + a.slice) : E;
    const uint32_t n = (uint32_t)(hi - lo);
    const uint8_t* src = a.images + img * E + lo;

    // the image's contrast f and noise std s: one Philox block, no moments needed
    const uint32_t g = a.image_offset + (uint32_t)img;
    const uint4 pw = philox_k(g, a.batch, CH_IMG_PARAM, 0, a.keys);
    const double f = a.contrast_lo + a.contrast_range * (double)uni(pw.x);
    const double s = a.noise_lo + a.noise_range * (double)uni(pw.y);
    NzConst nc;
    {
        const double s2 = s * s;
        nc.s2_lg = (float)(-1.38629436111989061883 * s2);
        nc.s2_c2 = (float)(0.666666666666666667 * s2);
        nc.s2_c1 = (float)s2;
        nc.s2_c0 = (float)(2.0 * s2);
    }
    const uint32_t b0 = (uint32_t)(lo >> 3);   // lo is a multiple of 16: 8-element noise blocks
    const uint32_t n8 = n >> 3;

    // ---- 1. slice -> shared memory (one TMA bulk copy); the first IMG_PRE groups' noise draws
    //         (Philox + the XU transforms) run while it lands ----
    NzRaw pre[IMG_EARLY > 0 ? IMG_EARLY : 1];
    if (a.aligned) {
        if (tid == 0) mbar_init1(&s_bar);
        __syncthreads();
        if (tid == 0) {
            mbar_expect(&s_bar, n);
            if (n) tma_bulk(s_img, src, n, &s_bar);
        }
#pragma unroll
        for (int q = 0; q < IMG_PRE; ++q) {
            const uint32_t i = tid + q * IMG_THREADS;
            if (i < n8) nz_group(philox_k(g, a.batch, CH_IMG_NOISE, b0 + i, a.keys), nc, pre[q]);
        }
        mbar_wait0(&s_bar);
    } else {
        for (uint32_t i = tid; i < n; i += IMG_THREADS) s_img[i] = __ldg(src + i);
        __syncthreads();
    }

    // ---- 2. exact integer moments, CTA then cluster ----
    uint32_t sum = 0, sq = 0;
    const uint32_t n4 = n >> 2;
    const uint32_t* w4 = reinterpret_cast<const uint32_t*>(s_img);
    for (uint32_t i = tid; i < n4; i += IMG_THREADS) {
        const uint32_t x = w4[i];
        sum = __dp4a(x, 0x01010101u, sum);
        sq = __dp4a(x, x, sq);
    }
    for (uint32_t i = 4 * n4 + tid; i < n; i += IMG_THREADS) {
        const uint32_t x = s_img[i];
        sum += x;
        sq += x * x;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        sum += __shfl_xor_sync(0xFFFFFFFFu, sum, o);
        sq += __shfl_xor_sync(0xFFFFFFFFu, sq, o);
    }
    if (lane == 0) {
        s_warp[0][wid] = sum;
        s_warp[1][wid] = sq;
    }
    __syncthreads();
    if (tid == 0) {
        unsigned long long S = 0, Q = 0;
#pragma unroll
        for (int k = 0; k < IMG_THREADS / 32; ++k) {
            S += s_warp[0][k];
            Q += s_warp[1][k];
        }
        s_part[0] = S;
        s_part[1] = Q;
    }
    cluster_arrive();   // publishes s_part to the cluster
    if (a.aligned) {
#pragma unroll
        for (int q = IMG_PRE; q < IMG_EARLY; ++q) {
            const uint32_t i = tid + q * IMG_THREADS;
            if (i < n8) nz_group(philox_k(g, a.batch, CH_IMG_NOISE, b0 + i, a.keys), nc, pre[q]);
        }
    }
    cluster_wait();
    unsigned long long S = 0, Q = 0;
    for (uint32_t q = 0; q < K; ++q) {   // fixed rank order: identical totals in every CTA
        S += ld_dsmem_u64(smem_addr(&s_part[0]), q);
        Q += ld_dsmem_u64(smem_addr(&s_part[1]), q);
    }
    cluster_arrive();   // done reading the other CTAs' shared memory (matched by the wait at exit)
    if (!a.early_write) img_pdl_wait();   // the previous kernel of the stream has completed: this CTA may write

    // ---- 3. normalise, contrast, noise ----
    const double mean = (double)S / (double)E;
    const unsigned long long vnum = Q * E - S * S;   // E^2 var, exact (no overflow below the size limit)
    const double sd = sqrt((double)vnum / ((double)E * (double)E));
    const float scale = (float)(f / (sd > a.std_floor ? sd : a.std_floor));
    // out = (x - mu_i) * scale + (s z + k), mu_i = rint(mean), k = -(mean - mu_i) * scale: a byte x is
    // read as the float 2^23 + x (one PRMT of the packed bytes under the exponent 0x4B, no I2F on the
    // XU pipe the noise draws' MUFUs share: 35.9 -> 34.5 us per batch) and (2^23 + x) - (2^23 + mu_i)
    // is exact; |x - mean| >= |mean - mu_i| for every byte x, so k never dominates the result it is
    // rounded into.  Every element of every image takes the same expression, whatever the slice /
    // cluster size.
    const float mu_i = (float)rint(mean), c_b = 8388608.0f + mu_i;   // exact: integer < 2^24
    const float kq = (float)(-(mean - (double)mu_i) * (double)scale);
    if (r == 0 && tid == 0 && a.img_stats)
        reinterpret_cast<float4*>(a.img_stats)[img] = make_float4((float)mean, (float)sd, (float)f, (float)s);

    float* out = a.out + img * E + lo;
    if (a.aligned) {
        // whole 8-element groups: one Philox block, four Box-Muller pairs, one 256-bit streaming store
        const uint2* w8 = reinterpret_cast<const uint2*>(s_img);
        float4* o4 = reinterpret_cast<float4*>(out);
        auto emit = [&](uint32_t i, const NzRaw& q) {
            float z[8];
            nz_fold(q, kq, z);
            const uint2 x = w8[i];
            float v[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const float xb = __uint_as_float(__byte_perm(k < 4 ? x.x : x.y, 0x4B000000u, 0x7540u | (k & 3)));
                v[k] = fmaf(xb - c_b, scale, z[k]);   // (2^23 + x) - (2^23 + mu_i), exact
            }
#if DR_IMG_PROBE == 2   // roofline probe (A/B only): no output stores
            if (v[0] + v[1] + v[2] + v[3] + v[4] + v[5] + v[6] + v[7] == 12345.f) out[0] = 0.f;
#else
            // a warp writes 32 whole sectors (1 KB contiguous) per store
            asm volatile("st.global.cs.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(o4 + 2 * i), "f"(v[0]),
                         "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
                         : "memory");
#endif
        };
#pragma unroll
        for (int q = 0; q < IMG_EARLY; ++q) {
            const uint32_t i = tid + q * IMG_THREADS;
            if (i < n8) emit(i, pre[q]);
        }
        for (uint32_t i = tid + IMG_EARLY * IMG_THREADS; i < n8; i += IMG_THREADS) {
            NzRaw q;
#if DR_IMG_PROBE == 1   // roofline probe (A/B only): no noise draws
            for (int j = 0; j < 4; ++j) q.rs[j] = q.sn[j] = q.cs[j] = (float)(i & (1u << j));
#else
            nz_group(philox_k(g, a.batch, CH_IMG_NOISE, b0 + i, a.keys), nc, q);
#endif
            emit(i, q);
        }
    } else {
        for (uint32_t i = tid; i < (n + 7) / 8; i += IMG_THREADS) {
            NzRaw q;
            nz_group(philox_k(g, a.batch, CH_IMG_NOISE, b0 + i, a.keys), nc, q);
            float z[8];
            nz_fold(q, kq, z);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const uint32_t e = 8 * i + k;
                if (e < n) out[e] = fmaf(__uint_as_float(0x4B000000u | s_img[e]) - c_b, scale, z[k]);
            }
        }
    }
    cluster_wait();   // no CTA leaves while another may still read its s_part
    img_pdl_wait();   // ... nor before the previous kernel of the stream has completed
}

// ---- appearance draws: one thread per sample, fp64 (no contraction in the decision chain) ----
struct SceneArgs {
    dr_vision_params p;
    uint32_t batch;
    uint32_t sample_offset;
    uint32_t n;
    PhiloxKeys keys;
};

__device__ __forceinline__ double ud(uint32_t x) { return (double)uni(x); }   // exact
__device__ __forceinline__ double range_d(double lo, double hi, uint32_t x) {
    return __dadd_rn(lo, __dmul_rn(__dsub_rn(hi, lo), ud(x)));
}

__global__ void scene_draw_kernel(const SceneArgs a, dr_scene_draw* __restrict__ out) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= a.n) return;
    const uint32_t g = a.sample_offset + k;
    const dr_vision_params& p = a.p;
    float o[64];
#pragma unroll
    for (int i = 0; i < 64; ++i) o[i] = 0.f;
    constexpr double TWO_PI = 6.283185307179586476925;
#pragma unroll
    for (int c = 0; c < DR_VIS_N_CAMERAS; ++c) {
        uint4 w = philox_k(g, a.batch, CH_SCENE_CAM, 2 * c, a.keys);
        o[3 * c + 0] = (float)range_d(-p.cam_pos_range, p.cam_pos_range, w.x);   // [V1]
        o[3 * c + 1] = (float)range_d(-p.cam_pos_range, p.cam_pos_range, w.y);
        o[3 * c + 2] = (float)range_d(-p.cam_pos_range, p.cam_pos_range, w.z);
        o[21 + c] = (float)range_d(-p.cam_fov_range, p.cam_fov_range, w.w);
        w = philox_k(g, a.batch, CH_SCENE_CAM, 2 * c + 1, a.keys);
        const double th = range_d(0.0, p.cam_rot_max, w.x);                       // [V2]
        const double zc = __dsub_rn(__dmul_rn(2.0, ud(w.y)), 1.0);
        const double phi = __dmul_rn(TWO_PI, ud(w.z));
        const double rho = sqrt(__dsub_rn(1.0, __dmul_rn(zc, zc)));
        double sh, ch, sp, cp;
        sincos(0.5 * th, &sh, &ch);
        sincos(phi, &sp, &cp);
        o[9 + 4 * c + 0] = (float)ch;
        o[9 + 4 * c + 1] = (float)(sh * rho * cp);
        o[9 + 4 * c + 2] = (float)(sh * rho * sp);
        o[9 + 4 * c + 3] = (float)(sh * zc);
    }
    const uint4 m0 = philox_k(g, a.batch, CH_SCENE_MAT, 0, a.keys);
    const uint4 m1 = philox_k(g, a.batch, CH_SCENE_MAT, 1, a.keys);
    const uint4 m2 = philox_k(g, a.batch, CH_SCENE_MAT, 2, a.keys);
    o[24] = uni(m0.x);
    o[25] = uni(m0.y);
    o[26] = uni(m0.z);
    o[27] = (float)range_d(p.robot_metallic_lo, p.robot_metallic_hi, m0.w);
    o[28] = (float)range_d(p.robot_gloss_lo, p.robot_gloss_hi, m1.x);
    {   // [V3] additive offsets; hue wraps, saturation / value clamp -- decided in exact-order fp64
        const double h = __dadd_rn(p.obj_hue_cal, range_d(-p.obj_hue_range, p.obj_hue_range, m1.y));
        const double s = __dadd_rn(p.obj_sat_cal, range_d(-p.obj_sat_range, p.obj_sat_range, m1.z));
        const double v = __dadd_rn(p.obj_val_cal, range_d(-p.obj_val_range, p.obj_val_range, m1.w));
        o[29] = (float)__dsub_rn(h, floor(h));
        o[30] = (float)fmin(fmax(s, 0.0), 1.0);
        o[31] = (float)fmin(fmax(v, 0.0), 1.0);
    }
    o[32] = (float)range_d(p.obj_metallic_lo, p.obj_metallic_hi, m2.x);
    o[33] = (float)range_d(p.obj_gloss_lo, p.obj_gloss_hi, m2.y);
    const int nl = p.lights_min + (int)(((unsigned long long)m2.z * (unsigned long long)(p.lights_max - p.lights_min + 1)) >> 32);
    const double total = range_d(p.light_total_lo, p.light_total_hi, m2.w);   // [V5]
    double rel[DR_VIS_MAX_LIGHTS];
    double rsum = 0.0;
    for (int i = 0; i < nl; ++i) {
        const uint4 w = philox_k(g, a.batch, CH_SCENE_LIGHT, i, a.keys);
        const double z = ud(w.x);
        const double phi = __dmul_rn(TWO_PI, ud(w.y));
        const double rho = sqrt(__dsub_rn(1.0, __dmul_rn(z, z)));
        double sp, cp;
        sincos(phi, &sp, &cp);
        o[35 + 3 * i + 0] = (float)(rho * cp);
        o[35 + 3 * i + 1] = (float)(rho * sp);
        o[35 + 3 * i + 2] = (float)z;
        rel[i] = range_d(p.light_rel_lo, p.light_rel_hi, w.z);
        rsum += rel[i];
    }
    for (int i = 0; i < nl; ++i) o[53 + i] = (float)(total * rel[i] / rsum);
    o[59] = (float)total;
    float4* d4 = reinterpret_cast<float4*>(out + k);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        float4 v = make_float4(o[4 * i], o[4 * i + 1], o[4 * i + 2], o[4 * i + 3]);
        if (i == 8) v.z = __uint_as_float((uint32_t)nl);   // word 34: n_lights (u32)
        d4[i] = v;
    }
}

// ---- pose augmentation [Q28]: one thread per sample ----
struct PoseArgs {
    unsigned long long t_keep, t_rot;   // floor(p_keep 2^32), floor((p_keep + p_rot90) 2^32)
    float pos_std, rot_std;
    uint32_t batch, offset, n;
    PhiloxKeys keys;
};

__global__ void pose_augment_kernel(const PoseArgs a, const float* in, float* out,   // may alias
                                    uint8_t* __restrict__ branch) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= a.n) return;
    const uint32_t g = a.offset + k;
    float v[7];
#pragma unroll
    for (int c = 0; c < 7; ++c) v[c] = in[(size_t)k * 7 + c];
    const float q[4] = {v[3], v[4], v[5], v[6]};
    const uint4 w = philox_k(g, a.batch, CH_POSE, 0, a.keys);
    const int b = ((unsigned long long)w.x < a.t_keep) ? 0 : (((unsigned long long)w.x < a.t_rot) ? 1 : 2);
    float o[7] = {v[0], v[1], v[2], q[0], q[1], q[2], q[3]};
    if (b == 1) {
        // exactly 90 deg about body axis kk / 2 with sign from kk's parity: q (x) r
        const int kk = (int)(((unsigned long long)w.y * 6ull) >> 32);
        const float h = 0.70710678118654752f;
        float r[4] = {h, 0.f, 0.f, 0.f};
        r[1 + kk / 2] = (kk & 1) ? -h : h;
        qmul(q, r, o + 3);
    } else if (b == 2) {
        const uint4 u = philox_k(g, a.batch, CH_POSE, 1, a.keys);
        float z0, z1, z2, z3;
        box_muller(u.x, u.y, z0, z1);
        box_muller(u.z, u.w, z2, z3);
        o[0] = v[0] + a.pos_std * z0;
        o[1] = v[1] + a.pos_std * z1;
        o[2] = v[2] + a.pos_std * z2;
        float qj[4];
        rotation<false>(a.rot_std, philox_k(g, a.batch, CH_POSE, 2, a.keys), qj);
        qmul(qj, q, o + 3);
    }
#pragma unroll
    for (int c = 0; c < 7; ++c) out[(size_t)k * 7 + c] = o[c];
    if (branch) branch[k] = (uint8_t)b;
}

static PhiloxKeys make_keys(uint64_t seed) {
    PhiloxKeys k;
    const uint32_t k0 = (uint32_t)(seed & 0xFFFFFFFFull), k1 = (uint32_t)(seed >> 32);
    for (int r = 0; r < 10; ++r) {
        k.rk0[r] = k0 + (uint32_t)r * 0x9E3779B9u;
        k.rk1[r] = k1 + (uint32_t)r * 0xBB67AE85u;
    }
    return k;
}

static int check_vision(const dr_vision_params* p) {
    if (!p) return set_error(DR_EINVAL, "vision params: NULL");
    if (p->abi_version != DR_ABI_VERSION || p->struct_size != sizeof(dr_vision_params))
        return set_error(DR_EINVAL, "vision params: abi_version / struct_size mismatch");
    struct { const char* n; double lo, hi; } rg[] = {
        {"robot_metallic", p->robot_metallic_lo, p->robot_metallic_hi}, {"robot_gloss", p->robot_gloss_lo, p->robot_gloss_hi},
        {"obj_metallic", p->obj_metallic_lo, p->obj_metallic_hi}, {"obj_gloss", p->obj_gloss_lo, p->obj_gloss_hi},
        {"light_rel", p->light_rel_lo, p->light_rel_hi}, {"light_total", p->light_total_lo, p->light_total_hi},
        {"contrast", p->contrast_lo, p->contrast_hi}, {"noise_std", p->noise_std_lo, p->noise_std_hi}};
    for (auto& x : rg)
        if (!(x.lo <= x.hi) || !std::isfinite(x.lo) || !std::isfinite(x.hi))
            return set_error(DR_EINVAL, "%s_lo/%s_hi: need finite lo <= hi", x.n, x.n);
    struct { const char* n; double v; } nn[] = {
        {"cam_pos_range", p->cam_pos_range}, {"cam_rot_max", p->cam_rot_max}, {"cam_fov_range", p->cam_fov_range},
        {"obj_hue_range", p->obj_hue_range}, {"obj_sat_range", p->obj_sat_range}, {"obj_val_range", p->obj_val_range},
        {"contrast_lo", p->contrast_lo}, {"noise_std_lo", p->noise_std_lo}, {"light_rel_lo", p->light_rel_lo},
        {"light_total_lo", p->light_total_lo}};
    for (auto& x : nn)
        if (!(x.v >= 0.0) || !std::isfinite(x.v)) return set_error(DR_EINVAL, "%s: must be a finite value >= 0", x.n);
    if (!(p->light_rel_lo > 0.0)) return set_error(DR_EINVAL, "light_rel_lo: must be > 0");
    if (!(p->std_floor > 0.0)) return set_error(DR_EINVAL, "std_floor: must be > 0");
    if (p->lights_min < 1 || p->lights_max > DR_VIS_MAX_LIGHTS || p->lights_min > p->lights_max)
        return set_error(DR_EINVAL, "lights_min/lights_max: need 1 <= min <= max <= 6");
    return DR_OK;
}

}  // namespace dr

using namespace dr;

extern "C" {

int dr_vision_params_default(dr_vision_params* p) {
    if (!p) return set_error(DR_EINVAL, "params: NULL");
    *p = dr_vision_params{};
    p->abi_version = DR_ABI_VERSION;
    p->struct_size = sizeof(dr_vision_params);
    const double deg = 3.14159265358979323846 / 180.0;
    p->cam_pos_range = 1.5e-3;   // Table vision-randomization
    p->cam_rot_max = 3.0 * deg;
    p->cam_fov_range = 1.0 * deg;
    p->robot_metallic_lo = 0.05; p->robot_metallic_hi = 0.25;
    p->robot_gloss_lo = 0.0; p->robot_gloss_hi = 1.0;
    p->obj_hue_cal = 0.005; p->obj_sat_cal = 0.9; p->obj_val_cal = 0.5;   // workload choice
    p->obj_hue_range = 0.01; p->obj_sat_range = 0.15; p->obj_val_range = 0.15;
    p->obj_metallic_lo = 0.05; p->obj_metallic_hi = 0.15;
    p->obj_gloss_lo = 0.05; p->obj_gloss_hi = 0.15;
    p->lights_min = 4; p->lights_max = 6;
    p->light_rel_lo = 1.0; p->light_rel_hi = 5.0;
    p->light_total_lo = 0.0; p->light_total_hi = 15.0;
    p->contrast_lo = 0.5; p->contrast_hi = 1.5;
    p->noise_std_lo = 0.1; p->noise_std_hi = 0.1;   // [V6]
    p->std_floor = 1e-8;
    return DR_OK;
}

int dr_scene_draw_batch(const dr_vision_params* p, uint64_t seed, uint64_t batch_index, int64_t sample_offset,
                        int64_t n_samples, dr_scene_draw* out_dev, void* stream) {
    int rc = check_vision(p);
    if (rc != DR_OK) return rc;
    if (n_samples < 0 || sample_offset < 0 || sample_offset + n_samples > (int64_t(1) << 32))
        return set_error(DR_EINVAL, "n_samples/sample_offset: outside [0, 2^32)");
    if (n_samples == 0) return DR_OK;
    if (!out_dev || ((uintptr_t)out_dev & 15u)) return set_error(DR_EINVAL, "out: NULL or not 16-byte aligned");
    SceneArgs a{};
    a.p = *p;
    a.batch = (uint32_t)batch_index;
    a.sample_offset = (uint32_t)sample_offset;
    a.n = (uint32_t)n_samples;
    a.keys = make_keys(seed);
    const int threads = 128;
    scene_draw_kernel<<<(unsigned)((n_samples + threads - 1) / threads), threads, 0, static_cast<cudaStream_t>(stream)>>>(
        a, out_dev);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_error(DR_ECUDA, "scene_draw_kernel: %s", cudaGetErrorString(e));
    count_launch();
    note_stream_launch(stream, nullptr);
    return DR_OK;
}

int dr_pose_aug_params_default(dr_pose_aug_params* p) {
    if (!p) return set_error(DR_EINVAL, "params: NULL");
    *p = dr_pose_aug_params{};
    p->abi_version = DR_ABI_VERSION;
    p->struct_size = sizeof(dr_pose_aug_params);
    p->p_keep = 0.2;
    p->p_rot90 = 0.4;
    p->pos_std = 5e-3;   // not in the paper, Q28
    p->rot_std = 0.05;
    return DR_OK;
}

int dr_pose_augment(const dr_pose_aug_params* p, uint64_t seed, uint64_t batch_index, int64_t sample_offset,
                    const float* pose_in, int64_t n, float* pose_out, uint8_t* branch_out, void* stream) {
    if (!p) return set_error(DR_EINVAL, "pose params: NULL");
    if (p->abi_version != DR_ABI_VERSION || p->struct_size != sizeof(dr_pose_aug_params))
        return set_error(DR_EINVAL, "pose params: abi_version / struct_size mismatch");
    if (!(p->p_keep >= 0.0 && p->p_rot90 >= 0.0 && p->p_keep + p->p_rot90 <= 1.0))
        return set_error(DR_EINVAL, "p_keep/p_rot90: need p_keep, p_rot90 >= 0 and p_keep + p_rot90 <= 1");
    if (!(p->pos_std >= 0.0) || !(p->rot_std >= 0.0) || !std::isfinite(p->pos_std) || !std::isfinite(p->rot_std))
        return set_error(DR_EINVAL, "pos_std/rot_std: must be finite values >= 0");
    if (n < 0 || sample_offset < 0 || sample_offset + n > (int64_t(1) << 32))
        return set_error(DR_EINVAL, "n/sample_offset: outside [0, 2^32)");
    if (n == 0) return DR_OK;
    if (!pose_in || !pose_out) return set_error(DR_EINVAL, "pose_in/pose_out: NULL");
    auto thr = [](double q) -> unsigned long long {
        if (!(q > 0.0)) return 0ull;
        if (q >= 1.0) return 1ull << 32;
        return (unsigned long long)std::floor(q * 4294967296.0);
    };
    PoseArgs a{};
    a.t_keep = thr(p->p_keep);
    a.t_rot = thr(p->p_keep + p->p_rot90);
    a.pos_std = (float)p->pos_std;
    a.rot_std = (float)p->rot_std;
    a.batch = (uint32_t)batch_index;
    a.offset = (uint32_t)sample_offset;
    a.n = (uint32_t)n;
    a.keys = make_keys(seed);
    pose_augment_kernel<<<(unsigned)((n + 127) / 128), 128, 0, static_cast<cudaStream_t>(stream)>>>(a, pose_in, pose_out,
                                                                                                     branch_out);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_error(DR_ECUDA, "pose_augment_kernel: %s", cudaGetErrorString(e));
    count_launch();
    note_stream_launch(stream, nullptr);
    return DR_OK;
}

}  // extern "C"

namespace {
bool g_img_attr_set = false;

uint32_t img_slice_of(uint64_t E, uint32_t K) { return (uint32_t)(((E + K - 1) / K + 15) / 16 * 16); }

// Cluster size K (1..8, DR_IMG_K=1..8 forces it).  Images whose slice fits 32 KB at some K <= 8:
// among the K with slice <= 32 KB (and >= 8 KB, or K = 1), the one minimising waves x slice bytes,
// with waves = ceil(n_images / co-resident clusters of K) from cudaOccupancyMaxActiveClusters --
// the per-CTA time scales with its slice and a partial second wave doubles it.  Measured (B200,
// 192 images of 200 x 200 x 3, us per batch): K = 3 43.2, 4 40.0, 5 39.2 (chosen), 6 44.5
// (187 co-resident clusters < 192: two waves), 7 44.0, 8 44.2.  Larger images: the smallest
// power of two whose slice fits 200 KB.
uint32_t img_cluster_size(uint64_t E, uint64_t n) {
    static const int forced = [] {
        const char* v = std::getenv("DR_IMG_K");
        return v ? std::atoi(v) : 0;
    }();
    if (forced >= 1 && forced <= 8 && img_slice_of(E, (uint32_t)forced) <= IMG_SLICE_MAX) return (uint32_t)forced;
    if (img_slice_of(E, 8) > 32u * 1024u) {   // large images: the smallest power of two that fits
        uint32_t K = 1;
        while (K < 8 && img_slice_of(E, K) > 32u * 1024u) K *= 2;
        return K;
    }
    thread_local uint64_t c_E = 0, c_n = 0;
    thread_local uint32_t c_K = 0;
    if (c_E == E && c_n == n && c_K) return c_K;
    uint32_t best = 0;
    double best_cost = 0.0;
    for (uint32_t K = 1; K <= 8; ++K) {
        const uint32_t sl = img_slice_of(E, K);
        if (sl > 32u * 1024u || (K > 1 && sl < 8u * 1024u)) continue;
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(K, 1, 1);
        cfg.blockDim = dim3(IMG_THREADS, 1, 1);
        cfg.dynamicSmemBytes = sl;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = K;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int clusters = 0;
        if (cudaOccupancyMaxActiveClusters(&clusters, dr::image_augment_kernel, &cfg) != cudaSuccess || clusters < 1) {
            cudaGetLastError();
            continue;
        }
        const double waves = (double)((n + (uint64_t)clusters - 1) / (uint64_t)clusters);
        const double cost = waves * (double)sl;
        if (!best || cost < best_cost) {
            best = K;
            best_cost = cost;
        }
    }
    if (!best) {   // no occupancy answer: the smallest power of two whose slice fits 32 KB
        best = 1;
        while (best < 8 && img_slice_of(E, best) > 32u * 1024u) best *= 2;
    }
    c_E = E;
    c_n = n;
    c_K = best;
    return best;
}

}  // namespace

extern "C" {

int dr_image_augment(const dr_vision_params* p, uint64_t seed, uint64_t batch_index, int64_t image_offset,
                     const uint8_t* images, int64_t n_images, int32_t height, int32_t width, int32_t channels,
                     float* out, float* img_stats, void* stream) {
    int rc = check_vision(p);
    if (rc != DR_OK) return rc;
    if (height < 1 || width < 1 || channels < 1) return set_error(DR_EINVAL, "height/width/channels: must be >= 1");
    if (n_images < 0 || image_offset < 0 || image_offset + n_images > (int64_t(1) << 32))
        return set_error(DR_EINVAL, "n_images/image_offset: outside [0, 2^32)");
    const uint64_t E = (uint64_t)height * (uint64_t)width * (uint64_t)channels;
    if (E > (uint64_t)DR_VIS_MAX_IMAGE_BYTES)
        return set_error(DR_EUNSUPPORTED, "image of %llu bytes exceeds DR_VIS_MAX_IMAGE_BYTES", (unsigned long long)E);
    if (n_images == 0) return DR_OK;
    if (!images || !out) return set_error(DR_EINVAL, "images/out: NULL");
    if (img_stats && ((uintptr_t)img_stats & 15u)) return set_error(DR_EINVAL, "img_stats: not 16-byte aligned");
    if (n_images * (int64_t)2 > (int64_t)0x7FFFFFFF / 8) return set_error(DR_EINVAL, "n_images: too many for one launch");
    if (!g_img_attr_set) {   // once per process (the attribute is per function, not per launch)
        const cudaError_t ea = cudaFuncSetAttribute(image_augment_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                    (int)IMG_SLICE_MAX);
        if (ea != cudaSuccess) return set_error(DR_ECUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(ea));
        g_img_attr_set = true;
    }
    const uint32_t K = img_cluster_size(E, (uint64_t)n_images);
    const uint32_t slice = img_slice_of(E, K);
    if (slice > IMG_SLICE_MAX) return set_error(DR_EUNSUPPORTED, "image slice of %u bytes too large", slice);
    ImgArgs a{};
    a.images = images;
    a.out = out;
    a.img_stats = img_stats;
    a.E = E;
    a.slice = slice;
    a.aligned = (E % 16 == 0 && ((uintptr_t)images & 15u) == 0 && ((uintptr_t)out & 15u) == 0) ? 1u : 0u;
    a.batch = (uint32_t)batch_index;
    a.image_offset = (uint32_t)image_offset;
    a.contrast_lo = p->contrast_lo;
    a.contrast_range = p->contrast_hi - p->contrast_lo;
    a.noise_lo = p->noise_std_lo;
    a.noise_range = p->noise_std_hi - p->noise_std_lo;
    a.std_floor = p->std_floor;
    a.keys = make_keys(seed);
    // early reads / writes only directly behind the previous augmentation of this stream (the last
    // libdr launch on it): reads when its outputs do not overlap these images (RAW), writes when in
    // addition this call's outputs overlap neither its outputs (WAW) nor its images (WAR); a user
    // kernel in between completes before this call starts (it does not trigger its dependents
    // early), so it needs no check
    const size_t out_bytes = (size_t)n_images * E * 4, st_bytes = img_stats ? (size_t)n_images * 16 : 0;
    const auto disjoint = [](const void* a0, size_t na, const void* b0, size_t nb) {
        const uintptr_t a1 = (uintptr_t)a0, b1 = (uintptr_t)b0;
        return na == 0 || nb == 0 || a1 + na <= b1 || b1 + nb <= a1;
    };
    AugRec prev{};
    const AugRec cur{images, (size_t)n_images * E, out, out_bytes, img_stats, st_bytes};
    const bool early_read = last_launch_is_augment(stream, &prev) &&
                            disjoint(cur.images, cur.img_bytes, prev.out, prev.out_bytes) &&
                            disjoint(cur.images, cur.img_bytes, prev.st, prev.st_bytes);
    const bool early = early_read &&
                       disjoint(cur.out, cur.out_bytes, prev.out, prev.out_bytes) &&
                       disjoint(cur.out, cur.out_bytes, prev.st, prev.st_bytes) &&
                       disjoint(cur.out, cur.out_bytes, prev.images, prev.img_bytes) &&
                       disjoint(cur.st, cur.st_bytes, prev.out, prev.out_bytes) &&
                       disjoint(cur.st, cur.st_bytes, prev.st, prev.st_bytes) &&
                       disjoint(cur.st, cur.st_bytes, prev.images, prev.img_bytes);
    a.early_read = early_read ? 1u : 0u;
    a.early_write = early ? 1u : 0u;
    cudaError_t e = cudaSuccess;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(n_images * K), 1, 1);
    cfg.blockDim = dim3(IMG_THREADS, 1, 1);
    cfg.dynamicSmemBytes = slice;
    cfg.stream = static_cast<cudaStream_t>(stream);
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = K;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // see image_augment_kernel
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    e = cudaLaunchKernelEx(&cfg, image_augment_kernel, a);
    if (e != cudaSuccess) return set_error(DR_ECUDA, "image_augment_kernel: %s", cudaGetErrorString(e));
    count_launch();
    note_stream_launch(stream, &cur);
    return DR_OK;
}

}  // extern "C"

static_assert(sizeof(dr_scene_draw) == 256, "dr_scene_draw must be 64 words");
