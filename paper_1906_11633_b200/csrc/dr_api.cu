// dr_api.cu -- host side of libdr.so: the C-ABI of include/dr.h.
// Validation, workspace layout/allocation (or adoption of a caller-owned PyTorch buffer),
// host-side constant tables (Philox round keys, Bernoulli thresholds, the 65,536-entry
// loguniform force table, the 0.99^k decay table), kernel launches on the library stream.
// There is no CPU fallback: every step of the path runs in the kernels of dr_kernels.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "dr.h"
#include "dr_internal.h"

using namespace dr;

namespace {

struct Layout {
    size_t rec, st, phys, t_tab, rs_phys, rs_src, dec, sync,
        stats, ctl, total;
    uint64_t pitch;
};

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

int device_sm_count() {
    int dev = 0, n = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 148;
}

Layout make_layout(int64_t n_env, int n_phys, int max_ctas) {
    Layout L{};
    L.pitch = align_up((size_t)n_env, TILE);   // envs rounded up to whole tiles
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off = align_up(off + bytes, 256); return o; };
    L.rec = take((size_t)REC_WORDS * L.pitch * 4);    // [n_tiles][REC_GROUPS][TILE][8]
    L.st = take((size_t)ST_PLANES * L.pitch * 4);     // [n_tiles][ST_PLANES][TILE]
    L.phys = take((size_t)n_env * n_phys * 4);
    L.t_tab = take(65536 * 4);
    L.rs_phys = take(MAX_PHYS * 16);
    L.rs_src = take(MAX_PHYS * 4);
    L.dec = take(512 * 8);
    L.stats = take(N_STAT_SLOTS * N_STATS * 8);
    L.ctl = take(8 * 8);
    L.sync = take((N_STAT_SLOTS + 2 * (size_t)max_ctas) * 4);   // done | cta_done | cta_ready
    L.total = off;
    return L;
}

struct Ctx {
    dr_params prm;
    int64_t n_env = 0;
    uint64_t seed = 0;
    int device = 0;
    cudaStream_t stream = nullptr;
    Layout lay{};
    char* ws = nullptr;
    bool owns_ws = false;
    DevPtrs p{};
    double* internal_stats = nullptr;
    int sm_count = 148;
    int max_ctas = 0;
    int step_grid = 1, reset_grid = 1;
    int step_mode = 0;
    uint64_t t_host = 0;
    uint64_t launches = 0;
    bool chain_enabled = true;   // DR_CHAIN
    bool chain_next = false;     // the last library launch on the stream was a step kernel
    // dr_step_host: double-buffered device I/O, H2D / D2H streams and their events
    float* io = nullptr;
    size_t io_bytes = 0;
    cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
    cudaEvent_t ev_h[2] = {nullptr, nullptr}, ev_k[2] = {nullptr, nullptr}, ev_d[2] = {nullptr, nullptr};
    uint64_t host_calls = 0;
};

Ctx* g_ctx = nullptr;
char g_err[512] = "";
bool g_sticky = false;

int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}

int cuda_fail(cudaError_t e, const char* where) {
    g_sticky = true;
    return fail(DR_ECUDA, "%s: %s", where, cudaGetErrorString(e));
}

#define CK(call)                                            \
    do {                                                    \
        cudaError_t _e = (call);                            \
        if (_e != cudaSuccess) return cuda_fail(_e, #call); \
    } while (0)

int validate(const dr_params* p, int64_t n_env) {
    if (!p) return fail(DR_EINVAL, "params: NULL");
    if (p->abi_version != DR_ABI_VERSION) return fail(DR_EINVAL, "abi_version: %u != %u", p->abi_version, DR_ABI_VERSION);
    if (p->struct_size != sizeof(dr_params)) return fail(DR_EINVAL, "struct_size: %u != %zu", p->struct_size, sizeof(dr_params));
    if (p->layer_mask & ~DR_ALL_EXT) return fail(DR_EINVAL, "layer_mask: unknown bits 0x%x", p->layer_mask);
    if ((p->layer_mask & DR_SUBSTEP_BACKLASH) && !(p->layer_mask & DR_BACKLASH))
        return fail(DR_EINVAL, "layer_mask: DR_SUBSTEP_BACKLASH needs DR_BACKLASH");
    if (!(p->act_smooth_coef >= 0.0 && p->act_smooth_coef <= 1.0)) return fail(DR_EINVAL, "act_smooth_coef: outside [0, 1]");
    if (p->n_act != DR_N_ACT || p->n_tips != DR_N_TIPS || p->n_substeps != DR_N_SUBSTEPS)
        return fail(DR_EUNSUPPORTED, "n_act/n_tips/n_substeps: kernels specialise (20, 5, 10)");
    if (n_env < 1 || n_env > (int64_t(1) << 31)) return fail(DR_EINVAL, "n_env: %lld outside [1, 2^31]", (long long)n_env);
    const int64_t ng = p->n_env_global ? p->n_env_global : n_env;
    if (p->env_offset < 0 || p->env_offset + n_env > ng || ng > (int64_t(1) << 32))
        return fail(DR_EINVAL, "env_offset/n_env_global: shard [%lld, %lld) outside [0, %lld)",
                    (long long)p->env_offset, (long long)(p->env_offset + n_env), (long long)ng);
    struct { const char* n; double v; } stds[] = {
        {"act_sigma_uadd", p->act_sigma_uadd}, {"act_sigma_cadd", p->act_sigma_cadd},
        {"act_sigma_mult", p->act_sigma_mult}, {"delta_jitter_std", p->delta_jitter_std},
        {"tip_corr", p->tip_corr}, {"tip_uncorr", p->tip_uncorr}, {"obj_corr", p->obj_corr},
        {"obj_uncorr", p->obj_uncorr}, {"rot_corr", p->rot_corr}, {"rot_uncorr", p->rot_uncorr},
        {"tip_marker", p->tip_marker}, {"base_marker", p->base_marker},
        {"force_accel_std", p->force_accel_std}, {"backlash_eps", p->backlash_eps},
        {"dropout_rate_hz", p->dropout_rate_hz}, {"occl_dist", p->occl_dist}};
    for (auto& s : stds)
        if (!(s.v >= 0.0) || !std::isfinite(s.v)) return fail(DR_EINVAL, "%s: must be a finite value >= 0", s.n);
    // The kernels evaluate the backlash gate as alpha = eps / (|s' - s| + eps) whenever num < den
    // (dr_step.cuh backlash_alpha): exact only while s' can sit within eps of a rail by landing on
    // it, i.e. for eps below the fp32 spacing just inside +-1 (2^-24 ~ 6e-8).  The paper's eps is
    // 1e-12.
    if (!(p->backlash_eps <= 1e-8)) return fail(DR_EINVAL, "backlash_eps: must be <= 1e-8 (the paper's is 1e-12)");
    if (!(p->delay_prob >= 0.0 && p->delay_prob <= 1.0)) return fail(DR_EINVAL, "delay_prob: outside [0, 1]");
    if (!(p->dt_base > 0.0)) return fail(DR_EINVAL, "dt_base: must be > 0");
    if (!(p->step_nominal > 0.0)) return fail(DR_EINVAL, "step_nominal: must be > 0");
    if (!(p->lambda_lo > 0.0 && p->lambda_lo <= p->lambda_hi && std::isfinite(p->lambda_hi)))
        return fail(DR_EINVAL, "lambda_lo/lambda_hi: need 0 < lo <= hi");
    for (int j = 0; j < DR_N_ACT; ++j) {
        if (!(p->delta_cal_neg[j] >= 0.0)) return fail(DR_EINVAL, "delta_cal_neg[%d]: must be >= 0", j);
        if (!(p->delta_cal_pos[j] >= 0.0)) return fail(DR_EINVAL, "delta_cal_pos[%d]: must be >= 0", j);
    }
    if (p->dropout_hold_steps < 0 || p->dropout_hold_steps > 15) return fail(DR_EINVAL, "dropout_hold_steps: outside [0, 15]");
    if (!(p->force_p_lo > 0.0 && p->force_p_lo <= p->force_p_hi && p->force_p_hi <= 1.0))
        return fail(DR_EINVAL, "force_p_lo/force_p_hi: need 0 < lo <= hi <= 1");
    if (!(p->force_decay_per_step > 0.0 && p->force_decay_per_step <= 1.0))
        return fail(DR_EINVAL, "force_decay_per_step: outside (0, 1]");
    if (p->n_phys < 1 || p->n_phys > DR_MAX_PHYS) return fail(DR_EINVAL, "n_phys: outside [1, 256]");
    if (p->mass_index < 0 || p->mass_index >= p->n_phys) return fail(DR_EINVAL, "mass_index: outside [0, n_phys)");
    if (!(p->phys[p->mass_index].base > 0.0)) return fail(DR_EINVAL, "phys[mass_index].base: mass must be > 0");
    for (int i = 0; i < p->n_phys; ++i) {
        const dr_phys_desc& d = p->phys[i];
        if (d.kind > DR_PHYS_MUL_LOGNORMAL) return fail(DR_EINVAL, "phys[%d].kind: unknown %u", i, d.kind);
        if ((d.kind == DR_PHYS_UNIFORM_SCALE) && !(d.a <= d.b)) return fail(DR_EINVAL, "phys[%d]: lo > hi", i);
        if ((d.kind == DR_PHYS_LOGUNIFORM_SCALE) && !(d.a > 0.0 && d.a <= d.b))
            return fail(DR_EINVAL, "phys[%d]: loguniform needs 0 < lo <= hi", i);
        if ((d.kind == DR_PHYS_ADD_GAUSS || d.kind == DR_PHYS_MUL_LOGNORMAL) && !(d.a >= 0.0))
            return fail(DR_EINVAL, "phys[%d]: std < 0", i);
    }
    if (p->workspace && ((uintptr_t)p->workspace % 256)) return fail(DR_EINVAL, "workspace: not 256-byte aligned");
    return DR_OK;
}

// Bernoulli threshold floor(p * 2^32) for the exact integer decision x < T.
unsigned long long bernoulli_threshold(double p) {
    if (!(p > 0.0)) return 0ull;
    if (p >= 1.0) return 1ull << 32;
    return (unsigned long long)std::floor(p * 4294967296.0);
}

// Host-side constants and tables of parameter set p (Philox round keys, Bernoulli thresholds,
// the loguniform force table, the decay table, the reset task tables and physics coefficients),
// uploaded in stream order on the library stream: kernels enqueued before see the previous set,
// kernels enqueued after see p.  Used by dr_init and dr_update_params.
cudaError_t upload_params(Ctx* c, const dr_params& p, const char** what) {
    // ---- host-side constants ----
    DevConst dc{};
    dc.layer_mask = p.layer_mask;
    dc.n_env = (uint32_t)c->n_env;
    dc.pitch = c->lay.pitch;
    dc.env_offset = (uint32_t)p.env_offset;
    dc.hold_steps = (uint32_t)p.dropout_hold_steps;
    const uint32_t k0 = (uint32_t)(c->seed & 0xFFFFFFFFull), k1 = (uint32_t)(c->seed >> 32);
    for (int r = 0; r < 10; ++r) {   // Philox key schedule: key + r * (W0, W1)
        dc.rk0[r] = k0 + (uint32_t)r * 0x9E3779B9u;
        dc.rk1[r] = k1 + (uint32_t)r * 0xBB67AE85u;
    }
    dc.t_delay = bernoulli_threshold(p.delay_prob);
    dc.t_drop = bernoulli_threshold(1.0 - std::exp(-p.dropout_rate_hz * p.step_nominal));  // Q11
    dc.su = (float)p.act_sigma_uadd;
    dc.sc = (float)p.act_sigma_cadd;
    dc.sm = (float)p.act_sigma_mult;
    dc.dt_base = (float)p.dt_base;
    dc.lam_lo = (float)p.lambda_lo;
    dc.lam_range = (float)(p.lambda_hi - p.lambda_lo);
    for (int j = 0; j < DR_N_ACT; ++j) {
        dc.dcal_neg[j] = (float)p.delta_cal_neg[j];
        dc.dcal_pos[j] = (float)p.delta_cal_pos[j];
    }
    dc.jitter = (float)p.delta_jitter_std;
    dc.eps = (float)p.backlash_eps;
    dc.tip_corr = (float)p.tip_corr;
    dc.tip_uncorr = (float)p.tip_uncorr;
    dc.obj_corr = (float)p.obj_corr;
    dc.obj_uncorr = (float)p.obj_uncorr;
    dc.rot_corr = (float)p.rot_corr;
    dc.rot_uncorr = (float)p.rot_uncorr;
    dc.tip_marker = (float)p.tip_marker;
    dc.base_marker = (float)p.base_marker;
    dc.base_to_tips = p.base_marker_to_tips ? 1 : 0;
    dc.occl_on = p.occl_dist > 0.0 ? 1 : 0;
    dc.occl_r2 = p.occl_dist * p.occl_dist;
    dc.occl_r2_lo = (float)(dc.occl_r2 * (1.0 - 1e-5));
    dc.occl_r2_hi = (float)(dc.occl_r2 * (1.0 + 1e-5));
    dc.occl_exact_only = (dc.occl_r2 < 1e-30 || dc.occl_r2 > 1e30) ? 1u : 0u;
    dc.accel_std = (float)p.force_accel_std;
    dc.smooth_c = (float)p.act_smooth_coef;
    dc.smooth_keep = (float)(1.0 - p.act_smooth_coef);
    {
        // moment slots 16..23: bound each job total (n_env_global x a per-env-step bound x 4) and
        // round CTA sums to 2^-k with bound * 2^k < 2^52, so fp64 atomic sums are exact
        double mass_max = 0.0;
        {
            const dr_phys_desc& d = p.phys[p.mass_index];
            const bool on = (p.layer_mask & DR_PHYS) != 0;
            switch (on ? d.kind : (uint32_t)DR_PHYS_FIXED) {
            case DR_PHYS_UNIFORM_SCALE: mass_max = d.base * std::max(std::fabs(d.a), std::fabs(d.b)); break;
            case DR_PHYS_LOGUNIFORM_SCALE: mass_max = d.base * d.b; break;
            case DR_PHYS_ADD_GAUSS: mass_max = std::fabs(d.base) + 6.0 * d.a; break;
            case DR_PHYS_MUL_LOGNORMAL: mass_max = d.base * std::exp(6.0 * d.a); break;
            default: mass_max = std::fabs(d.base); break;
            }
        }
        const double z2 = 36.0;   // |z| <= sqrt(-2 ln 2^-24) < 6
        const double dtmax = 10.0 * (p.dt_base + 17.0 / p.lambda_lo);
        const double fmax = mass_max * p.force_accel_std * 6.0;
        const double per_env[8] = {dtmax, dtmax * dtmax, 40.0, 80.0, 20.0, 20.0 * z2, 15.0 * z2, 3.0 * fmax * fmax};
        const double ng = (double)(p.n_env_global ? p.n_env_global : c->n_env);
        for (int i = 0; i < 8; ++i) {
            const double bound = std::max(ng * per_env[i] * 4.0, 1.0);
            const int k = 52 - (int)std::ceil(std::log2(bound));
            dc.mq_scale[i] = std::ldexp(1.0, k);
            dc.mq_inv[i] = std::ldexp(1.0, -k);
        }
    }
    dc.n_phys = p.n_phys;
    dc.mass_index = p.mass_index;

    int nu = 0, nn = 0;   // uniform-kind / normal-kind parameter counts (draw ranks)
    for (int i = 0; i < p.n_phys; ++i) {
        const uint32_t kd = p.phys[i].kind;
        if (kd == DR_PHYS_UNIFORM_SCALE || kd == DR_PHYS_LOGUNIFORM_SCALE) ++nu;
        else if (kd == DR_PHYS_ADD_GAUSS || kd == DR_PHYS_MUL_LOGNORMAL) ++nn;
    }
    dc.n_phys_u = nu;
    dc.n_phys_n = nn;

    const uint32_t lm = p.layer_mask;
    // physics: v = C0 + C1 * f(A + B x) (dr_internal.h), f = 2^(.) for the exp kinds (A, B in log2 units)
    std::vector<float> rphys(MAX_PHYS * 4, 0.f);
    std::vector<uint32_t> rsrc(MAX_PHYS, 0u);
    {
        int u = 0, n = 0;
        for (int i = 0; i < p.n_phys; ++i) {
            const dr_phys_desc& d = p.phys[i];
            float A = 0.f, B = 0.f, C0 = (float)d.base, C1 = 0.f;
            uint32_t src = RS_OFF_ZERO;
            const bool on_phys = (lm & DR_PHYS) != 0;
            switch (d.kind) {
            case DR_PHYS_UNIFORM_SCALE:   // base * (a + (b - a) U)
                if (on_phys) { A = (float)d.a; B = (float)(d.b - d.a); C0 = 0.f; C1 = (float)d.base; src = rs_slot((uint32_t)u); }
                ++u;
                break;
            case DR_PHYS_LOGUNIFORM_SCALE:   // base * exp(ln a + (ln b - ln a) U) = base * 2^(log2 a + log2(b/a) U)
                if (on_phys) {
                    A = (float)std::log2(d.a); B = (float)(std::log2(d.b) - std::log2(d.a)); C0 = 0.f; C1 = (float)d.base;
                    src = rs_slot((uint32_t)u) | RS_EXP;
                }
                ++u;
                break;
            case DR_PHYS_ADD_GAUSS:   // base + sigma z
                if (on_phys) { B = (float)d.a; C0 = (float)d.base; C1 = 1.f; src = RS_OFF_NORMAL + rs_slot((uint32_t)n); }
                ++n;
                break;
            case DR_PHYS_MUL_LOGNORMAL:   // base * exp(sigma z) = base * 2^(sigma log2(e) z)
                if (on_phys) {
                    B = (float)(d.a * 1.4426950408889634074); C0 = 0.f; C1 = (float)d.base;
                    src = (RS_OFF_NORMAL + rs_slot((uint32_t)n)) | RS_EXP;
                }
                ++n;
                break;
            default:   // FIXED
                break;
            }
            rphys[4 * i + 0] = A;
            rphys[4 * i + 1] = B;
            rphys[4 * i + 2] = C0;
            rphys[4 * i + 3] = C1;
            rsrc[i] = src;
        }
    }
    // loguniform force probability quantised to 65,536 midpoints of ln p (Q19)
    std::vector<uint32_t> ttab(65536);
    {
        const double llo = std::log(p.force_p_lo), lhi = std::log(p.force_p_hi);
        for (uint32_t j = 0; j < 65536u; ++j) {
            const double pj = std::exp(llo + (((double)j + 0.5) / 65536.0) * (lhi - llo));
            const unsigned long long T = bernoulli_threshold(pj);
            ttab[j] = (uint32_t)(T > 0xFFFFFFFFull ? 0xFFFFFFFFull : T);
        }
    }
    // decay 0.99^k = dec[k & 255] * dec[256 + (k >> 8)], fp64 (Q17)
    std::vector<double> dec(512);
    for (int j = 0; j < 256; ++j) {
        dec[j] = std::pow(p.force_decay_per_step, (double)j);
        dec[256 + j] = std::pow(p.force_decay_per_step, 256.0 * j);
    }
    cudaStream_t s = c->stream;
    cudaError_t e;
    const DevPtrs& P = c->p;
    if ((e = upload_const(dc, s)) != cudaSuccess) { *what = "upload_const"; return e; };
    if ((e = cudaMemcpyAsync(P.t_tab, ttab.data(), 65536 * 4, cudaMemcpyHostToDevice, s)) != cudaSuccess) { *what = "memcpy t_tab"; return e; };
    if ((e = cudaMemcpyAsync(P.rs_phys, rphys.data(), MAX_PHYS * 16, cudaMemcpyHostToDevice, s)) != cudaSuccess) { *what = "memcpy rs_phys"; return e; };
    if ((e = cudaMemcpyAsync(P.rs_src, rsrc.data(), MAX_PHYS * 4, cudaMemcpyHostToDevice, s)) != cudaSuccess) { *what = "memcpy rs_src"; return e; };
    if ((e = cudaMemcpyAsync(P.dec_tab, dec.data(), 512 * 8, cudaMemcpyHostToDevice, s)) != cudaSuccess) { *what = "memcpy dec"; return e; };
    return cudaSuccess;
}

bool aligned16(const void* q) { return ((uintptr_t)q & 15u) == 0; }

uint64_t g_total_launches = 0;   // every libdr kernel launch of the process (context or not)

}  // namespace

namespace dr {
int set_error(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}
void count_launch() {
    ++g_total_launches;
    if (g_ctx) g_ctx->launches++;
}
// Per-stream record of the last libdr launch (a small table; a stream missing from it reads as
// "not an augmentation", the conservative answer).  Every libdr launch goes through here.
namespace {
struct StreamLast {
    bool used = false;
    void* stream = nullptr;
    int kind = LAUNCH_OTHER;
    AugRec rec{};
};
StreamLast g_stream_last[8];
int g_stream_next = 0;
StreamLast* stream_slot(void* stream) {
    for (auto& sl : g_stream_last)
        if (sl.used && sl.stream == stream) return &sl;
    return nullptr;
}
}  // namespace
void note_stream_launch(void* stream, const AugRec* aug, int kind) {
    StreamLast* sl = stream_slot(stream);
    if (!sl) {
        sl = &g_stream_last[g_stream_next];
        g_stream_next = (g_stream_next + 1) % 8;
    }
    sl->used = true;
    sl->stream = stream;
    sl->kind = aug ? LAUNCH_AUGMENT : kind;
    if (aug) sl->rec = *aug;
    // a chained step (no griddepcontrol.wait) may only follow a step of its context directly: the
    // augmentation triggers its dependents at once, so a step behind it must wait for the grid
    if (aug && g_ctx && static_cast<void*>(g_ctx->stream) == stream) g_ctx->chain_next = false;
}
bool last_launch_is_augment(void* stream, AugRec* prev) {
    const StreamLast* sl = stream_slot(stream);
    if (!sl || sl->kind != LAUNCH_AUGMENT) return false;
    *prev = sl->rec;
    return true;
}
int last_launch_kind(void* stream) {
    const StreamLast* sl = stream_slot(stream);
    return sl ? sl->kind : LAUNCH_UNKNOWN;
}
}  // namespace dr

extern "C" {

uint32_t dr_abi_version(void) { return DR_ABI_VERSION; }

const char* dr_last_error(void) { return g_err; }

int dr_params_default(dr_params* p) {
    if (!p) return fail(DR_EINVAL, "params: NULL");
    std::memset(p, 0, sizeof(*p));
    p->abi_version = DR_ABI_VERSION;
    p->struct_size = sizeof(dr_params);
    p->layer_mask = DR_ALL;
    p->n_act = DR_N_ACT;
    p->n_tips = DR_N_TIPS;
    p->n_substeps = DR_N_SUBSTEPS;
    // Table action-noise: % of the action range 2 (Q8)
    p->act_sigma_uadd = 0.10;
    p->act_sigma_cadd = 0.03;
    p->act_sigma_mult = 0.015;
    p->delay_prob = 0.5;
    p->dt_base = 0.008;
    p->lambda_lo = 1250.0;
    p->lambda_hi = 10000.0;
    p->step_nominal = 0.08;
    for (int j = 0; j < DR_N_ACT; ++j) {   // calibrated widths: not given, Q21
        p->delta_cal_neg[j] = 3.5 + 0.1 * j;
        p->delta_cal_pos[j] = 4.0 + 0.1 * j;
    }
    p->delta_jitter_std = 0.1;
    p->backlash_eps = 1e-12;
    // Table obs-noise
    p->tip_corr = 1e-3;
    p->tip_uncorr = 2e-3;
    p->obj_corr = 5e-3;
    p->obj_uncorr = 1e-3;
    p->rot_corr = 0.1;
    p->rot_uncorr = 0.1;
    p->tip_marker = 3e-3;
    p->base_marker = 1e-3;
    p->base_marker_to_tips = 1;            // Q14
    p->dropout_hold_steps = 13;            // ceil(1 s / 80 ms), Q11
    p->dropout_rate_hz = 0.2;
    p->occl_dist = 0.015;                  // Q13
    p->force_p_lo = 0.001;
    p->force_p_hi = 0.1;
    p->force_accel_std = 1.0;
    p->force_decay_per_step = 0.99;
    p->act_smooth_coef = 0.3;              // PAPER.md:743 footnote (DR_SMOOTH, off by default)
    // physical parameters: the paper's table is missing; synthetic 256 slots, Q20
    p->n_phys = DR_MAX_PHYS;
    p->mass_index = 0;
    for (int i = 0; i < DR_MAX_PHYS; ++i) {
        dr_phys_desc& d = p->phys[i];
        d.base = 0.5 + 0.01 * i;
        switch (i % 4) {
        case 0: d.kind = DR_PHYS_UNIFORM_SCALE; d.a = 0.5; d.b = 1.5; break;
        case 1: d.kind = DR_PHYS_LOGUNIFORM_SCALE; d.a = 0.3; d.b = 3.0; break;
        case 2: d.kind = DR_PHYS_ADD_GAUSS; d.a = 0.15; d.b = 0.0; break;
        default: d.kind = DR_PHYS_MUL_LOGNORMAL; d.a = 0.2; d.b = 0.0; break;
        }
    }
    return DR_OK;
}

size_t dr_workspace_bytes(const dr_params* params, int64_t n_env) {
    if (!params || n_env < 1 || params->n_phys < 1 || params->n_phys > DR_MAX_PHYS) return 0;
    return make_layout(n_env, params->n_phys, device_sm_count() * 32).total;
}

int dr_init(const dr_params* params, int64_t n_env, uint64_t seed) {
    if (g_ctx) return fail(DR_EALREADY, "dr_init: context already initialised (call dr_finalize)");
    int rc = validate(params, n_env);
    if (rc != DR_OK) return rc;
    g_sticky = false;
    Ctx* c = new Ctx();
    c->prm = *params;
    if (c->prm.n_env_global == 0) c->prm.n_env_global = n_env;
    c->n_env = n_env;
    c->seed = seed;
    c->stream = static_cast<cudaStream_t>(params->stream);
    cudaError_t e = cudaGetDevice(&c->device);
    if (e != cudaSuccess) { delete c; return cuda_fail(e, "cudaGetDevice"); }
    c->sm_count = device_sm_count();
    c->max_ctas = c->sm_count * 32;
    c->lay = make_layout(n_env, params->n_phys, c->max_ctas);
    if (params->workspace) {
        if (params->workspace_bytes < c->lay.total) {
            size_t need = c->lay.total;
            delete c;
            return fail(DR_ENOMEM, "workspace_bytes: %zu < required %zu", params->workspace_bytes, need);
        }
        c->ws = static_cast<char*>(params->workspace);
        c->owns_ws = false;
    } else {
        e = cudaMalloc(&c->ws, c->lay.total);
        if (e != cudaSuccess) { delete c; return fail(DR_ENOMEM, "cudaMalloc(%zu): %s", c->lay.total, cudaGetErrorString(e)); }
        c->owns_ws = true;
    }
    const Layout& L = c->lay;
    DevPtrs& P = c->p;
    P.rec = reinterpret_cast<uint32_t*>(c->ws + L.rec);
    P.st = reinterpret_cast<uint32_t*>(c->ws + L.st);
    P.phys = reinterpret_cast<float*>(c->ws + L.phys);
    P.t_tab = reinterpret_cast<uint32_t*>(c->ws + L.t_tab);
    P.rs_phys = reinterpret_cast<float4*>(c->ws + L.rs_phys);
    P.rs_src = reinterpret_cast<uint32_t*>(c->ws + L.rs_src);
    P.dec_tab = reinterpret_cast<double*>(c->ws + L.dec);
    P.stats = reinterpret_cast<double*>(c->ws + L.stats);
    P.ctl = reinterpret_cast<unsigned long long*>(c->ws + L.ctl);
    P.done = reinterpret_cast<uint32_t*>(c->ws + L.sync);
    P.cta_done = P.done + N_STAT_SLOTS;
    P.cta_ready = P.cta_done + c->max_ctas;
    c->internal_stats = P.stats;

    cudaStream_t s = c->stream;
    auto bail = [&](cudaError_t err, const char* what) {
        if (c->owns_ws) cudaFree(c->ws);
        delete c;
        return cuda_fail(err, what);
    };
    const char* what = "";
    if ((e = upload_params(c, c->prm, &what)) != cudaSuccess) return bail(e, what);
    if ((e = cudaMemsetAsync(P.stats, 0, N_STAT_SLOTS * N_STATS * 8, s)) != cudaSuccess) return bail(e, "memset stats");
    if ((e = cudaMemsetAsync(P.ctl, 0, 8 * 8, s)) != cudaSuccess) return bail(e, "memset ctl");
    // state planes start zeroed so that never-reset lanes of a partial tile stay defined
    if ((e = cudaMemsetAsync(P.st, 0, (size_t)ST_PLANES * L.pitch * 4, s)) != cudaSuccess) return bail(e, "memset st");
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return bail(e, "sync init");

    // A/B knobs, read at every dr_init (unset = the defaults)
    // step mode by the job size (n_env_global, so every shard of a job runs the same kernel and
    // per-env results stay bit-identical across GPU counts); DR_STEP_MODE=throughput|latency forces
    const char* sm = std::getenv("DR_STEP_MODE");
    int mode = (c->prm.n_env_global <= LAT_MAX_ENVS) ? 1 : 0;
    if (sm && std::strcmp(sm, "throughput") == 0) mode = 0;
    if (sm && std::strcmp(sm, "latency") == 0) mode = 1;
    set_step_mode(mode);
    c->step_mode = mode;
    const int occ_step = step_max_ctas_per_sm(c->prm.layer_mask);
    const uint32_t units = mode ? (uint32_t)((n_env + LAT_ENVS_PER_CTA - 1) / LAT_ENVS_PER_CTA)
                                : (uint32_t)((n_env + TILE - 1) / TILE);
    // Persistent grid of min(units, resident slots) CTAs, the slots a multiple of the SM count: unit i
    // runs on CTA i % grid, i.e. on SM i % 148, so every SM gets the same number of units (+-1) even
    // when the CTAs do not (the fewest-waves grid ceil(units / waves) -- equal units per CTA but 3 or
    // 4 CTAs per SM -- measured slower, profiles/round2_notes.md).
    const long long slots = std::min<long long>((long long)c->sm_count * occ_step, (long long)c->max_ctas);
    c->step_grid = (int)std::min<long long>((long long)units, slots);
    // A/B: persistent grid size (clamped to the default). 1M envs: 592 (default) 4.90e9, 586 4.89e9,
    // 546 4.75e9, 512 4.60e9, 444 4.73e9 env-steps/s
    if (const char* sg = std::getenv("DR_STEP_GRID")) {
        const int v = std::atoi(sg);
        if (v >= 1 && v < c->step_grid) c->step_grid = v;
    }
    const char* pdl = std::getenv("DR_PDL");
    set_pdl(!(pdl && std::atoi(pdl) == 0));
    c->reset_grid = reset_grid_for((uint32_t)n_env, c->sm_count);
    // chained steps (dr_step.cuh): back-to-back dr_step calls overlap at their boundary; DR_CHAIN=0
    // (A/B) makes every step wait for its predecessor to complete
    const char* ch = std::getenv("DR_CHAIN");
    c->chain_enabled = !(ch && std::atoi(ch) == 0);
    c->chain_next = false;

    // the step protocol at t = 0, then episode 0 for every env (sampled at the
    // beginning of every episode)
    if ((e = launch_sync_init(P, 0, c->step_grid, c->max_ctas, s)) != cudaSuccess)
        return bail(e, "sync_init_kernel");
    if ((e = launch_reset(P, nullptr, true, (uint32_t)n_env, c->reset_grid, s)) != cudaSuccess) return bail(e, "reset_kernel");
    c->launches = 2;
    g_total_launches += 2;
    note_stream_launch(s, nullptr);
    g_ctx = c;
    g_err[0] = 0;
    return DR_OK;
}

int dr_update_params(const dr_params* params) {
    Ctx* c = g_ctx;
    if (!c) return fail(DR_ENOTINIT, "dr_update_params: no context");
    if (g_sticky) return fail(DR_ECUDA, "sticky CUDA error: %s", g_err);
    int rc = validate(params, c->n_env);
    if (rc != DR_OK) return rc;
    // what the context's shape, kernels and memory depend on cannot change without dr_init
    if (params->layer_mask != c->prm.layer_mask)
        return fail(DR_EINVAL, "layer_mask: cannot change on update (0x%x != 0x%x)", params->layer_mask, c->prm.layer_mask);
    if (params->n_phys != c->prm.n_phys) return fail(DR_EINVAL, "n_phys: cannot change on update");
    const int64_t ng = params->n_env_global ? params->n_env_global : c->n_env;
    if (params->env_offset != c->prm.env_offset || ng != c->prm.n_env_global)
        return fail(DR_EINVAL, "env_offset/n_env_global: cannot change on update");
    dr_params np = *params;
    np.n_env_global = c->prm.n_env_global;
    np.workspace = c->prm.workspace;           // memory and stream stay the context's
    np.workspace_bytes = c->prm.workspace_bytes;
    np.stream = c->prm.stream;
    const char* what = "";
    cudaError_t e = upload_params(c, np, &what);
    if (e != cudaSuccess) return cuda_fail(e, what);
    c->prm = np;
    return DR_OK;
}

int dr_reset(const uint8_t* env_mask) {
    Ctx* c = g_ctx;
    if (!c) return fail(DR_ENOTINIT, "dr_reset: no context");
    if (g_sticky) return fail(DR_ECUDA, "sticky CUDA error: %s", g_err);
    // the scan may overlap the previous kernel only if that is a step (it writes neither masks nor
    // episode counters); behind anything else (another reset: episode counters) the reset waits first
    const bool early_scan = last_launch_kind(static_cast<void*>(c->stream)) == LAUNCH_STEP;
    cudaError_t e = launch_reset(c->p, env_mask, false, (uint32_t)c->n_env, c->reset_grid, c->stream, early_scan);
    if (e != cudaSuccess) return cuda_fail(e, "reset_kernel");
    c->chain_next = false;   // the next step must wait for the reset to complete
    c->launches++;
    ++g_total_launches;
    note_stream_launch(c->stream, nullptr);
    return DR_OK;
}

static int step_common(const float* actions, const float* raw_obs, float* out_actions, float* out_sub, float* out_obs,
                       float* out_dt, float* out_force) {
    Ctx* c = g_ctx;
    if (!c) return fail(DR_ENOTINIT, "dr_step: no context");
    if (g_sticky) return fail(DR_ECUDA, "sticky CUDA error: %s", g_err);
    const bool sub = (c->prm.layer_mask & DR_SUBSTEP_BACKLASH) != 0;
    if (sub != (out_sub != nullptr))
        return fail(DR_EINVAL, sub ? "DR_SUBSTEP_BACKLASH context: use dr_step_substeps"
                                   : "dr_step_substeps: context has no DR_SUBSTEP_BACKLASH layer");
    const void* ptrs[7] = {actions, raw_obs, out_actions, out_obs, out_dt, out_force, sub ? out_sub : actions};
    const char* names[7] = {"actions", "raw_obs", "out_actions", "out_obs", "out_dt", "out_force", "out_actions_sub"};
    for (int i = 0; i < 7; ++i) {
        if (!ptrs[i]) return fail(DR_EINVAL, "%s: NULL", names[i]);
        if (!aligned16(ptrs[i])) return fail(DR_EINVAL, "%s: not 16-byte aligned", names[i]);
    }
    set_step_mode(c->step_mode);
    const int chain = (c->chain_enabled && c->chain_next) ? 1 : 0;
    cudaError_t e = launch_step(c->p, c->prm.layer_mask, actions, raw_obs, out_actions, out_obs, out_dt, out_force,
                                out_sub, (uint32_t)c->n_env, c->step_grid, chain, c->stream);
    if (e != cudaSuccess) return cuda_fail(e, "step_kernel");
    c->chain_next = true;
    c->t_host++;
    c->launches++;
    ++g_total_launches;
    note_stream_launch(c->stream, nullptr, LAUNCH_STEP);
    return DR_OK;
}

int dr_step(const float* actions, const float* raw_obs, float* out_actions, float* out_obs, float* out_dt,
            float* out_force) {
    return step_common(actions, raw_obs, out_actions, nullptr, out_obs, out_dt, out_force);
}

int dr_step_substeps(const float* actions, const float* raw_obs, float* out_actions, float* out_actions_sub,
                     float* out_obs, float* out_dt, float* out_force) {
    if (!out_actions_sub) return fail(DR_EINVAL, "out_actions_sub: NULL");
    return step_common(actions, raw_obs, out_actions, out_actions_sub, out_obs, out_dt, out_force);
}

// End-to-end step on host buffers, pipelined over consecutive calls: the H2D copy of call t runs on
// its own stream into device buffer set t % 2 (after kernel t-2 released it), the kernel waits for
// that copy and for the D2H of call t-2 (which frees output set t % 2), and the D2H of call t runs
// on a third stream -- so with back-to-back calls, inputs of t+1 go up while outputs of t come
// down (PCIe is full duplex) and kernel t+1 computes.
int dr_step_host(const float* actions, const float* raw_obs, float* out_actions, float* out_obs, float* out_dt,
                 float* out_force) {
    Ctx* c = g_ctx;
    if (!c) return fail(DR_ENOTINIT, "dr_step_host: no context");
    if (g_sticky) return fail(DR_ECUDA, "sticky CUDA error: %s", g_err);
    if (!actions || !raw_obs || !out_actions || !out_obs || !out_dt || !out_force)
        return fail(DR_EINVAL, "dr_step_host: NULL buffer");
    if (c->prm.layer_mask & DR_SUBSTEP_BACKLASH)
        return fail(DR_EINVAL, "dr_step_host: DR_SUBSTEP_BACKLASH contexts need dr_step_substeps on device buffers");
    const size_t n = (size_t)c->n_env;
    const size_t fa = n * N_ACT, fo = n * OBS_IN, foa = n * N_ACT, foo = n * OBS_OUT, fdt = n * N_SUB, ff = n * 3;
    auto up16 = [](size_t f) { return (f + 3) / 4 * 4; };
    const size_t set_floats = up16(fa) + up16(fo) + up16(foa) + up16(foo) + up16(fdt) + up16(ff);
    if (!c->io) {
        CK(cudaMalloc(&c->io, 2 * set_floats * 4));
        c->io_bytes = 2 * set_floats * 4;
        CK(cudaStreamCreateWithFlags(&c->s_h2d, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&c->s_d2h, cudaStreamNonBlocking));
        for (int i = 0; i < 2; ++i) {
            CK(cudaEventCreateWithFlags(&c->ev_h[i], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&c->ev_k[i], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&c->ev_d[i], cudaEventDisableTiming));
        }
        c->host_calls = 0;
    }
    const uint64_t t = c->host_calls;
    const int b = (int)(t & 1u);
    float* d_a = c->io + (size_t)b * set_floats;
    float* d_o = d_a + up16(fa);
    float* d_oa = d_o + up16(fo);
    float* d_oo = d_oa + up16(foa);
    float* d_dt = d_oo + up16(foo);
    float* d_f = d_dt + up16(fdt);
    // inputs of call t: after kernel t-2 is done reading this set
    if (t >= 2) CK(cudaStreamWaitEvent(c->s_h2d, c->ev_k[b], 0));
    // host buffers laid out back to back (one allocation, as the device set is): one copy each way
    const bool in_one = raw_obs == actions + fa && d_o == d_a + fa;
    const bool out_one = out_obs == out_actions + foa && out_dt == out_obs + foo && out_force == out_dt + fdt &&
                         d_oo == d_oa + foa && d_dt == d_oo + foo && d_f == d_dt + fdt;
    if (in_one) {
        CK(cudaMemcpyAsync(d_a, actions, (fa + fo) * 4, cudaMemcpyHostToDevice, c->s_h2d));
    } else {
        CK(cudaMemcpyAsync(d_a, actions, fa * 4, cudaMemcpyHostToDevice, c->s_h2d));
        CK(cudaMemcpyAsync(d_o, raw_obs, fo * 4, cudaMemcpyHostToDevice, c->s_h2d));
    }
    CK(cudaEventRecord(c->ev_h[b], c->s_h2d));
    // the step: after its inputs landed and the outputs of call t-2 left this set
    CK(cudaStreamWaitEvent(c->stream, c->ev_h[b], 0));
    if (t >= 2) CK(cudaStreamWaitEvent(c->stream, c->ev_d[b], 0));
    int rc = dr_step(d_a, d_o, d_oa, d_oo, d_dt, d_f);
    if (rc != DR_OK) return rc;
    CK(cudaEventRecord(c->ev_k[b], c->stream));
    // outputs of call t
    CK(cudaStreamWaitEvent(c->s_d2h, c->ev_k[b], 0));
    if (out_one) {
        CK(cudaMemcpyAsync(out_actions, d_oa, (foa + foo + fdt + ff) * 4, cudaMemcpyDeviceToHost, c->s_d2h));
    } else {
        CK(cudaMemcpyAsync(out_actions, d_oa, foa * 4, cudaMemcpyDeviceToHost, c->s_d2h));
        CK(cudaMemcpyAsync(out_obs, d_oo, foo * 4, cudaMemcpyDeviceToHost, c->s_d2h));
        CK(cudaMemcpyAsync(out_dt, d_dt, fdt * 4, cudaMemcpyDeviceToHost, c->s_d2h));
        CK(cudaMemcpyAsync(out_force, d_f, ff * 4, cudaMemcpyDeviceToHost, c->s_d2h));
    }
    CK(cudaEventRecord(c->ev_d[b], c->s_d2h));
    c->host_calls = t + 1;
    return DR_OK;
}

int dr_finalize(void) {
    Ctx* c = g_ctx;
    if (!c) return fail(DR_ENOTINIT, "dr_finalize: no context");
    cudaStreamSynchronize(c->stream);
    if (c->s_h2d) cudaStreamSynchronize(c->s_h2d);
    if (c->s_d2h) cudaStreamSynchronize(c->s_d2h);
    if (c->owns_ws) cudaFree(c->ws);
    if (c->io) cudaFree(c->io);
    for (int i = 0; i < 2; ++i) {
        if (c->ev_h[i]) cudaEventDestroy(c->ev_h[i]);
        if (c->ev_k[i]) cudaEventDestroy(c->ev_k[i]);
        if (c->ev_d[i]) cudaEventDestroy(c->ev_d[i]);
    }
    if (c->s_h2d) cudaStreamDestroy(c->s_h2d);
    if (c->s_d2h) cudaStreamDestroy(c->s_d2h);
    delete c;
    g_ctx = nullptr;
    g_sticky = false;
    return DR_OK;
}

int dr_set_occlusion_input(const uint8_t* occl_mask_dev) {
    if (!g_ctx) return fail(DR_ENOTINIT, "dr_set_occlusion_input: no context");
    g_ctx->p.occl_in = occl_mask_dev;
    return DR_OK;
}

int dr_set_stream(void* cuda_stream) {
    if (!g_ctx) return fail(DR_ENOTINIT, "dr_set_stream: no context");
    g_ctx->stream = static_cast<cudaStream_t>(cuda_stream);
    return DR_OK;
}

int dr_synchronize(void) {
    if (!g_ctx) return fail(DR_ENOTINIT, "dr_synchronize: no context");
    CK(cudaStreamSynchronize(g_ctx->stream));
    if (g_ctx->s_d2h) CK(cudaStreamSynchronize(g_ctx->s_d2h));
    if (g_ctx->s_h2d) CK(cudaStreamSynchronize(g_ctx->s_h2d));
    return DR_OK;
}

const float* dr_phys_params(void) { return g_ctx ? g_ctx->p.phys : nullptr; }
int dr_n_phys(void) { return g_ctx ? g_ctx->prm.n_phys : 0; }

const double* dr_stats(int slot) {
    if (!g_ctx || slot < 0 || slot >= N_STAT_SLOTS) return nullptr;
    return g_ctx->p.stats + slot * N_STATS;
}

int dr_set_stats_buffer(double* dev_buf) {
    if (!g_ctx) return fail(DR_ENOTINIT, "dr_set_stats_buffer: no context");
    if (dev_buf && ((uintptr_t)dev_buf & 7u)) return fail(DR_EINVAL, "stats buffer: not 8-byte aligned");
    g_ctx->p.stats = dev_buf ? dev_buf : g_ctx->internal_stats;
    // the ring must start cleared: step t accumulates into slot t % 4 (cleared by step t - 1)
    CK(cudaMemsetAsync(g_ctx->p.stats, 0, N_STAT_SLOTS * N_STATS * 8, g_ctx->stream));
    return DR_OK;
}

uint64_t dr_step_index(void) { return g_ctx ? g_ctx->t_host : 0; }

uint64_t dr_step_index_sync(void) {
    Ctx* c = g_ctx;
    if (!c) return 0;
    unsigned long long v = 0;
    if (cudaMemcpyAsync(&v, c->p.ctl, 8, cudaMemcpyDeviceToHost, c->stream) != cudaSuccess ||
        cudaStreamSynchronize(c->stream) != cudaSuccess)
        return c->t_host;
    c->t_host = v;   // graph replays advanced the device counter
    return v;
}

int dr_set_step_index(uint64_t t) {
    Ctx* c = g_ctx;
    if (!c) return fail(DR_ENOTINIT, "dr_set_step_index: no context");
    CK(cudaMemsetAsync(c->p.stats, 0, N_STAT_SLOTS * N_STATS * 8, c->stream));   // restart the stats ring
    cudaError_t e = launch_sync_init(c->p, t, c->step_grid, c->max_ctas, c->stream);
    if (e != cudaSuccess) return cuda_fail(e, "sync_init_kernel");
    c->launches++;
    ++g_total_launches;
    note_stream_launch(c->stream, nullptr);
    CK(cudaStreamSynchronize(c->stream));
    c->t_host = t;
    c->chain_next = false;
    return DR_OK;
}

size_t dr_state_bytes(void) { return g_ctx ? sizeof(dr_env_state) * (size_t)g_ctx->n_env : 0; }

static int state_range(int64_t& lo, int64_t& hi) {
    if (lo == 0 && hi == 0) hi = g_ctx->n_env;
    if (lo < 0 || hi > g_ctx->n_env || lo >= hi) return fail(DR_EINVAL, "env range [%lld, %lld) invalid", (long long)lo, (long long)hi);
    return DR_OK;
}

int dr_state_export(void* host_dst, int64_t env_lo, int64_t env_hi) {
    Ctx* c = g_ctx;
    if (!c) return fail(DR_ENOTINIT, "dr_state_export: no context");
    if (!host_dst) return fail(DR_EINVAL, "host_dst: NULL");
    int rc = state_range(env_lo, env_hi);
    if (rc) return rc;
    const size_t bytes = sizeof(dr_env_state) * (size_t)(env_hi - env_lo);
    void* d = nullptr;
    CK(cudaMallocAsync(&d, bytes, c->stream));
    cudaError_t e = launch_export(c->p, d, (uint32_t)env_lo, (uint32_t)env_hi, c->stream);
    if (e != cudaSuccess) return cuda_fail(e, "export_kernel");
    c->launches++;
    ++g_total_launches;
    note_stream_launch(c->stream, nullptr);
    CK(cudaMemcpyAsync(host_dst, d, bytes, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaFreeAsync(d, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return DR_OK;
}

int dr_state_import(const void* host_src, int64_t env_lo, int64_t env_hi) {
    Ctx* c = g_ctx;
    if (!c) return fail(DR_ENOTINIT, "dr_state_import: no context");
    if (!host_src) return fail(DR_EINVAL, "host_src: NULL");
    int rc = state_range(env_lo, env_hi);
    if (rc) return rc;
    const size_t bytes = sizeof(dr_env_state) * (size_t)(env_hi - env_lo);
    void* d = nullptr;
    CK(cudaMallocAsync(&d, bytes, c->stream));
    CK(cudaMemcpyAsync(d, host_src, bytes, cudaMemcpyHostToDevice, c->stream));
    cudaError_t e = launch_import(c->p, d, (uint32_t)env_lo, (uint32_t)env_hi, c->stream);
    if (e != cudaSuccess) return cuda_fail(e, "import_kernel");
    c->launches += 2;   // import_kernel + import_phys_kernel
    g_total_launches += 2;
    note_stream_launch(c->stream, nullptr);
    CK(cudaFreeAsync(d, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return DR_OK;
}

int dr_phys_export(void* host_dst, int64_t env_lo, int64_t env_hi) {
    Ctx* c = g_ctx;
    if (!c) return fail(DR_ENOTINIT, "dr_phys_export: no context");
    if (!host_dst) return fail(DR_EINVAL, "host_dst: NULL");
    int rc = state_range(env_lo, env_hi);
    if (rc) return rc;
    const size_t row = (size_t)c->prm.n_phys * 4;
    CK(cudaMemcpyAsync(host_dst, reinterpret_cast<const char*>(c->p.phys) + (size_t)env_lo * row,
                       (size_t)(env_hi - env_lo) * row, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return DR_OK;
}

uint64_t dr_kernel_launches(void) { return g_ctx ? g_ctx->launches : 0; }
uint64_t dr_total_kernel_launches(void) { return g_total_launches; }

int dr_debug_philox(uint32_t domain, uint32_t channel, uint32_t block, uint32_t* out_dev) {
    Ctx* c = g_ctx;
    if (!c) return fail(DR_ENOTINIT, "dr_debug_philox: no context");
    if (!out_dev || !aligned16(out_dev)) return fail(DR_EINVAL, "out_dev: NULL or not 16-byte aligned");
    cudaError_t e = launch_debug_philox((uint32_t)c->n_env, domain, channel, block, out_dev, c->stream);
    if (e != cudaSuccess) return cuda_fail(e, "debug_philox_kernel");
    c->launches++;
    ++g_total_launches;
    note_stream_launch(c->stream, nullptr);
    return DR_OK;
}

int dr_debug_philox_keyed(const uint32_t* ctr_dev, const uint32_t* key_dev, uint32_t* out_dev, uint64_t n,
                          void* stream) {
    if (n == 0) return DR_OK;
    if (!ctr_dev || !key_dev || !out_dev) return fail(DR_EINVAL, "dr_debug_philox_keyed: NULL pointer");
    if (!aligned16(ctr_dev) || !aligned16(out_dev) || ((uintptr_t)key_dev & 7u))
        return fail(DR_EINVAL, "dr_debug_philox_keyed: ctr/out need 16-byte, key 8-byte alignment");
    if (n > (1ull << 32)) return fail(DR_EINVAL, "dr_debug_philox_keyed: n > 2^32");
    cudaError_t e = launch_debug_philox_keyed(ctr_dev, key_dev, out_dev, (unsigned long long)n,
                                              static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "debug_philox_keyed_kernel");
    ++g_total_launches;
    note_stream_launch(stream, nullptr);
    return DR_OK;
}

}  // extern "C"

static_assert(sizeof(dr_env_state) == 168 * 4, "dr_env_state must be 168 words");
