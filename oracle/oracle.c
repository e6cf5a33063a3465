/*
 * oracle.c -- plain, slow, fp64 CPU oracle of the domain-randomization pipeline of
 * PAPER.md:1-115 ("Randomizations" appendix).  TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * The method is a stochastic transform with state, so this file follows the algorithm
 * step by step in the paper's order, one environment at a time, with every random draw
 * taken from a counter-based Philox4x32-10 stream whose counter layout is the contract
 * written down in DESIGN.md ("RNG conventions").  Where the paper is silent or
 * ambiguous the reading used is the one listed in DESIGN.md ("Readings"), cited below
 * as [Qn].  Build: gcc -O2 -ffp-contract=off -fPIC -shared (no FMA contraction).
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------------------
 * Philox4x32-10, written from Salmon, Moraes, Dror, Shaw, "Parallel random numbers:
 * as easy as 1, 2, 3" (SC'11), section 5: the Philox S-box on four 32-bit words
 * (L0, R0, L1, R1) multiplies R-words... in the 4x32 variant the round is
 *   hi_a:lo_a = M0 * c0,  hi_b:lo_b = M1 * c2
 *   c' = (hi_b ^ c1 ^ k0,  lo_b,  hi_a ^ c3 ^ k1,  lo_a)
 * with multipliers M0 = 0xD2511F53, M1 = 0xCD9E8D57, and the key schedule adds the
 * Weyl constants W0 = 0x9E3779B9, W1 = 0xBB67AE85 between rounds; 10 rounds.
 * Seeded reproducible randomizers: ORRB PAPER.md:245; counter-split streams keyed by
 * (seed, instance, episode, layer): SPEC.md:231.
 * ------------------------------------------------------------------------------------ */
void orc_philox(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4])
{
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    int round;
    for (round = 0; round < 10; ++round) {
        uint64_t pa = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t pb = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t hi_a = (uint32_t)(pa >> 32), lo_a = (uint32_t)pa;
        uint32_t hi_b = (uint32_t)(pb >> 32), lo_b = (uint32_t)pb;
        uint32_t n0 = hi_b ^ c1 ^ k0;
        uint32_t n1 = lo_b;
        uint32_t n2 = hi_a ^ c3 ^ k1;
        uint32_t n3 = lo_a;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        if (round < 9) {            /* key bump between rounds */
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* ------------------------------------------------------------------------------------
 * Draw transforms.
 * ------------------------------------------------------------------------------------ */

/* U(x) = ((x >> 9) + 0.5) * 2^-23, in [2^-24, 1 - 2^-24]: 23 random bits, an odd multiple of
 * 2^-24, so exactly representable in fp32 as well as fp64. */
double orc_uniform(uint32_t x)
{
    return ((double)(x >> 9) + 0.5) * (1.0 / 8388608.0);
}

/* Box-Muller: r = sqrt(-2 ln U(x)), z0 = r cos(2 pi U(y)), z1 = r sin(2 pi U(y)). */
void orc_normal_pair(uint32_t x, uint32_t y, double* z0, double* z1)
{
    double r = sqrt(-2.0 * log(orc_uniform(x)));
    double th = 2.0 * M_PI * orc_uniform(y);
    *z0 = r * cos(th);
    *z1 = r * sin(th);
}

/* Exp(lambda), rate parameterisation [Q10]: -ln U(x) / lambda.  PAPER.md:85-88. */
double orc_exponential(uint32_t x, double lambda)
{
    return -log(orc_uniform(x)) / lambda;
}

/* Bernoulli threshold T = floor(p * 2^32): the event is x < T (exact integer decision). */
uint64_t orc_bernoulli_threshold(double p)
{
    if (!(p > 0.0)) return 0;
    if (p >= 1.0) return (uint64_t)1 << 32;
    return (uint64_t)floor(p * 4294967296.0);
}

/* Hamilton product, scalar-first quaternions. */
void orc_quat_mul(const double a[4], const double b[4], double o[4])
{
    double w = a[0] * b[0] - a[1] * b[1] - a[2] * b[2] - a[3] * b[3];
    double x = a[0] * b[1] + a[1] * b[0] + a[2] * b[3] - a[3] * b[2];
    double y = a[0] * b[2] - a[1] * b[3] + a[2] * b[0] + a[3] * b[1];
    double z = a[0] * b[3] + a[1] * b[2] - a[2] * b[1] + a[3] * b[0];
    o[0] = w; o[1] = x; o[2] = y; o[3] = z;
}

/* Random rotation with angle std sigma about a uniform random axis [Q15]
 * (orientation noise "0.1 rad", Table obs-noise):
 * theta = sigma * z0(w0, w1); zc = 2 U(w2) - 1; phi = 2 pi U(w3);
 * axis = (sqrt(1 - zc^2) cos phi, sqrt(1 - zc^2) sin phi, zc);
 * q = (cos(theta/2), sin(theta/2) * axis). */
void orc_rotation(double sigma, const uint32_t w[4], double q[4])
{
    double z0, z1;
    orc_normal_pair(w[0], w[1], &z0, &z1);
    double theta = sigma * z0;
    double zc = 2.0 * orc_uniform(w[2]) - 1.0;
    double phi = 2.0 * M_PI * orc_uniform(w[3]);
    double rho = sqrt(1.0 - zc * zc);
    double h = 0.5 * theta;
    double sh = sin(h);
    q[0] = cos(h);
    q[1] = sh * (rho * cos(phi));
    q[2] = sh * (rho * sin(phi));
    q[3] = sh * zc;
}

/* Backlash model, verbatim [Q4]:
 *   s' = [s + a * delta_sgn(a) * dt]_{-1}^{+1}
 *   alpha = 1 - [ |sgn(a) - s| / (|s' - s| + eps) ]_0^1
 *   a_out = alpha * a
 * sgn(+-0) = 0 and delta_0 = 0 [Q3]. */
void orc_backlash(double s, double a, double dneg, double dpos, double dt, double eps,
                  double* s_new, double* alpha, double* out)
{
    double sg = (a > 0.0) ? 1.0 : ((a < 0.0) ? -1.0 : 0.0);
    double d = (sg > 0.0) ? dpos : ((sg < 0.0) ? dneg : 0.0);
    double sp = s + a * d * dt;
    if (sp > 1.0) sp = 1.0;
    if (sp < -1.0) sp = -1.0;
    double ratio = fabs(sg - s) / (fabs(sp - s) + eps);
    if (ratio > 1.0) ratio = 1.0;
    if (ratio < 0.0) ratio = 0.0;
    double al = 1.0 - ratio;
    *s_new = sp;
    *alpha = al;
    *out = al * a;
}

/* Squared distance in fp64, ((dx*dx + dy*dy) + dz*dz), from fp32 positions [Q13]. */
static double dist2(const float* a, const float* b)
{
    double dx = (double)a[0] - (double)b[0];
    double dy = (double)a[1] - (double)b[1];
    double dz = (double)a[2] - (double)b[2];
    double s = dx * dx;
    s = s + dy * dy;
    s = s + dz * dz;
    return s;
}

/* Marker occlusion: a fingertip marker is occluded when another fingertip or
 * the object centre is strictly closer than r [Q13; SPEC.md:165]. */
int orc_occluded(const float* tips15, const float* obj3, double r, int i)
{
    double r2 = r * r;
    int j;
    for (j = 0; j < ORC_N_TIPS; ++j) {
        if (j == i) continue;
        if (dist2(tips15 + 3 * i, tips15 + 3 * j) < r2) return 1;
    }
    if (dist2(tips15 + 3 * i, obj3) < r2) return 1;
    return 0;
}

/* ------------------------------------------------------------------------------------
 * Context
 * ------------------------------------------------------------------------------------ */

/* Channels. Step-domain draws use counter word 1 = t,
 * reset-domain draws use counter word 1 = the env's episode index k_e. */
enum {
    /* step-domain word channel: words 0-9 substep durations, 10-14 dropout of tips 0-4,
     * 15 force trigger */
    CH_STEP = 0x01, W_TIMING = 0, W_DROPOUT = 10, W_FORCE = 15,
    CH_ACT_UADD = 0x02, CH_ACT_MULT = 0x03,
    CH_TIP_NOISE = 0x05, CH_OBJ_NOISE = 0x06, CH_ROT_NOISE = 0x07, CH_FORCE = 0x08,
    CH_PHYS_U = 0x101, CH_DELAY = 0x102, CH_BACKLASH = 0x103, CH_LAMBDA = 0x104,
    CH_FORCE_P = 0x105, CH_CORR_ACT = 0x106, CH_CORR_TIP = 0x107, CH_MARKER_TIP = 0x108,
    CH_MARKER_BASE = 0x109, CH_CORR_OBJ = 0x10A, CH_CORR_ROT = 0x10B, CH_PHYS_N = 0x10C
};

#define P_TABLE_N 65536

struct orc_ctx {
    orc_params p;
    int64_t n;
    uint32_t key[2];
    uint64_t t;                 /* global step counter */
    uint64_t resets_pending;    /* resets applied since the previous step (stats slot 10) */
    uint64_t t_delay, t_drop;
    double p_tab[P_TABLE_N];
    uint64_t t_tab[P_TABLE_N];
    orc_env* env;
    double* st_env;             /* [n][ORC_N_STATS] per-env stats contributions of the current step */
    const uint8_t* occl_mask;   /* simulator occlusion bits per env, or NULL (distance rule) */
};

/* 4 words of channel ch, block blk, for global env gid and domain index (t or k_e). */
static void draw_block(const orc_ctx* c, int64_t gid, uint32_t dom, uint32_t ch, uint32_t blk,
                       uint32_t w[4])
{
    uint32_t ctr[4];
    ctr[0] = (uint32_t)gid;
    ctr[1] = dom;
    ctr[2] = ch;
    ctr[3] = blk;
    orc_philox(ctr, c->key, w);
}

/* Word i of a channel: word i%4 of block i/4. */
static uint32_t draw_word(const orc_ctx* c, int64_t gid, uint32_t dom, uint32_t ch, uint32_t i)
{
    uint32_t w[4];
    draw_block(c, gid, dom, ch, i / 4, w);
    return w[i % 4];
}

/* Normal n of a channel: block n/4; pair (w0,w1) gives normals 4b+0 (cos), 4b+1 (sin);
 * pair (w2,w3) gives 4b+2 (cos), 4b+3 (sin). */
static double draw_normal(const orc_ctx* c, int64_t gid, uint32_t dom, uint32_t ch, uint32_t n)
{
    uint32_t w[4];
    double z0, z1;
    draw_block(c, gid, dom, ch, n / 4, w);
    if ((n % 4) < 2) orc_normal_pair(w[0], w[1], &z0, &z1);
    else orc_normal_pair(w[2], w[3], &z0, &z1);
    return (n % 2 == 0) ? z0 : z1;
}

/* Parameters and their host constants: delay Bernoulli(p), dropout per-step
 * probability 1 - exp(-rate * 80 ms) at the nominal step [Q11], and the
 * loguniform force probability as a 65,536-level midpoint table [Q19]. */
static void set_params(orc_ctx* c, const orc_params* p)
{
    uint32_t j;
    double llo, lhi;
    c->p = *p;
    c->t_delay = orc_bernoulli_threshold(p->delay_prob);
    c->t_drop = orc_bernoulli_threshold(1.0 - exp(-p->dropout_rate_hz * p->step_nominal));
    llo = log(p->force_p_lo);
    lhi = log(p->force_p_hi);
    for (j = 0; j < P_TABLE_N; ++j) {
        double pj = exp(llo + (((double)j + 0.5) / 65536.0) * (lhi - llo));
        c->p_tab[j] = pj;
        c->t_tab[j] = orc_bernoulli_threshold(pj);
    }
}

int orc_init(const orc_params* p, int64_t n_env, const int64_t* gids, uint64_t seed, orc_ctx** out)
{
    orc_ctx* c;
    int64_t i;
    if (!p || !out || n_env < 1) return -1;
    if (p->n_phys < 1 || p->n_phys > ORC_MAX_PHYS) return -1;
    if (p->mass_index < 0 || p->mass_index >= p->n_phys) return -1;
    c = (orc_ctx*)calloc(1, sizeof(orc_ctx));
    if (!c) return -4;
    c->env = (orc_env*)calloc((size_t)n_env, sizeof(orc_env));
    if (!c->env) { free(c); return -4; }
    c->st_env = (double*)calloc((size_t)n_env * ORC_N_STATS, sizeof(double));
    if (!c->st_env) { free(c->env); free(c); return -4; }
    c->n = n_env;
    c->key[0] = (uint32_t)(seed & 0xFFFFFFFFu);
    c->key[1] = (uint32_t)(seed >> 32);
    c->t = 0;
    c->resets_pending = 0;
    set_params(c, p);
    for (i = 0; i < n_env; ++i) {
        c->env[i].gid = gids ? gids[i] : i;
        c->env[i].episode = 0;
    }
    *out = c;
    /* episode 0 for every env */
    {
        uint8_t* all = (uint8_t*)malloc((size_t)n_env);
        int rc;
        if (!all) { orc_free(c); *out = NULL; return -4; }
        memset(all, 1, (size_t)n_env);
        /* orc_reset bumps the episode index; start at -1 so episode 0 is drawn. */
        for (i = 0; i < n_env; ++i) c->env[i].episode = 0xFFFFFFFFu;
        rc = orc_reset(c, all);
        free(all);
        c->resets_pending = 0;
        return rc;
    }
}

/* Parameter update mid-run ("change randomization parameters during training"):
 * the new set replaces the old one for every draw made afterwards.  Step draws read c->p at
 * each step; episode records keep the values drawn at their reset until the next reset. */
int orc_update_params(orc_ctx* c, const orc_params* p)
{
    if (!c || !p) return -1;
    if (p->n_phys < 1 || p->n_phys > ORC_MAX_PHYS) return -1;
    if (p->mass_index < 0 || p->mass_index >= p->n_phys) return -1;
    set_params(c, p);
    return 0;
}

void orc_free(orc_ctx* c)
{
    if (!c) return;
    free(c->st_env);
    free(c->env);
    free(c);
}

/* Episode reset of one env: PAPER.md:7-8 (physics), 13 + 15-18 (correlated obs noise +
 * marker misplacement), 77-78 (delay flags), 87-88 (lambda), 100-101 (backlash widths),
 * 113 (force probability); SPEC.md:135-138 (state zeroed, slack 0, force 0). */
static void reset_env(orc_ctx* c, orc_env* e)
{
    const orc_params* p = &c->p;
    const uint32_t L = p->layer_mask;
    const int64_t g = e->gid;
    uint32_t k, j;
    int i;

    e->episode += 1u;
    k = e->episode;

    /* 1. physical parameters: sampled per episode, held fixed; descriptor
     *    schema SPEC.md:126 [Q20].  The u-th uniform-kind parameter uses word u of
     *    channel PHYS_U, the n-th normal-kind parameter normal n of channel PHYS_N. */
    {
        uint32_t u = 0, m = 0;
        for (i = 0; i < p->n_phys; ++i) {
            const orc_phys_desc* d = &p->phys[i];
            double v = d->base;
            if (L & ORC_PHYS) {
                switch (d->kind) {
                case ORC_PHYS_UNIFORM_SCALE: {
                    double U = orc_uniform(draw_word(c, g, k, CH_PHYS_U, u++));
                    v = d->base * (d->a + (d->b - d->a) * U);
                    break;
                }
                case ORC_PHYS_LOGUNIFORM_SCALE: {
                    double U = orc_uniform(draw_word(c, g, k, CH_PHYS_U, u++));
                    v = d->base * exp(log(d->a) + (log(d->b) - log(d->a)) * U);
                    break;
                }
                case ORC_PHYS_ADD_GAUSS: {
                    double z = draw_normal(c, g, k, CH_PHYS_N, m++);
                    v = d->base + d->a * z;
                    break;
                }
                case ORC_PHYS_MUL_LOGNORMAL: {
                    double z = draw_normal(c, g, k, CH_PHYS_N, m++);
                    v = d->base * exp(d->a * z);
                    break;
                }
                default: /* FIXED */
                    v = d->base;
                }
            }
            e->phys[i] = v;
        }
        for (; i < ORC_MAX_PHYS; ++i) e->phys[i] = 0.0;
        /* the object mass the force std refers to is this episode's mass [Q18] */
        e->mass = e->phys[p->mass_index];
    }

    /* 2. per-actuator delay flag, Bernoulli(0.5) per episode. */
    e->delay_bits = 0;
    if (L & ORC_DELAY) {
        for (j = 0; j < ORC_N_ACT; ++j) {
            uint32_t x = draw_word(c, g, k, CH_DELAY, j);
            if ((uint64_t)x < c->t_delay) e->delay_bits |= (1u << j);
        }
    }

    /* 3. backlash widths: calibrated + N(0, 0.1), clamped at 0 [Q7]. */
    for (j = 0; j < ORC_N_ACT; ++j) {
        if (L & ORC_BACKLASH) {
            double zn = draw_normal(c, g, k, CH_BACKLASH, j);
            double zp = draw_normal(c, g, k, CH_BACKLASH, ORC_N_ACT + j);
            double dn = p->delta_cal_neg[j] + p->delta_jitter_std * zn;
            double dp = p->delta_cal_pos[j] + p->delta_jitter_std * zp;
            e->dneg[j] = dn > 0.0 ? dn : 0.0;
            e->dpos[j] = dp > 0.0 ? dp : 0.0;
        } else {
            e->dneg[j] = 0.0;
            e->dpos[j] = 0.0;
        }
    }

    /* 4. timing coefficient lambda ~ U[1250, 10000] per episode. */
    if (L & ORC_TIMING) {
        double U = orc_uniform(draw_word(c, g, k, CH_LAMBDA, 0));
        e->lambda = p->lambda_lo + (p->lambda_hi - p->lambda_lo) * U;
    } else {
        e->lambda = 0.0;
    }

    /* 5. force probability p ~ loguniform[0.1%, 10%] per episode [Q19]. */
    if (L & ORC_FORCE) {
        uint32_t x = draw_word(c, g, k, CH_FORCE_P, 0);
        e->p_index = x >> 16;
        e->p_force = c->p_tab[e->p_index];
        e->t_force = (uint32_t)(c->t_tab[e->p_index] > 0xFFFFFFFFull ? 0xFFFFFFFFull
                                                                     : c->t_tab[e->p_index]);
    } else {
        e->p_index = 0;
        e->p_force = 0.0;
        e->t_force = 0;
    }

    /* 6. correlated action noise, 1.5% of the action range (range 2) [Q8]
     *    (Table action-noise). */
    for (j = 0; j < ORC_N_ACT; ++j)
        e->c_act[j] = (L & ORC_ACT_NOISE) ? p->act_sigma_cadd * draw_normal(c, g, k, CH_CORR_ACT, j) : 0.0;

    /* 7-9. correlated observation noise + marker misplacement (Table obs-noise
     *      PAPER.md:36-41) [Q14, Q15]. */
    if (L & ORC_OBS_NOISE) {
        for (i = 0; i < ORC_N_TIPS; ++i) {
            int cc;
            for (cc = 0; cc < 3; ++cc) {
                uint32_t n = (uint32_t)(3 * i + cc);
                double zc = draw_normal(c, g, k, CH_CORR_TIP, n);
                double zm = draw_normal(c, g, k, CH_MARKER_TIP, n);
                double v = p->tip_corr * zc + p->tip_marker * zm;
                if (p->base_marker_to_tips) {
                    double zb = draw_normal(c, g, k, CH_MARKER_BASE, (uint32_t)cc);
                    v = v - p->base_marker * zb;
                }
                e->off_tip[3 * i + cc] = v;
            }
        }
        for (i = 0; i < 3; ++i)
            e->c_obj[i] = p->obj_corr * draw_normal(c, g, k, CH_CORR_OBJ, (uint32_t)i);
        {
            uint32_t w[4];
            draw_block(c, g, k, CH_CORR_ROT, 0, w);
            orc_rotation(p->rot_corr, w, e->q_c);
        }
    } else {
        for (i = 0; i < ORC_N_TIPS * 3; ++i) e->off_tip[i] = 0.0;
        for (i = 0; i < 3; ++i) e->c_obj[i] = 0.0;
        e->q_c[0] = 1.0; e->q_c[1] = 0.0; e->q_c[2] = 0.0; e->q_c[3] = 0.0;
    }

    /* 10. state: slack 0, previous action 0, no last reading, timers 0, force 0
     *     (delay at episode start returns 0, SPEC.md:183 [Q9]; initial slack [Q6]). */
    for (j = 0; j < ORC_N_ACT; ++j) { e->prev[j] = 0.0; e->slack[j] = 0.0; e->ema[j] = 0.0; }
    for (i = 0; i < ORC_N_TIPS * 3; ++i) e->last[i] = 0.0;
    e->has_last = 0;
    for (i = 0; i < ORC_N_TIPS; ++i) e->timer[i] = 0;
    e->f_trig[0] = e->f_trig[1] = e->f_trig[2] = 0.0;
    e->k_f = 0;
}

/* Envs are independent (each draws from its own counters), so the all-core build (-fopenmp,
 * oracle.py "omp") runs the per-env loops of orc_reset / orc_step_sub in parallel; the result is
 * bit-identical to the single-thread build (tests/test_oracle_pipeline.py). */
int orc_reset(orc_ctx* c, const uint8_t* mask)
{
    int64_t i;
    if (!c) return -2;
#pragma omp parallel for schedule(static)
    for (i = 0; i < c->n; ++i) {
        if (mask && !mask[i]) continue;
        reset_env(c, &c->env[i]);
    }
    for (i = 0; i < c->n; ++i)
        if (!mask || mask[i]) c->resets_pending += 1;
    return 0;
}

/* One environment step of one env, PAPER.md:70-115 and 63-66 in the order of DESIGN.md
 * [Q1]: timing -> delay -> action noise (+clamp) -> backlash; occlusion -> dropout ->
 * fingertip noise + hold -> object position -> orientation -> force. */
static void step_env(orc_ctx* c, orc_env* e, const float* act, const float* obs, int occ_bits,
                     double* o_act, double* o_sub, double* o_obs, double* o_dt, double* o_force,
                     double* st, double* margin)
{
    const orc_params* p = &c->p;
    const uint32_t L = p->layer_mask;
    const int64_t g = e->gid;
    const uint32_t t = (uint32_t)c->t;
    double dt[ORC_N_SUB], dt_env;
    int i, j, cc;

    st[ORC_S_ENVS] += 1.0;

    /* 1. timing: each of the 10 substeps lasts 8 ms + Exp(lambda);
     *    dt_env = left-to-right sum of the 10 substeps [Q2]. */
    for (j = 0; j < ORC_N_SUB; ++j) {
        if (L & ORC_TIMING)
            dt[j] = p->dt_base + orc_exponential(draw_word(c, g, t, CH_STEP, (uint32_t)(W_TIMING + j)), e->lambda);
        else
            dt[j] = p->dt_base;
    }
    dt_env = dt[0];
    for (j = 1; j < ORC_N_SUB; ++j) dt_env = dt_env + dt[j];
    if (o_dt) for (j = 0; j < ORC_N_SUB; ++j) o_dt[j] = dt[j];
    st[ORC_S_SUM_DT] += dt_env;
    st[ORC_S_SUM_DT2] += dt_env * dt_env;

    /* 2-4. actions */
    for (j = 0; j < ORC_N_ACT; ++j) {
        double a = (double)act[j];
        double ad, an, out;
        /* 1b. EMA smoothing of the policy action before it is applied (PAPER.md:742-744,
         *     coefficient 0.3 per 80 ms) [Q25]: a <- (1 - c) a_s + c a, state 0 at reset. */
        if (L & ORC_SMOOTH) {
            a = (1.0 - p->act_smooth_coef) * e->ema[j] + p->act_smooth_coef * a;
            e->ema[j] = a;
        }
        /* 2. one-step delay of flagged actuators [Q9]; the buffer holds
         *    the policy action. */
        if (L & ORC_DELAY) {
            int delayed = (e->delay_bits >> j) & 1u;
            ad = delayed ? e->prev[j] : a;
            e->prev[j] = a;
            if (delayed) st[ORC_S_DELAYED] += 1.0;
        } else {
            ad = a;
        }
        /* 3. action noise: uncorrelated additive 5%, correlated additive 1.5%, uncorrelated
         *    multiplicative 1.5% (Table action-noise) [Q8], then clamp. */
        if (L & ORC_ACT_NOISE) {
            double zu = draw_normal(c, g, t, CH_ACT_UADD, (uint32_t)j);
            double zm = draw_normal(c, g, t, CH_ACT_MULT, (uint32_t)j);
            an = ad + ad * (p->act_sigma_mult * zm);
            an = an + p->act_sigma_uadd * zu;
            an = an + e->c_act[j];
            if (an > 1.0 || an < -1.0) st[ORC_S_ACT_CLAMPS] += 1.0;
            if (an > 1.0) an = 1.0;
            if (an < -1.0) an = -1.0;
            st[ORC_S_SUM_ZU2] += zu * zu;
        } else {
            an = ad;
        }
        st[ORC_S_SUM_DA] += an - ad;
        st[ORC_S_SUM_DA2] += (an - ad) * (an - ad);
        /* 4'. per-substep backlash [Q2 alternative, Q26]: the slack model runs once per
         *     substep k with dt_k, the action a_n held over the step; out_sub[k] = alpha_k a_n,
         *     the step's out_actions = the last substep's. */
        if ((L & ORC_BACKLASH) && (L & ORC_SUBSTEP_BL)) {
            double s = e->slack[j], sn, al, ok = an, mg = INFINITY;
            double sg = (an > 0.0) ? 1.0 : ((an < 0.0) ? -1.0 : 0.0);
            int k;
            for (k = 0; k < ORC_N_SUB; ++k) {
                orc_backlash(s, an, e->dneg[j], e->dpos[j], dt[k], p->backlash_eps, &sn, &al, &ok);
                if (sg != 0.0) {
                    double d = (sg > 0.0) ? e->dpos[j] : e->dneg[j];
                    double m = fabs((s + an * d * dt[k]) - sg);
                    if (m < mg) mg = m;
                    if (sn == sg && s != sg && fabs(sg - s) < mg) mg = fabs(sg - s);   /* eps-gate point */
                }
                if (sg != 0.0 && fabs(sn) == 1.0 && sn != s) st[ORC_S_RAIL_HITS] += 1.0;
                if (al == 1.0) st[ORC_S_ALPHA_ONE] += 1.0; else st[ORC_S_ALPHA_LT1] += 1.0;
                if (o_sub) o_sub[k * ORC_N_ACT + j] = ok;
                s = sn;
            }
            if (margin) margin[j] = mg;
            e->slack[j] = s;
            out = ok;
        } else
        /* 4. backlash with dt = dt_env [Q2]. */
        if (L & ORC_BACKLASH) {
            double s = e->slack[j], sn, al;
            double sg = (an > 0.0) ? 1.0 : ((an < 0.0) ? -1.0 : 0.0);
            orc_backlash(s, an, e->dneg[j], e->dpos[j], dt_env, p->backlash_eps, &sn, &al, &out);
            if (margin) {
                if (sg != 0.0) {
                    double d = (sg > 0.0) ? e->dpos[j] : e->dneg[j];
                    margin[j] = fabs((s + an * d * dt_env) - sg);
                    /* a rail hit from s != sgn gives alpha = eps / (|sgn - s| + eps): for |sgn - s|
                     * near or below sqrt(eps) that value moves with the last bits of s, so the
                     * distance |sgn - s| is the second knife-edge margin of the gate */
                    if (sn == sg && s != sg && fabs(sg - s) < margin[j]) margin[j] = fabs(sg - s);
                } else {
                    margin[j] = INFINITY;
                }
            }
            if (sg != 0.0 && fabs(sn) == 1.0 && sn != s) st[ORC_S_RAIL_HITS] += 1.0;
            if (al == 1.0) st[ORC_S_ALPHA_ONE] += 1.0; else st[ORC_S_ALPHA_LT1] += 1.0;
            e->slack[j] = sn;
        } else {
            out = an;
            if (margin) margin[j] = INFINITY;
            if (o_sub) {
                int k;
                for (k = 0; k < ORC_N_SUB; ++k) o_sub[k * ORC_N_ACT + j] = an;
            }
        }
        st[ORC_S_SUM_ABS_BL] += fabs(out - an);
        if (o_act) o_act[j] = out;
    }

    /* 5-7. fingertip markers */
    {
        const float* tips = obs;        /* raw_obs[0..14] */
        const float* obj = obs + 15;    /* raw_obs[15..17] */
        int occ[ORC_N_TIPS], masked[ORC_N_TIPS];
        /* 5. occlusion: distance rule on raw positions, exact fp64 [Q13]; or the
         *    simulator's own per-marker occlusion bits when it provides them [Q27]. */
        for (i = 0; i < ORC_N_TIPS; ++i) {
            if (occ_bits >= 0)
                occ[i] = (L & ORC_OCCLUSION) ? ((occ_bits >> i) & 1) : 0;
            else
                occ[i] = ((L & ORC_OCCLUSION) && p->occl_dist > 0.0) ? orc_occluded(tips, obj, p->occl_dist, i) : 0;
            if (occ[i]) st[ORC_S_OCCLUDED] += 1.0;
        }
        /* 6. dropout: each fingertip marker starts a 1 s mask with probability
         *    1 - exp(-0.2 * 0.08) per step [Q11]; mask held dropout_hold_steps = 13 steps,
         *    a retrigger restarts it. */
        for (i = 0; i < ORC_N_TIPS; ++i) {
            if (L & ORC_DROPOUT) {
                uint32_t x = draw_word(c, g, t, CH_STEP, (uint32_t)(W_DROPOUT + i));
                if ((uint64_t)x < c->t_drop) {
                    e->timer[i] = p->dropout_hold_steps;
                    st[ORC_S_DROP_INIT] += 1.0;
                }
                masked[i] = e->timer[i] > 0;
                if (e->timer[i] > 0) e->timer[i] -= 1;
            } else {
                masked[i] = 0;
            }
            if (masked[i]) st[ORC_S_MASKED] += 1.0;
        }
        /* 7. fingertip position = true + (correlated + misplaced-marker offset) + 2 mm
         *    uncorrelated noise; masked or occluded markers
         *    return their last available reading [Q12]. */
        for (i = 0; i < ORC_N_TIPS; ++i) {
            double y[3];
            int hold = e->has_last && (masked[i] || occ[i]);
            for (cc = 0; cc < 3; ++cc) {
                double v = (double)tips[3 * i + cc];
                if (L & ORC_OBS_NOISE) {
                    double z = draw_normal(c, g, t, CH_TIP_NOISE, (uint32_t)(3 * i + cc));
                    v = v + e->off_tip[3 * i + cc];
                    v = v + p->tip_uncorr * z;
                    st[ORC_S_SUM_ZTIP2] += z * z;
                }
                y[cc] = v;
            }
            if (hold) st[ORC_S_HELD] += 1.0;
            for (cc = 0; cc < 3; ++cc) {
                double o = hold ? e->last[3 * i + cc] : y[cc];
                e->last[3 * i + cc] = o;
                if (o_obs) o_obs[4 + 3 * i + cc] = o;
            }
        }
        /* 8. object position: 5 mm correlated + 1 mm uncorrelated. */
        for (cc = 0; cc < 3; ++cc) {
            double v = (double)obj[cc];
            if (L & ORC_OBS_NOISE) {
                double z = draw_normal(c, g, t, CH_OBJ_NOISE, (uint32_t)cc);
                v = v + e->c_obj[cc];
                v = v + p->obj_uncorr * z;
            }
            if (o_obs) o_obs[19 + cc] = v;
        }
    }

    /* 9. orientation noise (0.1 rad correlated + 0.1 rad uncorrelated) and the
     *    policy's "noisy relative goal" (Table policy-inputs) [Q15, Q16]:
     *    q_n = q_u (x) (q_c (x) q_obj); rel = goal (x) conj(q_n), w >= 0. */
    {
        double qo[4], goal[4], qn[4], tmp[4], cj[4], rel[4];
        for (cc = 0; cc < 4; ++cc) { qo[cc] = (double)obs[18 + cc]; goal[cc] = (double)obs[22 + cc]; }
        if (L & ORC_OBS_NOISE) {
            double qu[4];
            uint32_t w[4];
            draw_block(c, g, t, CH_ROT_NOISE, 0, w);
            orc_rotation(p->rot_uncorr, w, qu);
            orc_quat_mul(e->q_c, qo, tmp);
            orc_quat_mul(qu, tmp, qn);
        } else {
            for (cc = 0; cc < 4; ++cc) qn[cc] = qo[cc];
        }
        cj[0] = qn[0]; cj[1] = -qn[1]; cj[2] = -qn[2]; cj[3] = -qn[3];
        orc_quat_mul(goal, cj, rel);
        if (rel[0] < 0.0) for (cc = 0; cc < 4; ++cc) rel[cc] = -rel[cc];
        if (o_obs) for (cc = 0; cc < 4; ++cc) o_obs[cc] = rel[cc];
    }

    /* 10. random force on the object: with probability p per step a force ~ N(0, (1 m/s^2 *
     *     mass)^2) per axis replaces the stored one [Q17]; it decays by 0.99 per 80 ms step,
     *     closed form f_trig * 0.99^k. */
    {
        double f[3] = {0.0, 0.0, 0.0};
        if (L & ORC_FORCE) {
            uint32_t x = draw_word(c, g, t, CH_STEP, W_FORCE);
            if (x < e->t_force) {
                double z0, z1, z2, z3;
                uint32_t w[4];
                draw_block(c, g, t, CH_FORCE, 1, w);
                orc_normal_pair(w[0], w[1], &z0, &z1);
                orc_normal_pair(w[2], w[3], &z2, &z3);
                (void)z3;
                e->f_trig[0] = (e->mass * p->force_accel_std) * z0;
                e->f_trig[1] = (e->mass * p->force_accel_std) * z1;
                e->f_trig[2] = (e->mass * p->force_accel_std) * z2;
                e->k_f = 0;
                st[ORC_S_FORCE_TRIG] += 1.0;
            } else {
                if (e->k_f < 65535u) e->k_f += 1u;
            }
            {
                double dec = pow(p->force_decay_per_step, (double)e->k_f);
                for (cc = 0; cc < 3; ++cc) f[cc] = e->f_trig[cc] * dec;
            }
        }
        if (o_force) for (cc = 0; cc < 3; ++cc) o_force[cc] = f[cc];
        st[ORC_S_SUM_F2] += f[0] * f[0] + f[1] * f[1] + f[2] * f[2];
    }

    /* 11. a reading now exists for the hold rule */
    e->has_last = 1;
}

int orc_step(orc_ctx* c, const float* actions, const float* raw_obs,
             double* out_actions, double* out_obs, double* out_dt, double* out_force,
             double* stats, double* bl_margin)
{
    return orc_step_sub(c, actions, raw_obs, out_actions, NULL, out_obs, out_dt, out_force, stats, bl_margin);
}

int orc_step_sub(orc_ctx* c, const float* actions, const float* raw_obs,
                 double* out_actions, double* out_actions_sub, double* out_obs, double* out_dt,
                 double* out_force, double* stats, double* bl_margin)
{
    double st[ORC_N_STATS];
    int64_t i;
    int k;
    if (!c || !actions || !raw_obs) return -1;
    memset(c->st_env, 0, (size_t)c->n * ORC_N_STATS * sizeof(double));
#pragma omp parallel for schedule(static)
    for (i = 0; i < c->n; ++i) {
        step_env(c, &c->env[i], actions + i * ORC_N_ACT, raw_obs + i * ORC_OBS_IN,
                 c->occl_mask ? (int)(c->occl_mask[i] & 0x1Fu) : -1,
                 out_actions ? out_actions + i * ORC_N_ACT : NULL,
                 out_actions_sub ? out_actions_sub + i * ORC_N_SUB * ORC_N_ACT : NULL,
                 out_obs ? out_obs + i * ORC_OBS_OUT : NULL,
                 out_dt ? out_dt + i * ORC_N_SUB : NULL,
                 out_force ? out_force + i * 3 : NULL,
                 c->st_env + i * ORC_N_STATS,
                 bl_margin ? bl_margin + i * ORC_N_ACT : NULL);
    }
    /* the step's stats: per-env contributions summed in env order */
    memset(st, 0, sizeof(st));
    for (i = 0; i < c->n; ++i)
        for (k = 0; k < ORC_N_STATS; ++k) st[k] += c->st_env[i * ORC_N_STATS + k];
    st[ORC_S_RESETS] = (double)c->resets_pending;
    c->resets_pending = 0;
    if (stats) memcpy(stats, st, sizeof(st));
    c->t += 1;
    return 0;
}

void orc_set_occlusion_mask(orc_ctx* c, const uint8_t* mask) { if (c) c->occl_mask = mask; }

uint64_t orc_step_index(const orc_ctx* c) { return c ? c->t : 0; }
void orc_set_step_index(orc_ctx* c, uint64_t t) { if (c) c->t = t; }
int64_t orc_n_env(const orc_ctx* c) { return c ? c->n : 0; }

int orc_get_env(const orc_ctx* c, int64_t i, orc_env* dst)
{
    if (!c || !dst || i < 0 || i >= c->n) return -1;
    *dst = c->env[i];
    return 0;
}

/* State import: a plain field copy of *src into env i (its global id is kept: the Philox counter
 * of env i stays the context's).  The reproducibility principle of the paper (ORRB's seeded,
 * deterministic randomization) makes a run resumable from any exported state: the
 * next draws depend only on (seed, global id, t, k_e), so import -> continue equals the
 * uninterrupted run.  The test suite also uses it to start the oracle from a crafted state
 * (boundary cases) or from the GPU's exported state (windowed re-sync). */
int orc_set_env(orc_ctx* c, int64_t i, const orc_env* src)
{
    int64_t gid;
    if (!c || !src || i < 0 || i >= c->n) return -1;
    gid = c->env[i].gid;
    c->env[i] = *src;
    c->env[i].gid = gid;
    return 0;
}

uint64_t orc_force_threshold(const orc_ctx* c, uint32_t j) { return (c && j < P_TABLE_N) ? c->t_tab[j] : 0; }
double orc_force_p(const orc_ctx* c, uint32_t j) { return (c && j < P_TABLE_N) ? c->p_tab[j] : 0.0; }
