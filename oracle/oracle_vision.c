/*
 * oracle_vision.c -- plain fp64 CPU oracle of the vision randomizations (TEST INFRASTRUCTURE
 * ONLY; see oracle.h): the appearance draws of Table vision-randomization
 * and the post-render image augmentation of PAPER.md:127-129.  Scalar loops in the paper's
 * order; Philox, uniforms and Box-Muller normals are the oracle's own (oracle.c).  Readings of
 * what the paper leaves open are DESIGN.md V1-V6 and are cited at each use.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "oracle.h"

enum {
    CH_POSE = 0x401,
    CH_IMG_PARAM = 0x201, CH_IMG_NOISE = 0x202,
    CH_SCENE_CAM = 0x301, CH_SCENE_MAT = 0x302, CH_SCENE_LIGHT = 0x303
};

static void block(uint64_t seed, int64_t gid, uint64_t batch, uint32_t ch, uint32_t blk, uint32_t w[4])
{
    uint32_t ctr[4], key[2];
    ctr[0] = (uint32_t)gid;
    ctr[1] = (uint32_t)batch;
    ctr[2] = ch;
    ctr[3] = blk;
    key[0] = (uint32_t)(seed & 0xFFFFFFFFu);
    key[1] = (uint32_t)(seed >> 32);
    orc_philox(ctr, key, w);
}

/* lo + (hi - lo) U(x) */
static double range(double lo, double hi, uint32_t x) { return lo + (hi - lo) * orc_uniform(x); }

/* Appearance draws of one sample (Table vision-randomization). */
static void scene_one(const orc_vision_params* p, uint64_t seed, uint64_t batch, int64_t g, double* o)
{
    uint32_t w[4], m0[4], m1[4], m2[4];
    int c, i, n;
    double total, rsum, rel[ORC_VIS_MAX_LIGHTS];
    memset(o, 0, sizeof(double) * ORC_SCENE_WORDS);
    for (c = 0; c < ORC_VIS_N_CAMERAS; ++c) {
        /* "camera position +-1.5 mm" [V1]: per-axis offset U[-r, r];
         * "camera field of view +-1 deg": offset U[-r, r] (block 2c, words 0..3) */
        block(seed, g, batch, CH_SCENE_CAM, (uint32_t)(2 * c), w);
        o[3 * c + 0] = range(-p->cam_pos_range, p->cam_pos_range, w[0]);
        o[3 * c + 1] = range(-p->cam_pos_range, p->cam_pos_range, w[1]);
        o[3 * c + 2] = range(-p->cam_pos_range, p->cam_pos_range, w[2]);
        o[21 + c] = range(-p->cam_fov_range, p->cam_fov_range, w[3]);
        /* "camera rotation 0-3 deg around a random axis" [V2]: theta ~ U[0, max], axis uniform
         * on the sphere (zc = 2U - 1, phi = 2 pi U); q = (cos theta/2, sin theta/2 axis) */
        block(seed, g, batch, CH_SCENE_CAM, (uint32_t)(2 * c + 1), w);
        {
            double th = range(0.0, p->cam_rot_max, w[0]);
            double zc = 2.0 * orc_uniform(w[1]) - 1.0;
            double phi = 2.0 * M_PI * orc_uniform(w[2]);
            double rho = sqrt(1.0 - zc * zc);
            double sh = sin(0.5 * th);
            o[9 + 4 * c + 0] = cos(0.5 * th);
            o[9 + 4 * c + 1] = sh * rho * cos(phi);
            o[9 + 4 * c + 2] = sh * rho * sin(phi);
            o[9 + 4 * c + 3] = sh * zc;
        }
    }
    block(seed, g, batch, CH_SCENE_MAT, 0, m0);
    block(seed, g, batch, CH_SCENE_MAT, 1, m1);
    block(seed, g, batch, CH_SCENE_MAT, 2, m2);
    /* "robot material colors RGB": each channel U[0, 1] [V3]; metallic 5-25 %, glossiness 0-100 % */
    o[24] = orc_uniform(m0[0]);
    o[25] = orc_uniform(m0[1]);
    o[26] = orc_uniform(m0[2]);
    o[27] = range(p->robot_metallic_lo, p->robot_metallic_hi, m0[3]);
    o[28] = range(p->robot_gloss_lo, p->robot_gloss_hi, m1[0]);
    /* "object material hue: calibrated hue +-1 %, saturation / value +-15 %" [V3]: additive
     * offsets U[-r, r] on the [0, 1] scale; hue wraps (h - floor h), s and v clamp to [0, 1] */
    {
        double h = p->obj_hue_cal + range(-p->obj_hue_range, p->obj_hue_range, m1[1]);
        double s = p->obj_sat_cal + range(-p->obj_sat_range, p->obj_sat_range, m1[2]);
        double v = p->obj_val_cal + range(-p->obj_val_range, p->obj_val_range, m1[3]);
        o[29] = h - floor(h);
        o[30] = s < 0.0 ? 0.0 : (s > 1.0 ? 1.0 : s);
        o[31] = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
    }
    o[32] = range(p->obj_metallic_lo, p->obj_metallic_hi, m2[0]);
    o[33] = range(p->obj_gloss_lo, p->obj_gloss_hi, m2[1]);
    /* "number of lights 4-6": uniform integer, n = lo + floor(x (hi - lo + 1) / 2^32) [V4]
     * (an exact integer decision on the Philox word) */
    n = p->lights_min + (int)(((uint64_t)m2[2] * (uint64_t)(p->lights_max - p->lights_min + 1)) >> 32);
    o[34] = (double)n;
    /* "total light intensity 0-15" and "relative intensity 1-5" [V5]: intensities are the
     * relative draws rescaled to sum to the total; "light position uniform over upper
     * half-sphere": direction with z = U (area-uniform on the hemisphere), phi = 2 pi U */
    total = range(p->light_total_lo, p->light_total_hi, m2[3]);
    rsum = 0.0;
    for (i = 0; i < n; ++i) {
        double z, phi, rho;
        block(seed, g, batch, CH_SCENE_LIGHT, (uint32_t)i, w);
        z = orc_uniform(w[0]);
        phi = 2.0 * M_PI * orc_uniform(w[1]);
        rho = sqrt(1.0 - z * z);
        o[35 + 3 * i + 0] = rho * cos(phi);
        o[35 + 3 * i + 1] = rho * sin(phi);
        o[35 + 3 * i + 2] = z;
        rel[i] = range(p->light_rel_lo, p->light_rel_hi, w[2]);
        rsum += rel[i];
    }
    for (i = 0; i < n; ++i) o[53 + i] = total * rel[i] / rsum;
    o[59] = total;
}

int orc_scene_draw(const orc_vision_params* p, uint64_t seed, uint64_t batch, int64_t sample_offset, int64_t n,
                   double* out)
{
    int64_t k;
    if (!p || !out || n < 0 || p->lights_min < 0 || p->lights_max > ORC_VIS_MAX_LIGHTS || p->lights_min > p->lights_max)
        return -1;
    for (k = 0; k < n; ++k) scene_one(p, seed, batch, sample_offset + k, out + (size_t)k * ORC_SCENE_WORDS);
    return 0;
}

/* Post-render augmentation of one image, in the paper's order:
 *   1. "linearly normalized to have zero mean and unit variance": x^ = (x - mu) / max(sd, floor),
 *      mu and sd over all pixels and channels of the image, sd the population std [V6];
 *   2. "the image contrast is randomized" (Table: 50 %-150 %): x^ <- f x^, f ~ U[lo, hi] per image
 *      (contrast about the normalized mean, which is 0) [V6];
 *   3. "per-pixel Gaussian noise is added" (Table: +-10 %): + s z, z ~ N(0, 1) i.i.d. per pixel
 *      and channel, s ~ U[noise lo, noise hi] per image (default 0.1, 10 % of the unit std) [V6].
 * Noise draws (vision RNG map v2, DESIGN.md "Vision readings" V7): one 32-bit word gives one Box-Muller
 * pair -- the radius from its top 20 bits, U20 = ((x >> 12) + 1/2) 2^-20, the angle from its low 12
 * bits, A12 = ((x & 0xFFF) + 1/2) 2^-12 -- so element e (row-major H, W, C) takes normal e % 2
 * (cos, sin) of the pair of word (e % 8) / 2 of Philox block e / 8 of channel IMG_NOISE. */
static void noise_pair(uint32_t x, double* z0, double* z1)
{
    double u = ((double)(x >> 12) + 0.5) * (1.0 / 1048576.0);
    double a = ((double)(x & 0xFFFu) + 0.5) * (1.0 / 4096.0);
    double r = sqrt(-2.0 * log(u));
    double th = 2.0 * M_PI * a;
    *z0 = r * cos(th);
    *z1 = r * sin(th);
}
static void augment_one(const orc_vision_params* p, uint64_t seed, uint64_t batch, int64_t g, const uint8_t* x,
                        int64_t E, double* out, double* st)
{
    int64_t e;
    double mu = 0.0, ss = 0.0, sd, f, s;
    uint32_t w[4];
    for (e = 0; e < E; ++e) mu += (double)x[e];
    mu /= (double)E;
    for (e = 0; e < E; ++e) ss += ((double)x[e] - mu) * ((double)x[e] - mu);
    sd = sqrt(ss / (double)E);
    block(seed, g, batch, CH_IMG_PARAM, 0, w);
    f = range(p->contrast_lo, p->contrast_hi, w[0]);
    s = range(p->noise_std_lo, p->noise_std_hi, w[1]);
    for (e = 0; e < E; ++e) {
        double xh = ((double)x[e] - mu) / (sd > p->std_floor ? sd : p->std_floor);   /* 1 */
        double z0, z1, z;
        xh = f * xh;                                                                 /* 2 */
        block(seed, g, batch, CH_IMG_NOISE, (uint32_t)(e / 8), w);
        noise_pair(w[(e % 8) / 2], &z0, &z1);
        z = (e % 2 == 0) ? z0 : z1;
        out[e] = xh + s * z;                                                         /* 3 */
    }
    if (st) {
        st[0] = mu;
        st[1] = sd;
        st[2] = f;
        st[3] = s;
    }
}

int orc_image_augment(const orc_vision_params* p, uint64_t seed, uint64_t batch, int64_t image_offset,
                      const uint8_t* images, int64_t n, int32_t h, int32_t w, int32_t c, double* out,
                      double* img_stats)
{
    int64_t i, E;
    if (!p || !images || !out || n < 0 || h < 1 || w < 1 || c < 1) return -1;
    E = (int64_t)h * w * c;
    for (i = 0; i < n; ++i)
        augment_one(p, seed, batch, image_offset + i, images + i * E, E, out + i * E,
                    img_stats ? img_stats + 4 * i : NULL);
    return 0;
}

/* Pose augmentation of one sample [Q28]:
 *   x0 of block 0 picks the branch: x0 < floor(p_keep 2^32) keep; x0 < floor((p_keep + p_rot90)
 *   2^32) rotate; else jitter (exact integer decisions);
 *   rotate: k = floor(6 x1 / 2^32) -> body axis k / 2, sign (k odd ? -1 : +1); q_out = q (x) r with
 *   r = (cos 45 deg, sign sin 45 deg e_axis): exactly 90 deg about the object's own axis;
 *   jitter: position + pos_std z (normals 0..2 of block 1), q_out = q_j (x) q with q_j a rotation
 *   of angle rot_std z about a uniform axis from block 2 (the obs-noise rotation convention). */
static void pose_one(const orc_pose_aug_params* p, uint64_t seed, uint64_t batch, int64_t g, const float* in,
                     double* out, uint8_t* br)
{
    uint32_t w[4], v[4];
    double q[4], r[4];
    int c, b;
    uint64_t t1 = orc_bernoulli_threshold(p->p_keep);
    uint64_t t2 = orc_bernoulli_threshold(p->p_keep + p->p_rot90);
    for (c = 0; c < 3; ++c) out[c] = (double)in[c];
    for (c = 0; c < 4; ++c) q[c] = (double)in[3 + c];
    block(seed, g, batch, CH_POSE, 0, w);
    b = ((uint64_t)w[0] < t1) ? 0 : (((uint64_t)w[0] < t2) ? 1 : 2);
    if (b == 0) {
        for (c = 0; c < 4; ++c) out[3 + c] = q[c];
    } else if (b == 1) {
        int k = (int)(((uint64_t)w[1] * 6u) >> 32);
        double sh = (k & 1) ? -sqrt(0.5) : sqrt(0.5);
        r[0] = sqrt(0.5);
        r[1] = r[2] = r[3] = 0.0;
        r[1 + k / 2] = sh;
        orc_quat_mul(q, r, out + 3);
    } else {
        double z0, z1, z2, z3;
        block(seed, g, batch, CH_POSE, 1, v);
        orc_normal_pair(v[0], v[1], &z0, &z1);
        orc_normal_pair(v[2], v[3], &z2, &z3);
        (void)z3;
        out[0] = out[0] + p->pos_std * z0;
        out[1] = out[1] + p->pos_std * z1;
        out[2] = out[2] + p->pos_std * z2;
        block(seed, g, batch, CH_POSE, 2, v);
        orc_rotation(p->rot_std, v, r);
        orc_quat_mul(r, q, out + 3);
    }
    if (br) *br = (uint8_t)b;
}

int orc_pose_augment(const orc_pose_aug_params* p, uint64_t seed, uint64_t batch, int64_t offset,
                     const float* pose_in, int64_t n, double* pose_out, uint8_t* branch)
{
    int64_t i;
    if (!p || !pose_in || !pose_out || n < 0) return -1;
    for (i = 0; i < n; ++i)
        pose_one(p, seed, batch, offset + i, pose_in + 7 * i, pose_out + 7 * i, branch ? branch + i : NULL);
    return 0;
}
