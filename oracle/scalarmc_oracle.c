/*
 * scalarmc_oracle.c — CPU restatement of the reference hot path (TEST
 * INFRASTRUCTURE ONLY).
 *
 * This file is the parity oracle for the B200 forward map.  It restates, in
 * plain C, the algorithm of the reference library scalarmc
 * (/root/reference/proj, arXiv 1808.10580) for the forward map G(u): Philox
 * streams, Box-Muller normals, the Fourier velocity series, Euler-Maruyama
 * paths to a fixed time (advection-diffusion) and to the first exit
 * (Dirichlet), and the deterministic pairwise-tree reduction.  Each function
 * cites the reference file:line it follows.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load it, and only as the checker.  The product path (the CUDA library) never
 * links or calls it.
 *
 * Parity pinning: the oracle is checked (tests/test_oracle.py) against
 *   - the Random123 philox4x32-10 known-answer vectors,
 *   - golden outputs of the real reference compiled from its own sources
 *     (oracle/Makefile -> oracle/_ref/, fixtures in tests/golden/),
 * bit for bit.  Floating point follows the reference build: IEEE double, no
 * FMA contraction (compile with -ffp-contract=off), glibc libm for
 * log/sin/cos/exp/sqrt/floor/hypot.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../include/scalarmc_b200.h"

#define ORC_API __attribute__((visibility("default")))

static const double kPi = 3.141592653589793;          /* std::numbers::pi */
static const double kTwoPi = 2.0 * 3.141592653589793; /* fields.cpp:13 */

static char g_err[512];
static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}
ORC_API const char* orc_last_error(void) { return g_err; }

/* ------------------------------------------------------------------------ */
/* Philox4x32-10 (src/rng.cpp:13-41).                                        */
/* ------------------------------------------------------------------------ */
ORC_API void orc_philox4x32(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {       /* rng.cpp:35-39 */
        const uint64_t p0 = (uint64_t)0xD2511F53u * c0; /* kPhiloxM0, rng.cpp:13 */
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2; /* kPhiloxM1, rng.cpp:14 */
        const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        /* round: c = {hi1^c1^k0, lo1, hi0^c3^k1, lo0} (rng.cpp:24-29) */
        const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
        k0 += 0x9E3779B9u; /* kPhiloxW0 */
        k1 += 0xBB67AE85u; /* kPhiloxW1 */
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* NormalStream (include/scalarmc/rng.hpp:34-55, src/rng.cpp:45-94). */
typedef struct {
    uint32_t key[2];
    uint32_t obs, particle;
    uint64_t block;
    double normal_cache, uniform_cache;
    int has_normal, has_uniform;
} orc_stream;

static void stream_init(orc_stream* s, uint64_t seed, uint32_t obs, uint32_t particle) {
    memset(s, 0, sizeof *s);
    s->key[0] = (uint32_t)seed;          /* rng.cpp:48 */
    s->key[1] = (uint32_t)(seed >> 32);
    s->obs = obs;
    s->particle = particle;
}

/* next_uniform_block (rng.cpp:53-65): counter (block lo, block hi, obs,
 * particle); two uniforms ((r >> 11) + 0.5) * 2^-53. */
static void next_uniform_block(orc_stream* s, double u[2]) {
    const uint32_t ctr[4] = {(uint32_t)s->block, (uint32_t)(s->block >> 32), s->obs, s->particle};
    uint32_t r[4];
    ++s->block;
    orc_philox4x32(ctr, s->key, r);
    const uint64_t a = ((uint64_t)r[1] << 32) | r[0];
    const uint64_t b = ((uint64_t)r[3] << 32) | r[2];
    const double scale = 1.0 / 9007199254740992.0;
    u[0] = ((double)(a >> 11) + 0.5) * scale;
    u[1] = ((double)(b >> 11) + 0.5) * scale;
}

/* normal_pair (rng.cpp:67-72): Box-Muller, one block per pair. */
static void normal_pair(orc_stream* s, double z[2]) {
    double u[2];
    next_uniform_block(s, u);
    const double r = sqrt(-2.0 * log(u[0]));
    const double a = 2.0 * kPi * u[1];
    z[0] = r * cos(a);
    z[1] = r * sin(a);
}

/* normal (rng.cpp:74-83) with its one-value cache. */
static double stream_normal(orc_stream* s) {
    if (s->has_normal) {
        s->has_normal = 0;
        return s->normal_cache;
    }
    double z[2];
    normal_pair(s, z);
    s->normal_cache = z[1];
    s->has_normal = 1;
    return z[0];
}

/* uniform (rng.cpp:85-94) with its one-value cache. */
static double stream_uniform(orc_stream* s) {
    if (s->has_uniform) {
        s->has_uniform = 0;
        return s->uniform_cache;
    }
    double u[2];
    next_uniform_block(s, u);
    s->uniform_cache = u[1];
    s->has_uniform = 1;
    return u[0];
}

ORC_API void orc_normal_pairs(uint64_t seed, uint32_t obs, uint32_t particle, int64_t n_blocks,
                              double* out) {
    orc_stream s;
    stream_init(&s, seed, obs, particle);
    for (int64_t i = 0; i < n_blocks; ++i) normal_pair(&s, out + 2 * i);
}

ORC_API void orc_uniform_blocks(uint64_t seed, uint32_t obs, uint32_t particle, int64_t n_blocks,
                                double* out) {
    orc_stream s;
    stream_init(&s, seed, obs, particle);
    for (int64_t i = 0; i < n_blocks; ++i) next_uniform_block(&s, out + 2 * i);
}

/* Mixed draw sequence: ops[i] = 0 -> normal(), 1 -> uniform(), 2 -> normal_pair
 * (two outputs).  Exercises the caches exactly like pcn_step does. */
ORC_API int64_t orc_stream_draws(uint64_t seed, uint32_t obs, uint32_t particle, int64_t n,
                                 const int32_t* ops, double* out) {
    orc_stream s;
    stream_init(&s, seed, obs, particle);
    int64_t w = 0;
    for (int64_t i = 0; i < n; ++i) {
        if (ops[i] == 0) out[w++] = stream_normal(&s);
        else if (ops[i] == 1) out[w++] = stream_uniform(&s);
        else { normal_pair(&s, out + w); w += 2; }
    }
    return w;
}

/* ------------------------------------------------------------------------ */
/* Fourier velocity field (src/fields.cpp:17-89).                            */
/* ------------------------------------------------------------------------ */
typedef struct { double re, im; } cplx;

static cplx cmul(cplx a, cplx b) { /* fields.cpp:20 */
    cplx r = {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
    return r;
}

/* fill_powers (fields.cpp:23-31). */
static void fill_powers(cplx* p, double x, int n) {
    p[0].re = 1.0; p[0].im = 0.0;
    if (n == 0) return;
    const double a = kTwoPi * x;
    const cplx e = {cos(a), sin(a)};
    p[1] = e;
    for (int j = 2; j <= n; ++j) p[j] = cmul(p[j - 1], e);
}

typedef struct { int k1, k2; double re, im, d1, d2; } prepared_mode;

typedef struct {
    int is_constant;
    double c1, c2;
    int max_k;
    int64_t n;
    prepared_mode* modes;
    cplx *p1, *p2;
} orc_velocity;

static int mode_cmp(const void* a, const void* b) {
    const prepared_mode* x = (const prepared_mode*)a;
    const prepared_mode* y = (const prepared_mode*)b;
    if (x->k1 != y->k1) return x->k1 < y->k1 ? -1 : 1;
    if (x->k2 != y->k2) return x->k2 < y->k2 ? -1 : 1;
    return 0;
}

/* FourierVelocityField ctor (fields.cpp:35-69): validate, canonicalise
 * (k1 > 0 or k1 == 0, k2 > 0) with v -> -conj(v), sort by (k1, k2), reject
 * duplicates, precompute k_perp / |k|. */
static int velocity_build(const smc_velocity* v, orc_velocity* out) {
    memset(out, 0, sizeof *out);
    if (v->is_constant) {
        out->is_constant = 1;
        out->c1 = v->constant[0];
        out->c2 = v->constant[1];
        return 0;
    }
    if (v->max_wavenumber <= 0)
        return fail(SMC_EINVAL, "FourierVelocityField: max_wavenumber must be positive");
    const int K = v->max_wavenumber;
    out->max_k = K;
    out->n = v->n_modes;
    out->modes = (prepared_mode*)calloc((size_t)(v->n_modes > 0 ? v->n_modes : 1), sizeof(prepared_mode));
    for (int64_t i = 0; i < v->n_modes; ++i) {
        int k1 = v->k[2 * i], k2 = v->k[2 * i + 1];
        double re = v->coeff[2 * i], im = v->coeff[2 * i + 1];
        if (k1 == 0 && k2 == 0) { free(out->modes); return fail(SMC_EINVAL, "FourierVelocityField: k = (0,0) is not allowed"); }
        const double kn2 = (double)k1 * k1 + (double)k2 * k2;
        if (kn2 > (double)K * K + 1e-9) { free(out->modes); return fail(SMC_EINVAL, "FourierVelocityField: |k| exceeds max_wavenumber"); }
        if (!isfinite(re) || !isfinite(im)) { free(out->modes); return fail(SMC_EINVAL, "FourierVelocityField: non-finite coefficient"); }
        if (!(k1 > 0 || (k1 == 0 && k2 > 0))) { k1 = -k1; k2 = -k2; re = -re; /* -conj: (-re, +im) */ }
        out->modes[i].k1 = k1; out->modes[i].k2 = k2;
        out->modes[i].re = re; out->modes[i].im = im;
    }
    qsort(out->modes, (size_t)v->n_modes, sizeof(prepared_mode), mode_cmp);
    for (int64_t i = 1; i < v->n_modes; ++i)
        if (out->modes[i].k1 == out->modes[i - 1].k1 && out->modes[i].k2 == out->modes[i - 1].k2) {
            free(out->modes);
            return fail(SMC_EINVAL, "FourierVelocityField: duplicate mode (both members of a +/-k pair given?)");
        }
    for (int64_t i = 0; i < v->n_modes; ++i) {
        prepared_mode* m = &out->modes[i];
        const double kn = sqrt((double)m->k1 * m->k1 + (double)m->k2 * m->k2);
        m->d1 = -(double)m->k2 / kn;
        m->d2 = (double)m->k1 / kn;
    }
    out->p1 = (cplx*)malloc(sizeof(cplx) * (size_t)(K + 1));
    out->p2 = (cplx*)malloc(sizeof(cplx) * (size_t)(K + 1));
    return 0;
}

static void velocity_free(orc_velocity* v) {
    free(v->modes); free(v->p1); free(v->p2);
    memset(v, 0, sizeof *v);
}

/* FourierVelocityField::operator() (fields.cpp:71-89) behind the
 * VelocityField constant/Fourier dispatch (fields.hpp:73). */
static void velocity_eval(orc_velocity* f, double x1, double x2, double* v1o, double* v2o) {
    if (f->is_constant) { *v1o = f->c1; *v2o = f->c2; return; }
    if (f->n == 0) { *v1o = 0.0; *v2o = 0.0; return; }
    fill_powers(f->p1, x1, f->max_k);
    fill_powers(f->p2, x2, f->max_k);
    double v1 = 0.0, v2 = 0.0;
    for (int64_t i = 0; i < f->n; ++i) {
        const prepared_mode* m = &f->modes[i];
        const cplx a = f->p1[m->k1];
        cplx b = f->p2[m->k2 >= 0 ? m->k2 : -m->k2];
        if (m->k2 < 0) b.im = -b.im;
        const cplx e = cmul(a, b);
        const double w = 2.0 * (m->re * e.re - m->im * e.im);
        v1 += w * m->d1;
        v2 += w * m->d2;
    }
    *v1o = v1; *v2o = v2;
}

/* FourierVelocityField::amplitude_bound (fields.cpp:109-113) /
 * VelocityField::amplitude_bound (fields.cpp:140-142). */
static double velocity_amplitude_bound(const orc_velocity* f) {
    if (f->is_constant) return hypot(f->c1, f->c2);
    double s = 0.0;
    for (int64_t i = 0; i < f->n; ++i) s += 2.0 * hypot(f->modes[i].re, f->modes[i].im);
    return s;
}

ORC_API int orc_velocity_eval(const smc_velocity* v, int64_t n, const double* x, double* out) {
    orc_velocity f;
    int rc = velocity_build(v, &f);
    if (rc) return rc;
    for (int64_t i = 0; i < n; ++i) velocity_eval(&f, x[2 * i], x[2 * i + 1], &out[2 * i], &out[2 * i + 1]);
    velocity_free(&f);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* ScalarField::operator() (src/fields.cpp:235-253).                         */
/* ------------------------------------------------------------------------ */
static double scalar_eval(const smc_scalar_field* f, double x1, double x2) {
    switch (f->kind) {
        case SMC_SCALAR_CONSTANT:
            return f->constant;
        case SMC_SCALAR_COSINE: {
            double s = 0.0;
            for (int i = 0; i < f->n_terms; ++i) {
                /* freq.dot(x) = freq.x1*x.x1 + freq.x2*x.x2 (geometry.hpp:22) */
                const double dot = f->freq[2 * i] * x1 + f->freq[2 * i + 1] * x2;
                s += f->amplitude[i] * cos(dot + f->phase[i]);
            }
            return s;
        }
        case SMC_SCALAR_BUMPS: {
            double s = 0.0;
            for (int i = 0; i < f->n_terms; ++i) {
                const double d1 = x1 - f->center[2 * i], d2 = x2 - f->center[2 * i + 1];
                s += f->amplitude[i] * exp(-f->sharpness * (d1 * d1 + d2 * d2));
            }
            return s;
        }
        case SMC_SCALAR_LINEAR:
            return f->constant + (f->gradient[0] * x1 + f->gradient[1] * x2);
    }
    return 0.0;
}

ORC_API void orc_scalar_eval(const smc_scalar_field* f, int64_t n, const double* x, double* out) {
    for (int64_t i = 0; i < n; ++i) out[i] = scalar_eval(f, x[2 * i], x[2 * i + 1]);
}

/* ------------------------------------------------------------------------ */
/* Domain (src/geometry.cpp:22-114).                                         */
/* ------------------------------------------------------------------------ */
static int domain_contains(const smc_domain* d, double x1, double x2) { /* geometry.cpp:22-31 */
    if (d->kind == SMC_DOMAIN_BOX)
        return x1 > d->lower[0] && x1 < d->upper[0] && x2 > d->lower[1] && x2 < d->upper[1];
    if (d->kind == SMC_DOMAIN_DISK) {
        const double q1 = x1 - d->center[0], q2 = x2 - d->center[1];
        return q1 * q1 + q2 * q2 < d->radius * d->radius;
    }
    return 1;
}

static double domain_diameter(const smc_domain* d) { /* geometry.cpp:38-42 */
    if (d->kind == SMC_DOMAIN_BOX) return hypot(d->upper[0] - d->lower[0], d->upper[1] - d->lower[1]);
    if (d->kind == SMC_DOMAIN_DISK) return 2.0 * d->radius;
    return 1.4142135623730951; /* std::numbers::sqrt2 */
}

static double face_crossing(double from, double to, double c) { /* geometry.cpp:47-52 */
    const double d = to - from;
    if (d == 0.0) return INFINITY;
    const double t = (c - from) / d;
    return (t >= 0.0 && t <= 1.0) ? t : INFINITY;
}

static double clampd(double v, double lo, double hi) { return v < lo ? lo : (hi < v ? hi : v); }

/* boundary_exit (geometry.cpp:56-114).  Returns the fraction, writes the
 * crossing point. */
static double boundary_exit(const smc_domain* dom, double in1, double in2, double out1, double out2,
                            double* p1, double* p2) {
    if (dom->kind == SMC_DOMAIN_BOX) {
        const double d1 = out1 - in1, d2 = out2 - in2;
        double best_t = INFINITY, best_val = 0.0;
        int best_axis = -1;
        for (int axis = 0; axis < 2; ++axis) {
            const double from = axis == 0 ? in1 : in2;
            const double to = axis == 0 ? out1 : out2;
            const double faces[2] = {dom->lower[axis], dom->upper[axis]};
            for (int f = 0; f < 2; ++f) {
                const double t = face_crossing(from, to, faces[f]);
                if (t < best_t) { best_t = t; best_axis = axis; best_val = faces[f]; }
            }
        }
        double x = in1 + best_t * d1, y = in2 + best_t * d2;
        if (best_axis == 0) { x = best_val; y = clampd(y, dom->lower[1], dom->upper[1]); }
        else { y = best_val; x = clampd(x, dom->lower[0], dom->upper[0]); }
        *p1 = x; *p2 = y;
        return best_t;
    }
    /* disk */
    const double q1 = in1 - dom->center[0], q2 = in2 - dom->center[1];
    const double d1 = out1 - in1, d2 = out2 - in2;
    const double a = d1 * d1 + d2 * d2;
    const double bq = 2.0 * (q1 * d1 + q2 * d2);
    const double c = (q1 * q1 + q2 * q2) - dom->radius * dom->radius;
    const double disc = bq * bq - 4.0 * a * c;
    const double t = (-bq + sqrt(disc)) / (2.0 * a);
    const double tc = clampd(t, 0.0, 1.0);
    double x = in1 + tc * d1, y = in2 + tc * d2;
    const double r1 = x - dom->center[0], r2 = y - dom->center[1];
    const double rn = hypot(r1, r2);
    if (rn > 0.0) {
        const double s = dom->radius / rn;
        x = dom->center[0] + s * r1;
        y = dom->center[1] + s * r2;
    }
    *p1 = x; *p2 = y;
    return tc;
}

/* ------------------------------------------------------------------------ */
/* Euler-Maruyama paths (src/sde.cpp:8-77).                                  */
/* ------------------------------------------------------------------------ */
/* em_step (sde.cpp:8-16): x - v dt + (sigma sqrt(dt)) xi, with sigma =
 * sqrt(2 kappa) on both components (fields.cpp:158-165).  Milstein equals EM
 * for isotropic sigma (sde.cpp:21). */
static void em_step(orc_velocity* vel, double sigma, double* x1, double* x2, double dt, const double xi[2]) {
    double v1, v2;
    velocity_eval(vel, *x1, *x2, &v1, &v2);
    const double root_dt = sqrt(dt);
    const double n1 = *x1 - v1 * dt + sigma * root_dt * xi[0];
    const double n2 = *x2 - v2 * dt + sigma * root_dt * xi[1];
    *x1 = n1; *x2 = n2;
}

/* simulate_to_time on the torus (sde.cpp:37-50), then theta_0 at the terminal
 * point (forward_ad.cpp:41-47). */
static double ad_particle(orc_velocity* vel, double sigma, const smc_scalar_field* theta0, double t,
                          double x01, double x02, double dt, uint64_t seed, uint32_t obs,
                          uint32_t particle, double* term1, double* term2) {
    orc_stream s;
    stream_init(&s, seed, obs, particle);
    const int64_t n_steps = (int64_t)ceil(t / dt);
    double x1 = x01 - floor(x01), x2 = x02 - floor(x02); /* Domain::wrap, geometry.cpp:33-36 */
    for (int64_t i = 0; i < n_steps; ++i) {
        const double h = (i + 1 < n_steps) ? dt : t - (double)(n_steps - 1) * dt;
        double xi[2];
        normal_pair(&s, xi);
        em_step(vel, sigma, &x1, &x2, h, xi);
        x1 = x1 - floor(x1);
        x2 = x2 - floor(x2);
    }
    if (term1) { *term1 = x1; *term2 = x2; }
    return scalar_eval(theta0, x1, x2);
}

/* simulate_to_exit (sde.cpp:52-77) + the BVP work function
 * (forward_bvp.cpp:39-46). */
static void bvp_particle(orc_velocity* vel, double sigma, const smc_bvp_problem* p, double dt,
                         double x01, double x02, uint64_t seed, uint32_t obs, uint32_t particle,
                         double* value, double* aux, uint8_t* failed, int64_t* steps) {
    orc_stream s;
    stream_init(&s, seed, obs, particle);
    double x1 = x01, x2 = x02, f_int = 0.0;
    for (int64_t step = 0; step < p->max_steps; ++step) {
        double xi[2], n1 = x1, n2 = x2;
        normal_pair(&s, xi);
        em_step(vel, sigma, &n1, &n2, dt, xi);
        if (!domain_contains(&p->domain, n1, n2)) {
            double h1, h2;
            const double frac = boundary_exit(&p->domain, x1, x2, n1, n2, &h1, &h2);
            f_int += scalar_eval(&p->forcing, x1, x2) * frac * dt;
            const double tau = (double)step * dt + frac * dt;
            *value = scalar_eval(&p->boundary_data, h1, h2) - f_int;
            *aux = tau;
            *failed = 0;
            if (steps) *steps = step + 1;
            return;
        }
        f_int += scalar_eval(&p->forcing, x1, x2) * dt;
        x1 = n1; x2 = n2;
    }
    *value = 0.0; *aux = 0.0; *failed = 1; /* forward_bvp.cpp:44 */
    if (steps) *steps = p->max_steps;
}

/* ------------------------------------------------------------------------ */
/* Reduction (src/executor.cpp:11-26, :87-117).                              */
/* ------------------------------------------------------------------------ */
ORC_API double orc_pairwise_sum(const double* values, int64_t n) {
    if (n == 0) return 0.0;
    double* buf = (double*)malloc(sizeof(double) * (size_t)n);
    memcpy(buf, values, sizeof(double) * (size_t)n);
    int64_t m = n;
    while (m > 1) {
        const int64_t half = m / 2;
        for (int64_t i = 0; i < half; ++i) buf[i] = buf[2 * i] + buf[2 * i + 1];
        if (m % 2 == 1) { buf[half] = buf[m - 1]; m = half + 1; }
        else m = half;
    }
    const double r = buf[0];
    free(buf);
    return r;
}

static int reduce_observation(const double* values, const double* aux, const uint8_t* failed,
                              int64_t n_particles, smc_estimate* out) {
    double* valid = (double*)malloc(sizeof(double) * (size_t)n_particles);
    double* vaux = (double*)malloc(sizeof(double) * (size_t)n_particles);
    int64_t nv = 0, n_failed = 0;
    for (int64_t i = 0; i < n_particles; ++i) {
        if (failed && failed[i]) { ++n_failed; continue; }
        valid[nv] = values[i];
        vaux[nv] = aux ? aux[i] : 0.0;
        ++nv;
    }
    if (nv == 0) {
        free(valid); free(vaux);
        return fail(SMC_ERUNTIME, "map_reduce: every particle of an observation failed");
    }
    const double n = (double)nv;
    const double mean = orc_pairwise_sum(valid, nv) / n;
    double se = 0.0;
    if (nv > 1) {
        double* sq = (double*)malloc(sizeof(double) * (size_t)nv);
        for (int64_t i = 0; i < nv; ++i) { const double d = valid[i] - mean; sq[i] = d * d; }
        const double var = orc_pairwise_sum(sq, nv) / (n - 1.0);
        se = sqrt(var / n);
        free(sq);
    }
    out->mean = mean;
    out->std_error = se;
    out->n_particles = n_particles;
    out->n_failed = n_failed;
    out->aux_mean = orc_pairwise_sum(vaux, nv) / n;
    free(valid); free(vaux);
    return 0;
}

ORC_API int orc_reduce(const double* values, const double* aux, const uint8_t* failed, int64_t n,
                       smc_estimate* out) {
    return reduce_observation(values, aux, failed, n, out);
}

/* ------------------------------------------------------------------------ */
/* Forward maps (src/forward_ad.cpp, src/forward_bvp.cpp).                   */
/* ------------------------------------------------------------------------ */
static double ad_resolved_dt(const smc_ad_problem* p) { /* forward_ad.cpp:10-15 */
    if (p->dt > 0.0) return p->dt;
    double t_min = INFINITY;
    for (int64_t j = 0; j < p->n_obs; ++j) t_min = p->obs_t[j] < t_min ? p->obs_t[j] : t_min;
    return t_min / 200.0;
}

static int ad_validate(const smc_ad_problem* p) { /* forward_ad.cpp:17-28 */
    if (p->n_obs <= 0) return fail(SMC_EINVAL, "AdProblemSpec: no observations");
    for (int64_t j = 0; j < p->n_obs; ++j) {
        const double t = p->obs_t[j], x1 = p->obs_x[2 * j], x2 = p->obs_x[2 * j + 1];
        if (!(t > 0.0)) return fail(SMC_EINVAL, "AdProblemSpec: observation times must be positive");
        if (!isfinite(x1) || !isfinite(x2)) return fail(SMC_EINVAL, "AdProblemSpec: non-finite observation point");
        if (x1 < 0.0 || x1 >= 1.0 || x2 < 0.0 || x2 >= 1.0)
            return fail(SMC_EINVAL, "AdProblemSpec: observation points must lie in [0,1)^2");
    }
    if (p->n_particles < 2) return fail(SMC_EINVAL, "AdProblemSpec: need at least two particles");
    return 0;
}

static double isotropic_sigma(double kappa) { return sqrt(2.0 * kappa); } /* fields.cpp:158-165 */

ORC_API int orc_ad_particle_values(const smc_ad_problem* p, uint64_t obs_index, uint64_t seed,
                                   int64_t n, double* out, double* terminal) {
    orc_velocity vel;
    int rc = velocity_build(&p->velocity, &vel);
    if (rc) return rc;
    const double dt = ad_resolved_dt(p), sigma = isotropic_sigma(p->kappa);
    for (int64_t i = 0; i < n; ++i)
        out[i] = ad_particle(&vel, sigma, &p->initial_condition, p->obs_t[obs_index],
                             p->obs_x[2 * obs_index], p->obs_x[2 * obs_index + 1], dt, seed,
                             (uint32_t)obs_index, (uint32_t)i, terminal ? &terminal[2 * i] : NULL,
                             terminal ? &terminal[2 * i + 1] : NULL);
    velocity_free(&vel);
    return 0;
}

/* observe_ad (forward_ad.cpp:53-60): one map_reduce per observation, stream
 * key obs slot = spec slot (forward_ad.cpp:43). */
ORC_API int orc_ad_observe(const smc_ad_problem* p, uint64_t seed, smc_estimate* out) {
    if (!(p->kappa >= 0.0)) return fail(SMC_EINVAL, "DiffusionModel: kappa must be >= 0");
    int rc = ad_validate(p);
    if (rc) return rc;
    double* vals = (double*)malloc(sizeof(double) * (size_t)p->n_particles);
    for (int64_t j = 0; j < p->n_obs; ++j) {
        rc = orc_ad_particle_values(p, (uint64_t)j, seed, p->n_particles, vals, NULL);
        if (rc) break;
        rc = reduce_observation(vals, NULL, NULL, p->n_particles, &out[j]);
        if (rc) break;
    }
    free(vals);
    return rc;
}

static double bvp_resolved_dt_v(const smc_bvp_problem* p, const orc_velocity* vel) { /* forward_bvp.cpp:9-18 */
    if (p->dt > 0.0) return p->dt;
    const double diam = domain_diameter(&p->domain);
    const double kappa = p->kappa;
    const double speed = velocity_amplitude_bound(vel);
    const double denom = 2.0 * kappa + speed * diam;
    const double raw = denom > 0.0 ? 1e-3 * diam * diam / denom : 1e-2;
    return clampd(raw, 1e-6, 1e-2);
}

static int bvp_validate(const smc_bvp_problem* p) { /* forward_bvp.cpp:20-32 */
    if (p->domain.kind == SMC_DOMAIN_TORUS) return fail(SMC_EINVAL, "BvpProblemSpec: domain must be bounded");
    if (p->n_obs <= 0) return fail(SMC_EINVAL, "BvpProblemSpec: no observations");
    for (int64_t j = 0; j < p->n_obs; ++j) {
        const double x1 = p->obs_x[2 * j], x2 = p->obs_x[2 * j + 1];
        if (!isfinite(x1) || !isfinite(x2)) return fail(SMC_EINVAL, "BvpProblemSpec: non-finite observation point");
        if (!domain_contains(&p->domain, x1, x2))
            return fail(SMC_EINVAL, "BvpProblemSpec: observation points must be strictly interior");
    }
    if (p->n_particles < 2) return fail(SMC_EINVAL, "BvpProblemSpec: need at least two particles");
    if (p->max_steps < 1) return fail(SMC_EINVAL, "BvpProblemSpec: max_steps must be positive");
    return 0;
}

ORC_API double orc_bvp_resolved_dt(const smc_bvp_problem* p) {
    orc_velocity vel;
    if (velocity_build(&p->velocity, &vel)) return NAN;
    const double dt = bvp_resolved_dt_v(p, &vel);
    velocity_free(&vel);
    return dt;
}

ORC_API int orc_bvp_particle_values(const smc_bvp_problem* p, uint64_t obs_index, uint64_t seed,
                                    int64_t n, double* values, double* aux, uint8_t* failed,
                                    int64_t* steps) {
    orc_velocity vel;
    int rc = velocity_build(&p->velocity, &vel);
    if (rc) return rc;
    const double dt = bvp_resolved_dt_v(p, &vel), sigma = isotropic_sigma(p->kappa);
    for (int64_t i = 0; i < n; ++i)
        bvp_particle(&vel, sigma, p, dt, p->obs_x[2 * obs_index], p->obs_x[2 * obs_index + 1], seed,
                     (uint32_t)obs_index, (uint32_t)i, &values[i], &aux[i], &failed[i],
                     steps ? &steps[i] : NULL);
    velocity_free(&vel);
    return 0;
}

/* observe_bvp (forward_bvp.cpp:34-49): one map_reduce over all observations,
 * key obs slot = j. */
ORC_API int orc_bvp_observe(const smc_bvp_problem* p, uint64_t seed, smc_estimate* out) {
    if (!(p->kappa >= 0.0)) return fail(SMC_EINVAL, "DiffusionModel: kappa must be >= 0");
    int rc = bvp_validate(p);
    if (rc) return rc;
    const size_t n = (size_t)p->n_particles;
    double* vals = (double*)malloc(sizeof(double) * n);
    double* aux = (double*)malloc(sizeof(double) * n);
    uint8_t* failed = (uint8_t*)malloc(n);
    for (int64_t j = 0; j < p->n_obs; ++j) {
        rc = orc_bvp_particle_values(p, (uint64_t)j, seed, p->n_particles, vals, aux, failed, NULL);
        if (rc) break;
        rc = reduce_observation(vals, aux, failed, p->n_particles, &out[j]);
        if (rc) break;
    }
    free(vals); free(aux); free(failed);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* u -> field (src/inference.cpp:24-73).                                     */
/* ------------------------------------------------------------------------ */
typedef struct { int k1, k2; } mode_index;

static int prior_mode_cmp(const void* a, const void* b) { /* inference.cpp:33-38 */
    const mode_index* x = (const mode_index*)a;
    const mode_index* y = (const mode_index*)b;
    const double na = (double)x->k1 * x->k1 + (double)x->k2 * x->k2;
    const double nb = (double)y->k1 * y->k1 + (double)y->k2 * y->k2;
    if (na != nb) return na < nb ? -1 : 1;
    if (x->k1 != y->k1) return x->k1 < y->k1 ? -1 : 1;
    if (x->k2 != y->k2) return x->k2 < y->k2 ? -1 : 1;
    return 0;
}

/* PriorSpec::modes (inference.cpp:24-40).  Writes up to cap (k1,k2) pairs;
 * returns the count. */
ORC_API int64_t orc_prior_modes(int cutoff, int32_t* out, int64_t cap) {
    int64_t n = 0;
    const int64_t side = 2 * (int64_t)cutoff + 1;
    mode_index* m = (mode_index*)malloc(sizeof(mode_index) * (size_t)(side * side));
    for (int k1 = -cutoff; k1 <= cutoff; ++k1)
        for (int k2 = -cutoff; k2 <= cutoff; ++k2) {
            if (!(k1 > 0 || (k1 == 0 && k2 > 0))) continue;
            if ((double)k1 * k1 + (double)k2 * k2 > (double)cutoff * cutoff) continue;
            m[n].k1 = k1; m[n].k2 = k2; ++n;
        }
    qsort(m, (size_t)n, sizeof(mode_index), prior_mode_cmp);
    for (int64_t i = 0; i < n && i < cap; ++i) { out[2 * i] = m[i].k1; out[2 * i + 1] = m[i].k2; }
    free(m);
    return n;
}

/* prior_draw (inference.cpp:55-61): u_i = s_i * normal(), s = s0 |k|^-alpha. */
ORC_API int64_t orc_prior_draw(const smc_prior* prior, uint64_t seed, uint64_t obs, uint64_t particle,
                               double* out, int64_t cap) {
    int32_t* k = (int32_t*)malloc(sizeof(int32_t) * 2 * (size_t)(4 * (prior->cutoff + 1) * (prior->cutoff + 1)));
    const int64_t n = orc_prior_modes(prior->cutoff, k, 4 * (int64_t)(prior->cutoff + 1) * (prior->cutoff + 1));
    orc_stream s;
    stream_init(&s, seed, (uint32_t)obs, (uint32_t)particle);
    for (int64_t i = 0; i < n && 2 * i + 1 < cap; ++i) {
        const double kn = sqrt((double)k[2 * i] * k[2 * i] + (double)k[2 * i + 1] * k[2 * i + 1]);
        const double sd = prior->s0 * pow(kn, -prior->alpha);
        out[2 * i] = sd * stream_normal(&s);
        out[2 * i + 1] = sd * stream_normal(&s);
    }
    free(k);
    return 2 * n;
}
