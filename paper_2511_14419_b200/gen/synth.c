/*
 * synth.c — seeded synthetic well time-lapses for the BASELINE configurations.
 *
 * Model (per well): background i.i.d. N(mu, sigma^2) redrawn every frame; global flicker gain
 * g_t ~ U[1-f, 1+f]; cells are soft-edged ellipses (semi-axes U[amin, amax], orientation
 * U[0, pi), contrast N(cmean, csd^2)) adding c * erfc(d / (edge*sqrt 2)) / 2 with
 * d = (rho - 1) * min(a, b), rho the normalised elliptical radius; overlaps add.  Motion is a
 * correlated random walk v_t = p v_{t-1} + sqrt(1-p^2) xi, xi ~ N(0, step^2) per axis, reflected
 * at the margins, with the first floor(stationary_fraction * n) cells fixed; mode 1 moves every
 * cell once by N(0, step^2) (config 1), mode 2 repeats frame 0 (zero motion).  Samples are
 * clamped to [0, data_max] and rounded half away from zero.
 *
 * Determinism: the cell state comes from one splitmix64 stream per well; the background noise of
 * pixel i of frame t is a counter-based draw (splitmix64 of seed, well, t, i), so frames can be
 * generated in parallel (pthreads over frames) and identical bytes come out for any thread count.
 * This is the repository's own generator (the reference's synthetic.hpp models a different scene).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct froi_synth_spec {
    int width, height;
    int sample_bytes; /* 1 or 2 */
    double data_max;  /* 255 or 4095 */
    double mu, sigma;
    int n_cells;
    double cmean, csd;
    double amin, amax;
    double edge;        /* soft-edge sigma, px */
    double step;        /* per-axis step sigma */
    double persistence; /* p */
    double stationary_fraction;
    double flicker;     /* +-f */
    int mode;           /* 0 walk, 1 single displacement, 2 zero motion */
    uint64_t seed;
} froi_synth_spec;

static uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

typedef struct {
    uint64_t s;
    int have;
    double spare;
} rng_t;

static uint64_t rng_u64(rng_t* r) { return mix64(r->s += 0x9e3779b97f4a7c15ull); }
static double rng_unit(rng_t* r) { return (double)(rng_u64(r) >> 11) * 0x1.0p-53; }
static double rng_uniform(rng_t* r, double lo, double hi) { return lo + (hi - lo) * rng_unit(r); }
static double rng_normal(rng_t* r) {
    if (r->have) {
        r->have = 0;
        return r->spare;
    }
    double u1 = 0.0;
    while (u1 <= 0.0) u1 = rng_unit(r);
    const double u2 = rng_unit(r), rad = sqrt(-2.0 * log(u1)), a = 6.283185307179586 * u2;
    r->spare = rad * sin(a);
    r->have = 1;
    return rad * cos(a);
}

typedef struct {
    double x, y, vx, vy, a, b, cth, sth, c;
    int fixed;
} cell_t;

typedef struct {
    const froi_synth_spec* sp;
    int well, n_frames;
    const double* cx; /* [frame][cell] */
    const double* cy;
    const cell_t* cells;
    const double* gain; /* [frame] */
    void* out;
    int t0, t1;
} job_t;

static double counter_normal(uint64_t key, uint64_t i) {
    /* one Box-Muller draw from two counter-based uniforms */
    const uint64_t h1 = mix64(key ^ (i * 0x9e3779b97f4a7c15ull + 0x632be59bd9b4e019ull));
    const uint64_t h2 = mix64(h1 + 0xd1b54a32d192ed03ull);
    double u1 = (double)((h1 >> 11) + 1) * 0x1.0p-53; /* (0, 1] */
    const double u2 = (double)(h2 >> 11) * 0x1.0p-53;
    return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}

static void* render(void* arg) {
    job_t* j = (job_t*)arg;
    const froi_synth_spec* sp = j->sp;
    const int W = sp->width, H = sp->height;
    const size_t px = (size_t)W * H;
    double* acc = (double*)malloc(sizeof(double) * px);
    const double inv_edge = 1.0 / (sp->edge * sqrt(2.0));
    for (int t = j->t0; t < j->t1; ++t) {
        const int tn = sp->mode == 2 ? 0 : t; /* zero motion: every frame is frame 0 */
        const uint64_t key = mix64(sp->seed * 0x100000001b3ull ^ ((uint64_t)j->well << 32) ^ (uint64_t)tn);
        for (size_t i = 0; i < px; ++i) acc[i] = sp->mu + sp->sigma * counter_normal(key, i);
        for (int c = 0; c < sp->n_cells; ++c) {
            const cell_t* cl = &j->cells[c];
            const double x0 = j->cx[(size_t)tn * sp->n_cells + c], y0 = j->cy[(size_t)tn * sp->n_cells + c];
            const double r = (cl->a > cl->b ? cl->a : cl->b) + 6.0 * sp->edge;
            int xa = (int)floor(x0 - r), xb = (int)ceil(x0 + r), ya = (int)floor(y0 - r), yb = (int)ceil(y0 + r);
            if (xa < 0) xa = 0;
            if (ya < 0) ya = 0;
            if (xb > W - 1) xb = W - 1;
            if (yb > H - 1) yb = H - 1;
            const double mn = cl->a < cl->b ? cl->a : cl->b;
            for (int y = ya; y <= yb; ++y)
                for (int x = xa; x <= xb; ++x) {
                    const double dx = x - x0, dy = y - y0;
                    const double u = (dx * cl->cth + dy * cl->sth) / cl->a;
                    const double v = (-dx * cl->sth + dy * cl->cth) / cl->b;
                    const double rho = sqrt(u * u + v * v);
                    const double d = (rho - 1.0) * mn;
                    acc[(size_t)y * W + x] += cl->c * 0.5 * erfc(d * inv_edge);
                }
        }
        const double g = j->gain[tn];
        for (size_t i = 0; i < px; ++i) {
            double v = g * acc[i];
            v = v < 0.0 ? 0.0 : (v > sp->data_max ? sp->data_max : v);
            const double q = floor(v + 0.5);
            if (sp->sample_bytes == 1) ((uint8_t*)j->out)[(size_t)t * px + i] = (uint8_t)q;
            else ((uint16_t*)j->out)[(size_t)t * px + i] = (uint16_t)q;
        }
    }
    free(acc);
    return NULL;
}

/* Generates frames [n_frames][H][W] of well `well`.  Returns 0, or 1 on bad arguments. */
int froi_synth_well(const froi_synth_spec* sp, int well, int n_frames, void* out, int n_threads) {
    if (!sp || !out || n_frames < 1 || sp->width < 8 || sp->height < 8 || sp->n_cells < 0) return 1;
    if (sp->sample_bytes != 1 && sp->sample_bytes != 2) return 1;
    const int W = sp->width, H = sp->height, nc = sp->n_cells;
    rng_t r = {mix64(sp->seed ^ 0x9e3779b97f4a7c15ull ^ ((uint64_t)well * 0xbf58476d1ce4e5b9ull)), 0, 0.0};
    cell_t* cells = (cell_t*)calloc(nc > 0 ? nc : 1, sizeof(cell_t));
    double* cx = (double*)malloc(sizeof(double) * (size_t)n_frames * (nc > 0 ? nc : 1));
    double* cy = (double*)malloc(sizeof(double) * (size_t)n_frames * (nc > 0 ? nc : 1));
    double* gain = (double*)malloc(sizeof(double) * n_frames);
    const double margin = sp->amax + 4.0;
    const int n_fixed = (int)floor(sp->stationary_fraction * nc);
    for (int c = 0; c < nc; ++c) {
        cell_t* cl = &cells[c];
        cl->a = rng_uniform(&r, sp->amin, sp->amax);
        cl->b = rng_uniform(&r, sp->amin, sp->amax);
        const double th = rng_uniform(&r, 0.0, 3.141592653589793);
        cl->cth = cos(th);
        cl->sth = sin(th);
        cl->c = sp->cmean + sp->csd * rng_normal(&r);
        cl->x = rng_uniform(&r, margin, W - margin);
        cl->y = rng_uniform(&r, margin, H - margin);
        cl->vx = cl->vy = 0.0;
        cl->fixed = c < n_fixed;
    }
    const double q = sqrt(1.0 - sp->persistence * sp->persistence);
    for (int t = 0; t < n_frames; ++t) {
        gain[t] = rng_uniform(&r, 1.0 - sp->flicker, 1.0 + sp->flicker);
        for (int c = 0; c < nc; ++c) {
            cell_t* cl = &cells[c];
            if (t > 0 && !cl->fixed && sp->mode != 2) {
                if (sp->mode == 1) {
                    if (t == 1) {
                        cl->x += sp->step * rng_normal(&r);
                        cl->y += sp->step * rng_normal(&r);
                    }
                } else {
                    cl->vx = sp->persistence * cl->vx + q * sp->step * rng_normal(&r);
                    cl->vy = sp->persistence * cl->vy + q * sp->step * rng_normal(&r);
                    cl->x += cl->vx;
                    cl->y += cl->vy;
                }
                /* reflect at the margins */
                if (cl->x < margin) { cl->x = 2 * margin - cl->x; cl->vx = -cl->vx; }
                if (cl->x > W - margin) { cl->x = 2 * (W - margin) - cl->x; cl->vx = -cl->vx; }
                if (cl->y < margin) { cl->y = 2 * margin - cl->y; cl->vy = -cl->vy; }
                if (cl->y > H - margin) { cl->y = 2 * (H - margin) - cl->y; cl->vy = -cl->vy; }
            }
            cx[(size_t)t * nc + c] = cl->x;
            cy[(size_t)t * nc + c] = cl->y;
        }
    }
    if (n_threads < 1) n_threads = 1;
    if (n_threads > n_frames) n_threads = n_frames;
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * n_threads);
    job_t* jobs = (job_t*)malloc(sizeof(job_t) * n_threads);
    const int per = (n_frames + n_threads - 1) / n_threads;
    int started = 0;
    for (int k = 0; k < n_threads; ++k) {
        jobs[k].sp = sp;
        jobs[k].well = well;
        jobs[k].n_frames = n_frames;
        jobs[k].cx = cx;
        jobs[k].cy = cy;
        jobs[k].cells = cells;
        jobs[k].gain = gain;
        jobs[k].out = out;
        jobs[k].t0 = k * per;
        jobs[k].t1 = (k + 1) * per < n_frames ? (k + 1) * per : n_frames;
        if (jobs[k].t0 >= jobs[k].t1) break;
        pthread_create(&th[k], NULL, render, &jobs[k]);
        ++started;
    }
    for (int k = 0; k < started; ++k) pthread_join(th[k], NULL);
    free(jobs);
    free(th);
    free(gain);
    free(cx);
    free(cy);
    free(cells);
    return 0;
}

/* fnv1a64 content hash (core.hpp:155-162) for recording input identity in bench reports. */
uint64_t froi_fnv1a64(const void* data, size_t n, uint64_t h) {
    const uint8_t* p = (const uint8_t*)data;
    for (size_t i = 0; i < n; ++i) {
        h ^= p[i];
        h *= 0x100000001b3ull;
    }
    return h;
}
