/*
 * froi_oracle.c — CPU restatement of FlowRoI's RoI-extraction hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see froi_oracle.h).  Not part of the product; the product never
 * links it.  Each function cites the reference function it restates (paths relative to
 * /root/reference/proj/include/flowroi/).  The arithmetic is done in double in the reference's
 * operation order and this file must be compiled without FMA contraction
 * (-ffp-contract=off), so that results are bit-identical to the reference.
 */
#include "froi_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#define PI_LITERAL 3.14159265358979323846

static int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }
static double clampd(double v, double lo, double hi) { return v < lo ? lo : (hi < v ? hi : v); }

/* clamp_to_depth (core.hpp:148-152): std::min(std::max(v, 0.0), maxval), then std::lround. */
static uint16_t clamp_to_depth(double v, int depth) {
    const double maxval = (double)((1 << depth) - 1);
    v = (v < 0.0) ? 0.0 : v;
    v = (maxval < v) ? maxval : v;
    return (uint16_t)lround(v);
}

/* ------------------------------------------------------------------ denoise.hpp */

static void sort_u16(uint16_t* a, int n) {
    for (int i = 1; i < n; ++i) {
        uint16_t v = a[i];
        int j = i - 1;
        while (j >= 0 && a[j] > v) {
            a[j + 1] = a[j];
            --j;
        }
        a[j + 1] = v;
    }
}

/* median_filter (denoise.hpp:28-44): order statistic size/2 of the edge-replicated window. */
void oracle_median_filter(const uint16_t* in, int w, int h, int radius, uint16_t* out) {
    const int side = 2 * radius + 1;
    uint16_t* win = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)side * side);
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            int n = 0;
            for (int dy = -radius; dy <= radius; ++dy)
                for (int dx = -radius; dx <= radius; ++dx)
                    win[n++] = in[(size_t)clampi(y + dy, 0, h - 1) * w + clampi(x + dx, 0, w - 1)];
            sort_u16(win, n);
            out[(size_t)y * w + x] = win[n / 2];
        }
    free(win);
}

/* bilateral_filter (denoise.hpp:48-81): fp64, dy-major / dx-minor accumulation. */
void oracle_bilateral_filter(const uint16_t* in, int w, int h, int depth, int radius,
                             double sigma_spatial, double sigma_range, uint16_t* out) {
    const int maxval = (1 << depth) - 1;
    double* lut = (double*)malloc(sizeof(double) * ((size_t)maxval + 1));
    for (int d = 0; d <= maxval; ++d) {
        const double t = (double)d / maxval;
        lut[d] = exp(-t * t / (2.0 * sigma_range * sigma_range));
    }
    const int side = 2 * radius + 1;
    double* spatial = (double*)malloc(sizeof(double) * (size_t)side * side);
    for (int dy = -radius; dy <= radius; ++dy)
        for (int dx = -radius; dx <= radius; ++dx)
            spatial[(dy + radius) * side + (dx + radius)] =
                exp(-(dx * dx + dy * dy) / (2.0 * sigma_spatial * sigma_spatial));
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            const int center = in[(size_t)y * w + x];
            double num = 0.0, den = 0.0;
            for (int dy = -radius; dy <= radius; ++dy)
                for (int dx = -radius; dx <= radius; ++dx) {
                    const int v = in[(size_t)clampi(y + dy, 0, h - 1) * w + clampi(x + dx, 0, w - 1)];
                    const double wt = spatial[(dy + radius) * side + (dx + radius)] *
                                      lut[abs(v - center)];
                    num += wt * v;
                    den += wt;
                }
            out[(size_t)y * w + x] = clamp_to_depth(num / den, depth);
        }
    free(spatial);
    free(lut);
}

static int validate_denoise(const froi_params* p) {
    if (p->median_radius < 1 || p->bilateral_radius < 1) return FROI_ERR_USAGE;
    if (p->bilateral_sigma_spatial <= 0 || p->bilateral_sigma_range <= 0) return FROI_ERR_USAGE;
    return 0;
}

/* denoise (denoise.hpp:84-90). */
int oracle_denoise(const uint16_t* in, int w, int h, int depth, const froi_params* p,
                   uint16_t* out) {
    if (validate_denoise(p)) return FROI_ERR_USAGE;
    if (!p->denoise_enabled) {
        memcpy(out, in, sizeof(uint16_t) * (size_t)w * h);
        return 0;
    }
    uint16_t* m = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)w * h);
    oracle_median_filter(in, w, h, p->median_radius, m);
    oracle_bilateral_filter(m, w, h, depth, p->bilateral_radius, p->bilateral_sigma_spatial,
                            p->bilateral_sigma_range, out);
    free(m);
    return 0;
}

/* ------------------------------------------------------------------ fft.hpp */

typedef struct {
    double re, im;
} cpx;

/* std::complex<double> product as GCC expands it without -ffast-math: (ac-bd) + (ad+bc)i. */
static cpx cmul(cpx a, cpx b) {
    cpx r;
    r.re = a.re * b.re - a.im * b.im;
    r.im = a.re * b.im + a.im * b.re;
    return r;
}

static int next_pow2(int n) {
    int p = 1;
    while (p < n) p <<= 1;
    return p;
}

/* fft_inplace (fft.hpp:19-44): bit reversal, radix-2 butterflies with the w *= wlen twiddle
 * recurrence restarted per group, 1/n on the inverse. */
static void fft_inplace(cpx* a, int n, int inverse) {
    for (int i = 1, j = 0; i < n; ++i) {
        int bit = n >> 1;
        for (; j & bit; bit >>= 1) j ^= bit;
        j ^= bit;
        if (i < j) {
            cpx t = a[i];
            a[i] = a[j];
            a[j] = t;
        }
    }
    for (int len = 2; len <= n; len <<= 1) {
        const double ang = (inverse ? 2.0 : -2.0) * PI_LITERAL / len;
        cpx wlen;
        wlen.re = cos(ang);
        wlen.im = sin(ang);
        const int half = len / 2;
        for (int i = 0; i < n; i += len) {
            cpx wv;
            wv.re = 1.0;
            wv.im = 0.0;
            for (int k = 0; k < half; ++k) {
                const cpx u = a[i + k];
                const cpx v = cmul(a[i + k + half], wv);
                a[i + k].re = u.re + v.re;
                a[i + k].im = u.im + v.im;
                a[i + k + half].re = u.re - v.re;
                a[i + k + half].im = u.im - v.im;
                wv = cmul(wv, wlen);
            }
        }
    }
    if (inverse) {
        const double inv = 1.0 / n;
        for (int i = 0; i < n; ++i) {
            a[i].re *= inv;
            a[i].im *= inv;
        }
    }
}

/* fft2d_inplace (fft.hpp:47-55): rows, then columns. */
static void fft2d_inplace(cpx* a, int w, int h, int inverse) {
    for (int y = 0; y < h; ++y) fft_inplace(a + (size_t)y * w, w, inverse);
    cpx* col = (cpx*)malloc(sizeof(cpx) * (size_t)h);
    for (int x = 0; x < w; ++x) {
        for (int y = 0; y < h; ++y) col[y] = a[(size_t)y * w + x];
        fft_inplace(col, h, inverse);
        for (int y = 0; y < h; ++y) a[(size_t)y * w + x] = col[y];
    }
    free(col);
}

/* ------------------------------------------------------------------ registration.hpp */

/* windowed_spectrum_input (registration.hpp:26-42). */
static cpx* windowed_input(const uint16_t* f, int w, int h, int pw, int ph) {
    double mean = 0.0;
    const size_t n = (size_t)w * h;
    for (size_t i = 0; i < n; ++i) mean += f[i];
    mean /= (double)n;
    double* wx = (double*)malloc(sizeof(double) * pw);
    double* wy = (double*)malloc(sizeof(double) * ph);
    for (int x = 0; x < pw; ++x) wx[x] = 0.5 - 0.5 * cos(2.0 * PI_LITERAL * x / pw);
    for (int y = 0; y < ph; ++y) wy[y] = 0.5 - 0.5 * cos(2.0 * PI_LITERAL * y / ph);
    cpx* a = (cpx*)malloc(sizeof(cpx) * (size_t)pw * ph);
    for (int y = 0; y < ph; ++y) {
        const int sy = y < h - 1 ? y : h - 1;
        for (int x = 0; x < pw; ++x) {
            const int sx = x < w - 1 ? x : w - 1;
            a[(size_t)y * pw + x].re = (f[(size_t)sy * w + sx] - mean) * wx[x] * wy[y];
            a[(size_t)y * pw + x].im = 0.0;
        }
    }
    free(wx);
    free(wy);
    return a;
}

/* estimate_shift (registration.hpp:46-97). */
int oracle_estimate_shift(const uint16_t* reference, const uint16_t* moving, int w, int h,
                          int max_shift, froi_shift* out) {
    const int mn = w < h ? w : h;
    if (max_shift < 1 || max_shift >= mn / 4) return FROI_ERR_USAGE;
    const int pw = next_pow2(w), ph = next_pow2(h);
    cpx* fa = windowed_input(reference, w, h, pw, ph);
    cpx* fb = windowed_input(moving, w, h, pw, ph);
    fft2d_inplace(fa, pw, ph, 0);
    fft2d_inplace(fb, pw, ph, 0);
    const size_t n = (size_t)pw * ph;
    for (size_t i = 0; i < n; ++i) {
        cpx ca;
        ca.re = fa[i].re;
        ca.im = -fa[i].im;
        const cpx c = cmul(ca, fb[i]);
        const double m = hypot(c.re, c.im); /* std::abs -> cabs -> hypot */
        if (m > 1e-12) {
            fa[i].re = c.re / m;
            fa[i].im = c.im / m;
        } else {
            fa[i].re = 0.0;
            fa[i].im = 0.0;
        }
    }
    fft2d_inplace(fa, pw, ph, 1);
#define SURF(dx, dy) (fa[(size_t)((dy) < 0 ? (dy) + ph : (dy)) * pw + ((dx) < 0 ? (dx) + pw : (dx))].re)
    int bdx = 0, bdy = 0;
    double best = -1e300;
    for (int dy = -max_shift; dy <= max_shift; ++dy)
        for (int dx = -max_shift; dx <= max_shift; ++dx) {
            const double v = SURF(dx, dy);
            if (v > best) {
                best = v;
                bdx = dx;
                bdy = dy;
            }
        }
    double second = 0.0;
    for (int dy = -max_shift; dy <= max_shift; ++dy)
        for (int dx = -max_shift; dx <= max_shift; ++dx) {
            const int cx = abs(dx - bdx), cy = abs(dy - bdy);
            if ((cx > cy ? cx : cy) <= 2) continue;
            const double v = SURF(dx, dy);
            second = (second < v) ? v : second; /* std::max(second, v) */
        }
#undef SURF
    free(fa);
    free(fb);
    if (best <= 0.0) {
        out->dx = 0;
        out->dy = 0;
        out->confidence = 1.0;
        return 0;
    }
    out->dx = bdx;
    out->dy = bdy;
    out->confidence = best / ((second < 1e-12) ? 1e-12 : second);
    return 0;
}

/* apply_shift (registration.hpp:100-107): out(x,y) = in(x+dx, y+dy), edges replicated. */
void oracle_apply_shift(const uint16_t* in, int w, int h, int dx, int dy, uint16_t* out) {
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x)
            out[(size_t)y * w + x] = in[(size_t)clampi(y + dy, 0, h - 1) * w + clampi(x + dx, 0, w - 1)];
}

/* unshift_mask (registration.hpp:111-121): inverse translation, zero fill. */
void oracle_unshift_mask(const uint8_t* in, int w, int h, int dx, int dy, uint8_t* out) {
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            const int sx = x - dx, sy = y - dy;
            out[(size_t)y * w + x] =
                (sx >= 0 && sx < w && sy >= 0 && sy < h) ? (in[(size_t)sy * w + sx] != 0) : 0;
        }
}

/* ------------------------------------------------------------------ flow.hpp */

/* correlate_rows (flow.hpp:55-70). */
static void correlate_rows(const double* src, int w, int h, const double* k, int r, double* dst) {
    for (int y = 0; y < h; ++y) {
        const double* row = src + (size_t)y * w;
        double* o = dst + (size_t)y * w;
        for (int x = 0; x < w; ++x) {
            double acc = 0.0;
            for (int t = -r; t <= r; ++t) acc += k[t + r] * row[clampi(x + t, 0, w - 1)];
            o[x] = acc;
        }
    }
}

/* correlate_cols (flow.hpp:72-84): accumulates into a zero-initialised dst. */
static void correlate_cols(const double* src, int w, int h, const double* k, int r, double* dst) {
    memset(dst, 0, sizeof(double) * (size_t)w * h);
    for (int y = 0; y < h; ++y) {
        double* o = dst + (size_t)y * w;
        for (int t = -r; t <= r; ++t) {
            const double kk = k[t + r];
            const double* row = src + (size_t)clampi(y + t, 0, h - 1) * w;
            for (int x = 0; x < w; ++x) o[x] += kk * row[x];
        }
    }
}

/* polynomial_expansion (flow.hpp:118-153) with expansion_moments (flow.hpp:92-112). */
void oracle_polynomial_expansion(const double* img, int w, int h, int poly_n, double poly_sigma,
                                 double* planes) {
    const int r = (poly_n - 1) / 2;
    double* g0 = (double*)malloc(sizeof(double) * poly_n);
    double* g1 = (double*)malloc(sizeof(double) * poly_n);
    double* g2 = (double*)malloc(sizeof(double) * poly_n);
    for (int t = -r; t <= r; ++t) {
        const double wt = exp(-(double)t * t / (2.0 * poly_sigma * poly_sigma));
        g0[t + r] = wt;
        g1[t + r] = wt * t;
        g2[t + r] = wt * t * t;
    }
    double s0 = 0, s2 = 0, s4 = 0;
    for (int t = -r; t <= r; ++t) {
        const double wt = g0[t + r];
        s0 += wt;
        s2 += wt * t * t;
        s4 += wt * t * t * t * t;
    }
    const double m00 = s0 * s0, m20 = s2 * s0, m40 = s4 * s0, m22 = s2 * s2;
    const double det = m00 * (m40 * m40 - m22 * m22) - m20 * (m20 * m40 - m22 * m20) +
                       m20 * (m20 * m22 - m40 * m20);
    const double inv_m20 = 1.0 / m20, inv_m22 = 1.0 / m22;
    const double i00 = (m40 * m40 - m22 * m22) / det;
    const double i01 = (m20 * m22 - m20 * m40) / det;
    const double i11 = (m00 * m40 - m20 * m20) / det;
    const double i12 = (m20 * m20 - m00 * m22) / det;

    const size_t n = (size_t)w * h;
    double* buf = (double*)malloc(sizeof(double) * n * 9);
    double *r0 = buf, *r1 = buf + n, *r2 = buf + 2 * n;
    double *s1 = buf + 3 * n, *sx = buf + 4 * n, *sy = buf + 5 * n, *sxx = buf + 6 * n,
           *syy = buf + 7 * n, *sxy = buf + 8 * n;
    correlate_rows(img, w, h, g0, r, r0);
    correlate_rows(img, w, h, g1, r, r1);
    correlate_rows(img, w, h, g2, r, r2);
    correlate_cols(r0, w, h, g0, r, s1);
    correlate_cols(r1, w, h, g0, r, sx);
    correlate_cols(r0, w, h, g1, r, sy);
    correlate_cols(r2, w, h, g0, r, sxx);
    correlate_cols(r0, w, h, g2, r, syy);
    correlate_cols(r1, w, h, g1, r, sxy);
    double *c = planes, *bx = planes + n, *by = planes + 2 * n, *a11 = planes + 3 * n,
           *a12 = planes + 4 * n, *a22 = planes + 5 * n;
    for (size_t i = 0; i < n; ++i) {
        bx[i] = sx[i] * inv_m20;
        by[i] = sy[i] * inv_m20;
        a12[i] = 0.5 * sxy[i] * inv_m22;
        c[i] = i00 * s1[i] + i01 * (sxx[i] + syy[i]);
        a11[i] = i01 * s1[i] + i11 * sxx[i] + i12 * syy[i];
        a22[i] = i01 * s1[i] + i12 * sxx[i] + i11 * syy[i];
    }
    free(buf);
    free(g0);
    free(g1);
    free(g2);
}

/* bilinear (flow.hpp:157-168). */
static double bilinear(const double* p, int w, int h, double x, double y) {
    x = clampd(x, 0.0, (double)(w - 1));
    y = clampd(y, 0.0, (double)(h - 1));
    const int xl = w - 2 >= 0 ? w - 2 : 0, yl = h - 2 >= 0 ? h - 2 : 0;
    const int x0 = (int)x < xl ? (int)x : xl;
    const int y0 = (int)y < yl ? (int)y : yl;
    const int x1 = x0 + 1 < w - 1 ? x0 + 1 : w - 1;
    const int y1 = y0 + 1 < h - 1 ? y0 + 1 : h - 1;
    const double fx = x - x0, fy = y - y0;
    const double top = p[(size_t)y0 * w + x0] * (1 - fx) + p[(size_t)y0 * w + x1] * fx;
    const double bot = p[(size_t)y1 * w + x0] * (1 - fx) + p[(size_t)y1 * w + x1] * fx;
    return top * (1 - fy) + bot * fy;
}

/* box_mean (flow.hpp:171-195): running sums with shrinking windows, rows then columns. */
static void box_mean(double* f, int w, int h, int radius, double* tmp) {
    for (int y = 0; y < h; ++y) {
        const double* row = f + (size_t)y * w;
        double* o = tmp + (size_t)y * w;
        double acc = 0.0;
        int lo = 0, hi = -1;
        for (int x = 0; x < w; ++x) {
            const int nlo = x - radius > 0 ? x - radius : 0;
            const int nhi = x + radius < w - 1 ? x + radius : w - 1;
            while (hi < nhi) acc += row[++hi];
            while (lo < nlo) acc -= row[lo++];
            o[x] = acc / (hi - lo + 1);
        }
    }
    for (int x = 0; x < w; ++x) {
        double acc = 0.0;
        int lo = 0, hi = -1;
        for (int y = 0; y < h; ++y) {
            const int nlo = y - radius > 0 ? y - radius : 0;
            const int nhi = y + radius < h - 1 ? y + radius : h - 1;
            while (hi < nhi) {
                ++hi;
                acc += tmp[(size_t)hi * w + x];
            }
            while (lo < nlo) {
                acc -= tmp[(size_t)lo * w + x];
                ++lo;
            }
            f[(size_t)y * w + x] = acc / (hi - lo + 1);
        }
    }
}

/* flow_step (flow.hpp:204-255). */
void oracle_flow_step(const double* prev_planes, const double* next_planes, int w, int h,
                      const float* prior_u, const float* prior_v, int window_size, float* out_u,
                      float* out_v) {
    const size_t n = (size_t)w * h;
    const double *pbx = prev_planes + n, *pby = prev_planes + 2 * n, *pa11 = prev_planes + 3 * n,
                 *pa12 = prev_planes + 4 * n, *pa22 = prev_planes + 5 * n;
    const double *nbx = next_planes + n, *nby = next_planes + 2 * n, *na11 = next_planes + 3 * n,
                 *na12 = next_planes + 4 * n, *na22 = next_planes + 5 * n;
    double* g = (double*)malloc(sizeof(double) * n * 6);
    double *g11 = g, *g12 = g + n, *g22 = g + 2 * n, *gh1 = g + 3 * n, *gh2 = g + 4 * n,
           *tmp = g + 5 * n;
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            const size_t i = (size_t)y * w + x;
            const double du = prior_u[i], dv = prior_v[i];
            const double sxp = x + du, syp = y + dv;
            const double a11 = 0.5 * (pa11[i] + bilinear(na11, w, h, sxp, syp));
            const double a12 = 0.5 * (pa12[i] + bilinear(na12, w, h, sxp, syp));
            const double a22 = 0.5 * (pa22[i] + bilinear(na22, w, h, sxp, syp));
            const double db1 = -0.5 * (bilinear(nbx, w, h, sxp, syp) - pbx[i]) + a11 * du + a12 * dv;
            const double db2 = -0.5 * (bilinear(nby, w, h, sxp, syp) - pby[i]) + a12 * du + a22 * dv;
            g11[i] = a11 * a11 + a12 * a12;
            g12[i] = (a11 + a22) * a12;
            g22[i] = a12 * a12 + a22 * a22;
            gh1[i] = a11 * db1 + a12 * db2;
            gh2[i] = a12 * db1 + a22 * db2;
        }
    const int radius = (window_size - 1) / 2;
    box_mean(g11, w, h, radius, tmp);
    box_mean(g12, w, h, radius, tmp);
    box_mean(g22, w, h, radius, tmp);
    box_mean(gh1, w, h, radius, tmp);
    box_mean(gh2, w, h, radius, tmp);
    for (size_t i = 0; i < n; ++i) {
        const double det = g11[i] * g22[i] - g12[i] * g12[i];
        const double frob2 = g11[i] * g11[i] + 2.0 * g12[i] * g12[i] + g22[i] * g22[i];
        if (!(det > 1e-9 * frob2)) {
            out_u[i] = prior_u[i];
            out_v[i] = prior_v[i];
            continue;
        }
        out_u[i] = (float)((g22[i] * gh1[i] - g12[i] * gh2[i]) / det);
        out_v[i] = (float)((-g12[i] * gh1[i] + g11[i] * gh2[i]) / det);
    }
    free(g);
}

/* gaussian_blur3 (flow.hpp:259-272). */
static void gaussian_blur3(const double* src, int w, int h, double sigma, double* out) {
    int radius = (int)ceil(2.5 * sigma);
    if (radius < 1) radius = 1;
    double* k = (double*)malloc(sizeof(double) * (2 * radius + 1));
    double sum = 0.0;
    for (int t = -radius; t <= radius; ++t) {
        k[t + radius] = exp(-(double)t * t / (2.0 * sigma * sigma));
        sum += k[t + radius];
    }
    for (int i = 0; i < 2 * radius + 1; ++i) k[i] /= sum;
    double* tmp = (double*)malloc(sizeof(double) * (size_t)w * h);
    correlate_rows(src, w, h, k, radius, tmp);
    correlate_cols(tmp, w, h, k, radius, out);
    free(tmp);
    free(k);
}

/* resize_bilinear (flow.hpp:274-285). */
static void resize_bilinear(const double* src, int w, int h, int tw, int th, double* out) {
    const double sx = (double)w / tw, sy = (double)h / th;
    for (int y = 0; y < th; ++y) {
        const double srcy = (y + 0.5) * sy - 0.5;
        for (int x = 0; x < tw; ++x) {
            const double srcx = (x + 0.5) * sx - 0.5;
            out[(size_t)y * tw + x] = bilinear(src, w, h, srcx, srcy);
        }
    }
}

#define MAX_LEVELS 32

/* build_pyramid (flow.hpp:287-298): stops before a level narrower than 32 px. */
static int build_pyramid(double* base, int w, int h, int levels, double scale, double** pyr,
                         int* pw, int* ph) {
    pyr[0] = base;
    pw[0] = w;
    ph[0] = h;
    int n = 1;
    for (int l = 1; l < levels && l < MAX_LEVELS; ++l) {
        const int cw = pw[n - 1], ch = ph[n - 1];
        const int tw = (int)(cw * scale), th = (int)(ch * scale);
        if (tw < 32 || th < 32) break;
        double* blurred = (double*)malloc(sizeof(double) * (size_t)cw * ch);
        gaussian_blur3(pyr[n - 1], cw, ch, 1.0, blurred);
        pyr[n] = (double*)malloc(sizeof(double) * (size_t)tw * th);
        resize_bilinear(blurred, cw, ch, tw, th, pyr[n]);
        free(blurred);
        pw[n] = tw;
        ph[n] = th;
        ++n;
    }
    return n;
}

static int validate_flow(const froi_params* p) {
    if (p->pyramid_levels < 1) return FROI_ERR_USAGE;
    if (!(p->pyramid_scale > 0.0 && p->pyramid_scale < 1.0)) return FROI_ERR_USAGE;
    if (p->window_size < 3 || p->window_size % 2 == 0) return FROI_ERR_USAGE;
    if (p->poly_n < 3 || p->poly_n % 2 == 0) return FROI_ERR_USAGE;
    if (p->iterations < 1) return FROI_ERR_USAGE;
    if (p->poly_sigma <= 0.0) return FROI_ERR_USAGE;
    return 0;
}

/* normalize_frame (core.hpp:141-146). */
static double* normalize_frame(const uint16_t* f, int w, int h, int depth) {
    const size_t n = (size_t)w * h;
    double* out = (double*)malloc(sizeof(double) * n);
    const double scale = 1.0 / ((1 << depth) - 1);
    for (size_t i = 0; i < n; ++i) out[i] = f[i] * scale;
    return out;
}

/* compute_flow (flow.hpp:304-345). */
int oracle_compute_flow(const uint16_t* prev, const uint16_t* next, int w, int h, int depth,
                        const froi_params* p, float* u, float* v) {
    if (validate_flow(p)) return FROI_ERR_USAGE;
    double *pa[MAX_LEVELS], *pb[MAX_LEVELS];
    int lw[MAX_LEVELS], lh[MAX_LEVELS], lw2[MAX_LEVELS], lh2[MAX_LEVELS];
    const int na = build_pyramid(normalize_frame(prev, w, h, depth), w, h, p->pyramid_levels,
                                 p->pyramid_scale, pa, lw, lh);
    const int nb = build_pyramid(normalize_frame(next, w, h, depth), w, h, p->pyramid_levels,
                                 p->pyramid_scale, pb, lw2, lh2);
    (void)nb;
    float *fu = NULL, *fv = NULL;
    int fw = 0, fh = 0;
    for (int l = na - 1; l >= 0; --l) {
        const int aw = lw[l], ah = lh[l];
        const size_t n = (size_t)aw * ah;
        float* nu = (float*)calloc(n, sizeof(float));
        float* nv = (float*)calloc(n, sizeof(float));
        if (fw != 0) {
            const double fx = (double)aw / fw, fy = (double)ah / fh;
            const size_t fn = (size_t)fw * fh;
            double* cu = (double*)malloc(sizeof(double) * fn);
            double* cv = (double*)malloc(sizeof(double) * fn);
            for (size_t i = 0; i < fn; ++i) {
                cu[i] = fu[i];
                cv[i] = fv[i];
            }
            for (int y = 0; y < ah; ++y) {
                const double sy = (y + 0.5) / fy - 0.5;
                for (int x = 0; x < aw; ++x) {
                    const double sx = (x + 0.5) / fx - 0.5;
                    const size_t i = (size_t)y * aw + x;
                    nu[i] = (float)(bilinear(cu, fw, fh, sx, sy) * fx);
                    nv[i] = (float)(bilinear(cv, fw, fh, sx, sy) * fy);
                }
            }
            free(cu);
            free(cv);
        }
        free(fu);
        free(fv);
        fu = nu;
        fv = nv;
        fw = aw;
        fh = ah;
        double* ea = (double*)malloc(sizeof(double) * n * 6);
        double* eb = (double*)malloc(sizeof(double) * n * 6);
        oracle_polynomial_expansion(pa[l], aw, ah, p->poly_n, p->poly_sigma, ea);
        oracle_polynomial_expansion(pb[l], aw, ah, p->poly_n, p->poly_sigma, eb);
        float* tu = (float*)malloc(sizeof(float) * n);
        float* tv = (float*)malloc(sizeof(float) * n);
        for (int it = 0; it < p->iterations; ++it) {
            oracle_flow_step(ea, eb, aw, ah, fu, fv, p->window_size, tu, tv);
            float* s;
            s = fu; fu = tu; tu = s;
            s = fv; fv = tv; tv = s;
        }
        free(tu);
        free(tv);
        free(ea);
        free(eb);
    }
    memcpy(u, fu, sizeof(float) * (size_t)w * h);
    memcpy(v, fv, sizeof(float) * (size_t)w * h);
    free(fu);
    free(fv);
    for (int l = 0; l < na; ++l) free(pa[l]);
    for (int l = 0; l < na; ++l) free(pb[l]);
    return 0;
}

/* ------------------------------------------------------------------ roi.hpp */

/* k-th smallest (0-based) of a[0..n-1]; reorders a.  Any exact selection returns the same
 * value as std::nth_element; three-way partitioning keeps heavily tied inputs linear. */
static void swapd(double* a, double* b) {
    const double t = *a;
    *a = *b;
    *b = t;
}

static double select_kth(double* a, size_t n, size_t k) {
    size_t lo = 0, hi = n; /* [lo, hi) */
    while (hi - lo > 16) {
        double x = a[lo], y = a[lo + (hi - lo) / 2], z = a[hi - 1];
        double pivot = x < y ? (y < z ? y : (x < z ? z : x)) : (x < z ? x : (y < z ? z : y));
        size_t lt = lo, i = lo, gt = hi;
        while (i < gt) {
            if (a[i] < pivot) swapd(&a[lt++], &a[i++]);
            else if (pivot < a[i]) swapd(&a[i], &a[--gt]);
            else ++i;
        }
        if (k < lt) hi = lt;
        else if (k >= gt) lo = gt;
        else return pivot;
    }
    for (size_t i = lo + 1; i < hi; ++i) {
        const double v = a[i];
        size_t j = i;
        while (j > lo && a[j - 1] > v) {
            a[j] = a[j - 1];
            --j;
        }
        a[j] = v;
    }
    return a[k];
}

/* robust_normalize (roi.hpp:47-63). */
static void robust_normalize(double* v, size_t n, double* lo_out, double* hi_out) {
    if (n == 0) return;
    double* sorted = (double*)malloc(sizeof(double) * n);
    memcpy(sorted, v, sizeof(double) * n);
    const size_t ilo = (size_t)(0.01 * (double)(n - 1));
    const size_t ihi = (size_t)(0.99 * (double)(n - 1));
    const double lo = select_kth(sorted, n, ilo);
    const double hi = select_kth(sorted, n, ihi);
    free(sorted);
    if (lo_out) *lo_out = lo;
    if (hi_out) *hi_out = hi;
    if (!(hi - lo > 1e-12)) {
        memset(v, 0, sizeof(double) * n);
        return;
    }
    const double inv = 1.0 / (hi - lo);
    for (size_t i = 0; i < n; ++i) v[i] = clampd((v[i] - lo) * inv, 0.0, 1.0);
}

/* gradient_magnitude (roi.hpp:65-74). */
static void gradient_magnitude(const double* img, int w, int h, double* g) {
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            const double gx = 0.5 * (img[(size_t)y * w + clampi(x + 1, 0, w - 1)] -
                                     img[(size_t)y * w + clampi(x - 1, 0, w - 1)]);
            const double gy = 0.5 * (img[(size_t)clampi(y + 1, 0, h - 1) * w + x] -
                                     img[(size_t)clampi(y - 1, 0, h - 1) * w + x]);
            g[(size_t)y * w + x] = hypot(gx, gy);
        }
}

/* saliency (roi.hpp:81-103). */
int oracle_saliency(const float* u, const float* v, const uint16_t* frame, int w, int h,
                    int depth, double flow_weight, int gradient_source, double* out,
                    oracle_pair_debug* dbg) {
    const size_t n = (size_t)w * h;
    double* fmag = (double*)malloc(sizeof(double) * n);
    double* grad = (double*)malloc(sizeof(double) * n);
    for (size_t i = 0; i < n; ++i) fmag[i] = hypotf(u[i], v[i]); /* FlowField::mag, core.hpp:117 */
    if (gradient_source == FROI_GRADIENT_IMAGE) {
        double* img = normalize_frame(frame, w, h, depth);
        gradient_magnitude(img, w, h, grad);
        free(img);
    } else {
        gradient_magnitude(fmag, w, h, grad);
    }
    double flo = 0, fhi = 0, glo = 0, ghi = 0;
    robust_normalize(fmag, n, &flo, &fhi);
    robust_normalize(grad, n, &glo, &ghi);
    if (dbg) {
        dbg->fmag_lo = flo;
        dbg->fmag_hi = fhi;
        dbg->grad_lo = glo;
        dbg->grad_hi = ghi;
    }
    for (size_t i = 0; i < n; ++i) out[i] = flow_weight * fmag[i] + (1.0 - flow_weight) * grad[i];
    free(fmag);
    free(grad);
    return 0;
}

/* threshold_mask (roi.hpp:109-138). */
int oracle_threshold_mask(const double* map, int w, int h, double roi_threshold, uint8_t* mask,
                          oracle_threshold_info* info) {
    if (!(roi_threshold > 0.0 && roi_threshold < 1.0)) return FROI_ERR_USAGE;
    const size_t n = (size_t)w * h;
    oracle_threshold_info li;
    memset(&li, 0, sizeof(li));
    memset(mask, 0, n);
    const size_t target = (size_t)llround(roi_threshold * (double)n);
    li.target = target;
    if (target == 0) {
        li.degenerate = 1;
        if (info) *info = li;
        return 0;
    }
    double* sorted = (double*)malloc(sizeof(double) * n);
    memcpy(sorted, map, sizeof(double) * n);
    const double boundary = select_kth(sorted, n, n - target); /* (target-1)-th largest */
    free(sorted);
    li.boundary = boundary;
    if (!(boundary > 0.0)) {
        for (size_t i = 0; i < n; ++i) {
            mask[i] = map[i] > 0.0 ? 1 : 0;
            li.count_greater += mask[i];
        }
        li.degenerate = 1;
        if (info) *info = li;
        return 0;
    }
    size_t selected = 0;
    for (size_t i = 0; i < n; ++i) {
        if (map[i] > boundary) {
            mask[i] = 1;
            ++selected;
        }
        if (map[i] == boundary) ++li.count_equal;
    }
    li.count_greater = selected;
    for (size_t i = 0; i < n && selected < target; ++i)
        if (map[i] == boundary) {
            mask[i] = 1;
            ++selected;
            ++li.ties_admitted;
        }
    if (info) *info = li;
    return 0;
}

/* morph_square (roi.hpp:144-172): separable, shrinking windows at the borders. */
static void morph_square(const uint8_t* m, int w, int h, int radius, int erode, uint8_t* out) {
    if (radius <= 0) {
        memcpy(out, m, (size_t)w * h);
        return;
    }
    uint8_t* tmp = (uint8_t*)malloc((size_t)w * h);
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            const int lo = x - radius > 0 ? x - radius : 0;
            const int hi = x + radius < w - 1 ? x + radius : w - 1;
            uint8_t acc = erode ? 1 : 0;
            for (int t = lo; t <= hi; ++t) {
                const uint8_t b = m[(size_t)y * w + t] != 0;
                if (erode) acc &= b;
                else acc |= b;
            }
            tmp[(size_t)y * w + x] = acc != 0;
        }
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            const int lo = y - radius > 0 ? y - radius : 0;
            const int hi = y + radius < h - 1 ? y + radius : h - 1;
            uint8_t acc = erode ? 1 : 0;
            for (int t = lo; t <= hi; ++t) {
                const uint8_t b = tmp[(size_t)t * w + x] != 0;
                if (erode) acc &= b;
                else acc |= b;
            }
            out[(size_t)y * w + x] = acc != 0;
        }
    free(tmp);
}

/* morph_open / morph_close (roi.hpp:176-180). */
void oracle_morph_open(const uint8_t* in, int w, int h, int radius, uint8_t* out) {
    uint8_t* t = (uint8_t*)malloc((size_t)w * h);
    morph_square(in, w, h, radius, 1, t);
    morph_square(t, w, h, radius, 0, out);
    free(t);
}
void oracle_morph_close(const uint8_t* in, int w, int h, int radius, uint8_t* out) {
    uint8_t* t = (uint8_t*)malloc((size_t)w * h);
    morph_square(in, w, h, radius, 0, t);
    morph_square(t, w, h, radius, 1, out);
    free(t);
}

static int uf_find(int* parent, int a) {
    while (parent[a] != a) {
        parent[a] = parent[parent[a]];
        a = parent[a];
    }
    return a;
}

/* label_components (roi.hpp:184-234): two-pass 8-connected union-find (W, NW, N, NE). */
size_t oracle_label_components(const uint8_t* mask, int w, int h, int* labels, size_t* areas,
                               size_t areas_capacity) {
    const size_t n = (size_t)w * h;
    int* lab = labels ? labels : (int*)malloc(sizeof(int) * n);
    memset(lab, 0, sizeof(int) * n);
    size_t cap = 1024, count = 1;
    int* parent = (int*)malloc(sizeof(int) * cap);
    parent[0] = 0;
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            if (!mask[(size_t)y * w + x]) continue;
            int best = 0;
            const int nx[4] = {x - 1, x - 1, x, x + 1};
            const int ny[4] = {y, y - 1, y - 1, y - 1};
            for (int k = 0; k < 4; ++k) {
                if (nx[k] < 0 || nx[k] >= w || ny[k] < 0) continue;
                const int nl = lab[(size_t)ny[k] * w + nx[k]];
                if (nl == 0) continue;
                if (best == 0) best = nl;
                else {
                    int a = uf_find(parent, best), b = uf_find(parent, nl);
                    if (a != b) parent[a > b ? a : b] = a < b ? a : b;
                }
            }
            if (best == 0) {
                if (count == cap) {
                    cap *= 2;
                    parent = (int*)realloc(parent, sizeof(int) * cap);
                }
                best = (int)count;
                parent[count++] = best;
            }
            lab[(size_t)y * w + x] = best;
        }
    int* remap = (int*)calloc(count, sizeof(int));
    int next = 0;
    for (size_t i = 0; i < n; ++i) {
        if (lab[i] == 0) continue;
        const int root = uf_find(parent, lab[i]);
        if (remap[root] == 0) remap[root] = ++next;
        lab[i] = remap[root];
    }
    if (areas) {
        for (size_t i = 0; i < areas_capacity; ++i) areas[i] = 0;
        for (size_t i = 0; i < n; ++i)
            if (lab[i] > 0 && (size_t)(lab[i] - 1) < areas_capacity) ++areas[lab[i] - 1];
    }
    free(remap);
    free(parent);
    if (!labels) free(lab);
    return (size_t)next;
}

/* morph_cleanup (roi.hpp:237-246). */
void oracle_morph_cleanup(uint8_t* mask, int w, int h, int open_radius, int close_radius,
                          int min_area) {
    const size_t n = (size_t)w * h;
    uint8_t* t = (uint8_t*)malloc(n);
    oracle_morph_open(mask, w, h, open_radius, t);
    oracle_morph_close(t, w, h, close_radius, mask);
    free(t);
    if (min_area <= 1) return;
    int* labels = (int*)malloc(sizeof(int) * n);
    const size_t nc = oracle_label_components(mask, w, h, labels, NULL, 0);
    size_t* areas = (size_t*)calloc(nc + 1, sizeof(size_t));
    for (size_t i = 0; i < n; ++i)
        if (labels[i] > 0) ++areas[labels[i]];
    for (size_t i = 0; i < n; ++i)
        if (labels[i] > 0 && areas[labels[i]] < (size_t)min_area) mask[i] = 0;
    free(areas);
    free(labels);
}

/* temporal_ensemble (roi.hpp:249-261). */
int oracle_temporal_ensemble(const uint8_t* masks, int n, int w, int h, int t, int k,
                             uint8_t* out) {
    if (t < 0 || t >= n) return FROI_ERR_DATA;
    const size_t px = (size_t)w * h;
    memcpy(out, masks + (size_t)t * px, px);
    const int lo = t >= k ? t - k : 0;
    const int hi = (n - 1) < t + k ? n - 1 : t + k;
    for (int j = lo; j <= hi; ++j) {
        if (j == t) continue;
        const uint8_t* mj = masks + (size_t)j * px;
        for (size_t i = 0; i < px; ++i) out[i] |= mj[i];
    }
    return 0;
}

static int validate_roi(const froi_params* p) {
    if (!(p->roi_threshold > 0.0 && p->roi_threshold < 1.0)) return FROI_ERR_USAGE;
    if (p->flow_weight < 0.0 || p->flow_weight > 1.0) return FROI_ERR_USAGE;
    if (p->adjacent_factor < 0) return FROI_ERR_USAGE;
    if (p->min_area < 0) return FROI_ERR_USAGE;
    if (p->open_radius < 0 || p->close_radius < 0) return FROI_ERR_USAGE;
    return 0;
}

/* roi.hpp:337-345: saliency on the raw registered frame, threshold, cleanup, unshift. */
int oracle_mask_from_flow(const float* u, const float* v, const uint16_t* raw_frame, int w,
                          int h, int depth, int dx, int dy, const froi_params* p, uint8_t* mask,
                          oracle_pair_debug* dbg) {
    const size_t n = (size_t)w * h;
    uint16_t* reg = (uint16_t*)malloc(sizeof(uint16_t) * n);
    oracle_apply_shift(raw_frame, w, h, dx, dy, reg);
    double* sal = (double*)malloc(sizeof(double) * n);
    oracle_saliency(u, v, reg, w, h, depth, p->flow_weight, p->gradient_source, sal, dbg);
    uint8_t* m = (uint8_t*)malloc(n);
    oracle_threshold_info ti;
    const int st = oracle_threshold_mask(sal, w, h, p->roi_threshold, m, &ti);
    if (dbg) dbg->thr = ti;
    if (st == 0) {
        oracle_morph_cleanup(m, w, h, p->open_radius, p->close_radius, p->min_area);
        oracle_unshift_mask(m, w, h, dx, dy, mask);
    }
    free(m);
    free(sal);
    free(reg);
    return st;
}

/* parallel_for (parallel.hpp:20-49): static block partition; outputs independent of workers. */
typedef struct {
    void (*fn)(void*, size_t);
    void* arg;
    size_t lo, hi;
} pf_job;

static void* pf_run(void* a) {
    pf_job* j = (pf_job*)a;
    for (size_t i = j->lo; i < j->hi; ++i) j->fn(j->arg, i);
    return NULL;
}

static void parallel_for(size_t n, int workers, void (*fn)(void*, size_t), void* arg) {
    if (n == 0) return;
    if (workers <= 1 || n == 1) {
        for (size_t i = 0; i < n; ++i) fn(arg, i);
        return;
    }
    const size_t nt = (size_t)workers < n ? (size_t)workers : n;
    const size_t chunk = (n + nt - 1) / nt;
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * nt);
    pf_job* jobs = (pf_job*)malloc(sizeof(pf_job) * nt);
    size_t started = 0;
    for (size_t t = 0; t < nt; ++t) {
        const size_t lo = t * chunk, hi = lo + chunk < n ? lo + chunk : n;
        if (lo >= hi) break;
        jobs[t].fn = fn;
        jobs[t].arg = arg;
        jobs[t].lo = lo;
        jobs[t].hi = hi;
        pthread_create(&th[t], NULL, pf_run, &jobs[t]);
        ++started;
    }
    for (size_t t = 0; t < started; ++t) pthread_join(th[t], NULL);
    free(jobs);
    free(th);
}

typedef struct {
    const uint16_t* frames;
    int n, w, h, depth;
    const froi_params* p;
    uint16_t* den;
    uint8_t* masks;
    froi_shift* shifts;
} extract_job;

static void extract_denoise_one(void* a, size_t i) {
    extract_job* j = (extract_job*)a;
    const size_t px = (size_t)j->w * j->h;
    oracle_denoise(j->frames + i * px, j->w, j->h, j->depth, j->p, j->den + i * px);
}

static void extract_pair_one(void* a, size_t idx) {
    extract_job* j = (extract_job*)a;
    const size_t t = idx + 1, px = (size_t)j->w * j->h;
    const uint16_t* da = j->den + (t - 1) * px;
    const uint16_t* db = j->den + t * px;
    froi_shift s;
    oracle_estimate_shift(da, db, j->w, j->h, j->p->max_shift, &s);
    if (s.confidence < 1.5) { /* kShiftConfidenceThreshold, registration.hpp:19 */
        s.dx = 0;
        s.dy = 0;
    }
    uint16_t* nb = (uint16_t*)malloc(sizeof(uint16_t) * px);
    oracle_apply_shift(db, j->w, j->h, s.dx, s.dy, nb);
    float* u = (float*)malloc(sizeof(float) * px);
    float* v = (float*)malloc(sizeof(float) * px);
    oracle_compute_flow(da, nb, j->w, j->h, j->depth, j->p, u, v);
    oracle_mask_from_flow(u, v, j->frames + t * px, j->w, j->h, j->depth, s.dx, s.dy, j->p,
                          j->masks + t * px, NULL);
    j->shifts[t] = s;
    free(u);
    free(v);
    free(nb);
}

typedef struct {
    const uint8_t* masks;
    uint8_t* out;
    int n, w, h, k;
} ensemble_job;

static void ensemble_one(void* a, size_t t) {
    ensemble_job* j = (ensemble_job*)a;
    oracle_temporal_ensemble(j->masks, j->n, j->w, j->h, (int)t, j->k,
                             j->out + t * (size_t)j->w * j->h);
}

/* extract_roi (roi.hpp:309-364). */
int oracle_extract_roi(const uint16_t* frames, int n, int w, int h, int depth,
                       const froi_params* p, int workers, uint8_t* masks, froi_shift* shifts,
                       double* raw_fractions) {
    if (validate_roi(p) || validate_flow(p)) return FROI_ERR_USAGE;
    if (n < 2) return FROI_ERR_DATA;
    if (validate_denoise(p)) return FROI_ERR_USAGE;
    const int mn = w < h ? w : h;
    if (p->max_shift < 1 || p->max_shift >= mn / 4) return FROI_ERR_USAGE;
    const size_t px = (size_t)w * h;
    extract_job j;
    j.frames = frames;
    j.n = n;
    j.w = w;
    j.h = h;
    j.depth = depth;
    j.p = p;
    j.den = (uint16_t*)malloc(sizeof(uint16_t) * px * n);
    j.masks = masks;
    j.shifts = (froi_shift*)calloc((size_t)n, sizeof(froi_shift));
    parallel_for((size_t)n, workers, extract_denoise_one, &j);
    parallel_for((size_t)n - 1, workers, extract_pair_one, &j);
    memcpy(masks, masks + px, px); /* frame 0 borrows frame 1 (roi.hpp:348) */
    j.shifts[0].dx = 0;
    j.shifts[0].dy = 0;
    j.shifts[0].confidence = 1.0;
    if (shifts) memcpy(shifts, j.shifts, sizeof(froi_shift) * (size_t)n);
    if (raw_fractions)
        for (int t = 0; t < n; ++t) {
            size_t c = 0;
            const uint8_t* m = masks + (size_t)t * px;
            for (size_t i = 0; i < px; ++i) c += m[i] != 0;
            raw_fractions[t] = px ? (double)c / (double)px : 0.0;
        }
    if (p->adjacent_factor > 0) {
        uint8_t* merged = (uint8_t*)malloc(px * n);
        ensemble_job e;
        e.masks = masks;
        e.out = merged;
        e.n = n;
        e.w = w;
        e.h = h;
        e.k = p->adjacent_factor;
        parallel_for((size_t)n, workers, ensemble_one, &e);
        memcpy(masks, merged, px * n);
        free(merged);
    }
    free(j.shifts);
    free(j.den);
    return 0;
}

/* glibc 2.39 __hypot for finite arguments (sysdeps/ieee754/dbl-64/e_hypot.c, non-FMA kernel
 * after Borges, "An Improved Algorithm for hypot(a,b)"), restated; the GPU kernels use the
 * same sequence.  Only the range reached by gradient and cross-power values is restated
 * (no over/underflow scaling): ay == 0 or ay <= ax*2^-54 returns ax + ay. */
double oracle_hypot_restated(double x, double y) {
    x = fabs(x);
    y = fabs(y);
    const double ax = x < y ? y : x, ay = x < y ? x : y;
    if (ay <= ax * 0x1p-54) return ax + ay;
    double hh = sqrt(ax * ax + ay * ay);
    double t1, t2;
    if (hh <= 2.0 * ay) {
        const double delta = hh - ay;
        t1 = ax * (2.0 * delta - ax);
        t2 = (delta - 2.0 * (ax - ay)) * delta;
    } else {
        const double delta = hh - ax;
        t1 = 2.0 * delta * (ax - 2.0 * ay);
        t2 = (4.0 * delta - ay) * ay + delta * delta;
    }
    hh -= (t1 + t2) / (2.0 * hh);
    return hh;
}


/* ======================================================================== 5/3 DWT (codec side) */
/* lift_53_forward / lift_53_inverse (dwt.hpp:36-63): whole-sample symmetric extension; >> on
 * negative int32 is the arithmetic (floor) shift the reference relies on (C++20). */
static int dwt_r(int i, int n) { return i + 1 < n ? i + 1 : n - 2; }
static int dwt_l(int i) { return i > 0 ? i - 1 : 1; }

static void lift53(int32_t* x, int n, int inverse) {
    if (n < 2) return;
    if (!inverse) {
        for (int i = 1; i < n; i += 2) x[i] -= (x[i - 1] + x[dwt_r(i, n)]) >> 1;
        for (int i = 0; i < n; i += 2) x[i] += (x[dwt_l(i)] + x[dwt_r(i, n)] + 2) >> 2;
    } else {
        for (int i = 0; i < n; i += 2) x[i] -= (x[dwt_l(i)] + x[dwt_r(i, n)] + 2) >> 2;
        for (int i = 1; i < n; i += 2) x[i] += (x[i - 1] + x[dwt_r(i, n)]) >> 1;
    }
}

/* evens to the front half (ceil), odds behind (dwt.hpp:65-83), or back */
static void dwt_shuffle(const int32_t* x, int n, int32_t* out, int interleave) {
    const int half = (n + 1) / 2;
    for (int i = 0; i < n; ++i) {
        const int j = (i % 2 == 0) ? i / 2 : half + i / 2;
        if (interleave) out[i] = x[j];
        else out[j] = x[i];
    }
}

static int dwt_extent(int n, int level) {
    for (int l = 0; l < level; ++l) n = (n + 1) / 2;
    return n;
}

int oracle_dwt_forward(const uint16_t* frame, int w, int h, int depth, int levels, int32_t* g) {
    if (levels < 1) return 1;
    if (w < (1 << levels) || h < (1 << levels)) return 2;
    const int32_t dc = 1 << (depth - 1);
    for (size_t i = 0; i < (size_t)w * h; ++i) g[i] = (int32_t)frame[i] - dc;
    const int nmax = w > h ? w : h;
    int32_t* line = (int32_t*)malloc(sizeof(int32_t) * nmax);
    int32_t* scr = (int32_t*)malloc(sizeof(int32_t) * nmax);
    for (int l = 0; l < levels; ++l) {
        const int lw = dwt_extent(w, l), lh = dwt_extent(h, l);
        for (int y = 0; y < lh; ++y) {
            memcpy(line, g + (size_t)y * w, sizeof(int32_t) * lw);
            lift53(line, lw, 0);
            dwt_shuffle(line, lw, scr, 0);
            memcpy(g + (size_t)y * w, scr, sizeof(int32_t) * lw);
        }
        for (int x = 0; x < lw; ++x) {
            for (int y = 0; y < lh; ++y) line[y] = g[(size_t)y * w + x];
            lift53(line, lh, 0);
            dwt_shuffle(line, lh, scr, 0);
            for (int y = 0; y < lh; ++y) g[(size_t)y * w + x] = scr[y];
        }
    }
    free(line);
    free(scr);
    return 0;
}

int oracle_dwt_inverse(const int32_t* coeffs, int w, int h, int depth, int levels, uint16_t* frame) {
    if (levels < 1) return 1;
    int32_t* g = (int32_t*)malloc(sizeof(int32_t) * (size_t)w * h);
    memcpy(g, coeffs, sizeof(int32_t) * (size_t)w * h);
    const int nmax = w > h ? w : h;
    int32_t* line = (int32_t*)malloc(sizeof(int32_t) * nmax);
    int32_t* scr = (int32_t*)malloc(sizeof(int32_t) * nmax);
    for (int l = levels - 1; l >= 0; --l) {
        const int lw = dwt_extent(w, l), lh = dwt_extent(h, l);
        for (int x = 0; x < lw; ++x) {
            for (int y = 0; y < lh; ++y) line[y] = g[(size_t)y * w + x];
            dwt_shuffle(line, lh, scr, 1);
            lift53(scr, lh, 1);
            for (int y = 0; y < lh; ++y) g[(size_t)y * w + x] = scr[y];
        }
        for (int y = 0; y < lh; ++y) {
            memcpy(line, g + (size_t)y * w, sizeof(int32_t) * lw);
            dwt_shuffle(line, lw, scr, 1);
            lift53(scr, lw, 1);
            memcpy(g + (size_t)y * w, scr, sizeof(int32_t) * lw);
        }
    }
    /* clamp_to_depth(double(c + dc)) (core.hpp): integers clamp to [0, maxval] */
    const int32_t dc = 1 << (depth - 1), mx = (int32_t)((1u << depth) - 1u);
    for (size_t i = 0; i < (size_t)w * h; ++i) {
        const int32_t v = g[i] + dc;
        frame[i] = (uint16_t)(v < 0 ? 0 : (v > mx ? mx : v));
    }
    free(g);
    free(line);
    free(scr);
    return 0;
}

size_t oracle_map_mask_to_subbands(const uint8_t* mask, int w, int h, int levels, uint8_t* out) {
    int any = 0;
    for (size_t i = 0; i < (size_t)w * h && !any; ++i) any = mask[i] != 0;
    const uint8_t* cur = mask;
    int cw = w, ch = h;
    size_t off = 0;
    uint8_t* down = NULL;
    for (int l = 1; l <= levels; ++l) {
        const int nw = (cw + 1) / 2, nh = (ch + 1) / 2;
        free(down);
        down = (uint8_t*)calloc((size_t)nw * nh, 1);
        if (any)
            for (int y = 0; y < ch; ++y)
                for (int x = 0; x < cw; ++x)
                    if (cur[(size_t)y * cw + x]) down[(size_t)(y / 2) * nw + x / 2] = 1;
        uint8_t* lev = out + off;
        if (any) morph_square(down, nw, nh, 2, 0, lev);
        else memcpy(lev, down, (size_t)nw * nh);
        cur = lev;
        cw = nw;
        ch = nh;
        off += (size_t)nw * nh;
    }
    free(down);
    return off;
}
