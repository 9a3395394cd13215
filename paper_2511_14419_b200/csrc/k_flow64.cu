// k_flow64.cu — the bit-exact flow mode (froi_ctx_set_flow_exact): the reference's fp64
// compute_flow (flow.hpp:259-345) operation for operation, so the flow, and with it every mask,
// is byte-identical to the reference's instead of within the fp32 flow tolerance.
//
// Every fp64 step uses the explicit round-to-nearest intrinsics (no contraction), in the
// reference's evaluation order; host-side constants (Gaussian taps, moment inverses) are computed
// with the reference's expressions by the host compiler (make_flow64_const, runtime.cu).
//
//   k64_norm0[_shifted]  normalize_frame(apply_shift(den, s)) (core.hpp:141-146,
//                        registration.hpp:100-107) into the level-0 image, double
//   k64_blur_rows        gaussian_blur3's correlate_rows (flow.hpp:55-70, 259-272)
//   k64_blur_cols_resize correlate_cols (flow.hpp:72-84) at the four bilinear taps of each output
//                        pixel of resize_bilinear (flow.hpp:274-285) -> the next pyramid level
//   k64_polyexp          polynomial_expansion (flow.hpp:118-153): the three row correlations of a
//                        tile's rows into shared memory, then the six column correlations and the
//                        moment-inverse combination -> planes bx, by, a11, a12, a22 (c is unused)
//   k64_products         flow_step's per-pixel normal-equation terms (flow.hpp:204-233)
//   k64_box_rows         box_mean's row pass (flow.hpp:171-195): the reference's running sums are
//                        sequential along each row (the rounding of every partial sum is part of
//                        the result), so one thread walks one row of one plane, its inputs staged
//                        through shared memory in coalesced chunks
//   k64_box_cols_solve   box_mean's column pass, one thread per column with the five planes'
//                        running sums, fused with the 2x2 solve and its singular fallback
//                        (flow.hpp:236-253)
//   k64_upsample         compute_flow's coarse-to-fine prior (flow.hpp:318-337)
// Throughput is bounded by those sequential box-mean walks and by HBM (five double planes per
// pass); the default fp32 flow (k_flow.cu) remains the fast path.
#include "kernels.cuh"

namespace froi {
namespace {

constexpr int kNT = 256;

__device__ __forceinline__ double clampd(double v, double lo, double hi) {
    return v < lo ? lo : (hi < v ? hi : v);
}

// bilinear (flow.hpp:157-168): index split shared by the planes sampled at one point
struct Bl {
    int i00, i01, i10, i11;
    double fx, fy, ofx, ofy;
    __device__ __forceinline__ void setup(int w, int h, double x, double y) {
        x = clampd(x, 0.0, (double)(w - 1));
        y = clampd(y, 0.0, (double)(h - 1));
        const int xl = w - 2 >= 0 ? w - 2 : 0, yl = h - 2 >= 0 ? h - 2 : 0;
        const int x0 = (int)x < xl ? (int)x : xl;
        const int y0 = (int)y < yl ? (int)y : yl;
        const int x1 = x0 + 1 < w - 1 ? x0 + 1 : w - 1;
        const int y1 = y0 + 1 < h - 1 ? y0 + 1 : h - 1;
        fx = dsub(x, (double)x0);
        fy = dsub(y, (double)y0);
        ofx = dsub(1.0, fx);
        ofy = dsub(1.0, fy);
        i00 = y0 * w + x0;
        i01 = y0 * w + x1;
        i10 = y1 * w + x0;
        i11 = y1 * w + x1;
        FROI_DCHECK(x0 >= 0 && y0 >= 0 && i11 < w * h && i00 <= i11);
    }
    __device__ __forceinline__ double at(const double* p) const {
        const double top = dadd(dmul(p[i00], ofx), dmul(p[i01], fx));
        const double bot = dadd(dmul(p[i10], ofx), dmul(p[i11], fx));
        return dadd(dmul(top, ofy), dmul(bot, fy));
    }
};

// ------------------------------------------------------------------ pyramid
template <typename T>
__global__ void __launch_bounds__(kNT) k64_norm0(Geom g, double inv, const T* __restrict__ den,
                                                 double* __restrict__ img) {
    const int s = blockIdx.y;
    const long long n = (long long)g.W * g.H;
    const long long i = (long long)blockIdx.x * kNT + threadIdx.x;
    if (i >= n) return;
    img[(size_t)s * g.lsum + i] = dmul((double)den[(size_t)s * n + i], inv);
}

template <typename T>
__global__ void __launch_bounds__(kNT) k64_norm0_shifted(Geom g, double inv, const T* __restrict__ den,
                                                         const int* __restrict__ next,
                                                         const PairInfo* __restrict__ info,
                                                         double* __restrict__ img) {
    const int p = blockIdx.y;
    const PairInfo I = info[p];
    if (!I.shifted) return;
    const long long n = (long long)g.W * g.H;
    const long long i = (long long)blockIdx.x * kNT + threadIdx.x;
    if (i >= n) return;
    const int y = (int)(i / g.W), x = (int)(i - (long long)y * g.W);
    const T* f = den + (size_t)next[p] * n;
    const int v = f[(size_t)clampi(y + I.dy, 0, g.H - 1) * g.W + clampi(x + I.dx, 0, g.W - 1)];
    img[(size_t)p * g.lsum + i] = dmul((double)v, inv);
}

// correlate_rows with the normalised Gaussian of gaussian_blur3, level l -> tmp (item stride W*H)
__global__ void __launch_bounds__(kNT) k64_blur_rows(Geom g, Flow64Const C, int l, const double* __restrict__ img,
                                                     const PairInfo* __restrict__ info, double* __restrict__ tmp) {
    const int it = blockIdx.y;
    if (info && !info[it].shifted) return;
    const int w = g.lw[l], h = g.lh[l];
    const long long i = (long long)blockIdx.x * kNT + threadIdx.x;
    if (i >= (long long)w * h) return;
    const int y = (int)(i / w), x = (int)(i - (long long)y * w);
    const double* row = img + (size_t)it * g.lsum + g.loff[l] + (size_t)y * w;
    const int r = C.blur_r;
    double acc = 0.0;
    for (int t = -r; t <= r; ++t) acc = dadd(acc, dmul(C.blur[t + r], row[clampi(x + t, 0, w - 1)]));
    tmp[(size_t)it * g.W * g.H + i] = acc;
}

// correlate_cols of the row-blurred level l at the four taps of each level-(l+1) pixel, then the
// bilinear resample at ((x + 0.5) * sx - 0.5, (y + 0.5) * sy - 0.5)
__global__ void __launch_bounds__(kNT) k64_blur_cols_resize(Geom g, Flow64Const C, int l,
                                                            const double* __restrict__ tmp,
                                                            const PairInfo* __restrict__ info,
                                                            double* __restrict__ img) {
    const int it = blockIdx.y;
    if (info && !info[it].shifted) return;
    const int w = g.lw[l], h = g.lh[l], tw = g.lw[l + 1], th = g.lh[l + 1];
    const long long i = (long long)blockIdx.x * kNT + threadIdx.x;
    if (i >= (long long)tw * th) return;
    const int y = (int)(i / tw), x = (int)(i - (long long)y * tw);
    const double sx = ddiv((double)w, (double)tw), sy = ddiv((double)h, (double)th);
    const double srcx = dsub(dmul(dadd((double)x, 0.5), sx), 0.5);
    const double srcy = dsub(dmul(dadd((double)y, 0.5), sy), 0.5);
    Bl b;
    b.setup(w, h, srcx, srcy);
    const double* src = tmp + (size_t)it * g.W * g.H;
    const int r = C.blur_r;
    auto blurred = [&](int idx) {
        const int yy = idx / w, xx = idx - yy * w;
        double o = 0.0;
        for (int t = -r; t <= r; ++t) o = dadd(o, dmul(C.blur[t + r], src[(size_t)clampi(yy + t, 0, h - 1) * w + xx]));
        return o;
    };
    const double p00 = blurred(b.i00), p01 = blurred(b.i01), p10 = blurred(b.i10), p11 = blurred(b.i11);
    const double top = dadd(dmul(p00, b.ofx), dmul(p01, b.fx));
    const double bot = dadd(dmul(p10, b.ofx), dmul(p11, b.fx));
    img[(size_t)it * g.lsum + g.loff[l + 1] + i] = dadd(dmul(top, b.ofy), dmul(bot, b.fy));
}

// ------------------------------------------------------------------ polynomial expansion
constexpr int PEX = 32, PEY = 16, PER = 7;  // tile, max radius (poly_n <= 15)

__global__ void __launch_bounds__(kNT) k64_polyexp(Geom g, Flow64Const C, int l, const double* __restrict__ img,
                                                   const PairInfo* __restrict__ info, double* __restrict__ ex) {
    __shared__ double rs[3][PEY + 2 * PER][PEX];
    const int it = blockIdx.z;
    if (info && !info[it].shifted) return;
    const int w = g.lw[l], h = g.lh[l];
    const int x0 = blockIdx.x * PEX, y0 = blockIdx.y * PEY;
    const int r = C.poly_r;
    const double* src = img + (size_t)it * g.lsum + g.loff[l];
    // row correlations r0, r1, r2 (g0 = w, g1 = w t, g2 = w t^2) of rows y0 - r .. y0 + PEY + r
    for (int k = threadIdx.x; k < (PEY + 2 * r) * PEX; k += kNT) {
        const int j = k / PEX, i = k - j * PEX;
        const int x = x0 + i;
        if (x >= w) continue;
        const double* row = src + (size_t)clampi(y0 - r + j, 0, h - 1) * w;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0;
        for (int t = -r; t <= r; ++t) {
            const double v = row[clampi(x + t, 0, w - 1)];
            a0 = dadd(a0, dmul(C.g0[t + r], v));
            a1 = dadd(a1, dmul(C.g1[t + r], v));
            a2 = dadd(a2, dmul(C.g2[t + r], v));
        }
        rs[0][j][i] = a0;
        rs[1][j][i] = a1;
        rs[2][j][i] = a2;
    }
    __syncthreads();
    const size_t ls = g.lsum, base = (size_t)it * 5 * ls + g.loff[l];
    for (int k = threadIdx.x; k < PEY * PEX; k += kNT) {
        const int jj = k / PEX, i = k - jj * PEX;
        const int x = x0 + i, y = y0 + jj;
        if (x >= w || y >= h) continue;
        double s1 = 0.0, sx = 0.0, sy = 0.0, sxx = 0.0, syy = 0.0, sxy = 0.0;
        for (int t = -r; t <= r; ++t) {
            // correlate_cols reads row clamp(y + t): tile row jj + r + t holds exactly that row
            const int j = jj + r + t;
            const double q0 = rs[0][j][i], q1 = rs[1][j][i], q2 = rs[2][j][i];
            s1 = dadd(s1, dmul(C.g0[t + r], q0));
            sx = dadd(sx, dmul(C.g0[t + r], q1));
            sy = dadd(sy, dmul(C.g1[t + r], q0));
            sxx = dadd(sxx, dmul(C.g0[t + r], q2));
            syy = dadd(syy, dmul(C.g2[t + r], q0));
            sxy = dadd(sxy, dmul(C.g1[t + r], q1));
        }
        const size_t o = base + (size_t)y * w + x;
        ex[o] = dmul(sx, C.inv_m20);                                                  // bx
        ex[o + ls] = dmul(sy, C.inv_m20);                                             // by
        ex[o + 2 * ls] = dadd(dadd(dmul(C.i01, s1), dmul(C.i11, sxx)), dmul(C.i12, syy));  // a11
        ex[o + 3 * ls] = dmul(dmul(0.5, sxy), C.inv_m22);                             // a12
        ex[o + 4 * ls] = dadd(dadd(dmul(C.i01, s1), dmul(C.i12, sxx)), dmul(C.i11, syy));  // a22
    }
}

// ------------------------------------------------------------------ flow step
// flow_step's five normal-equation terms g11, g12, g22, gh1, gh2 at pixel (x, y) of level l:
// pe / ne are the previous / next frame's expansion planes at the level, (du, dv) the prior
struct Prod5 {
    double v[5];
};
__device__ __forceinline__ Prod5 products_at(int w, int h, size_t ls, const double* pe, const double* ne, int x,
                                             int y, double du, double dv) {
    const size_t i = (size_t)y * w + x;
    Bl b;
    b.setup(w, h, dadd((double)x, du), dadd((double)y, dv));
    const double a11 = dmul(0.5, dadd(pe[2 * ls + i], b.at(ne + 2 * ls)));
    const double a12 = dmul(0.5, dadd(pe[3 * ls + i], b.at(ne + 3 * ls)));
    const double a22 = dmul(0.5, dadd(pe[4 * ls + i], b.at(ne + 4 * ls)));
    const double db1 = dadd(dadd(dmul(-0.5, dsub(b.at(ne), pe[i])), dmul(a11, du)), dmul(a12, dv));
    const double db2 = dadd(dadd(dmul(-0.5, dsub(b.at(ne + ls), pe[ls + i])), dmul(a12, du)), dmul(a22, dv));
    Prod5 o;
    o.v[0] = dadd(dmul(a11, a11), dmul(a12, a12));
    o.v[1] = dmul(dadd(a11, a22), a12);
    o.v[2] = dadd(dmul(a12, a12), dmul(a22, a22));
    o.v[3] = dadd(dmul(a11, db1), dmul(a12, db2));
    o.v[4] = dadd(dmul(a12, db1), dmul(a22, db2));
    return o;
}

// products of flow_step: planes g11, g12, g22, gh1, gh2 into prod[pair][5][W*H]
__global__ void __launch_bounds__(kNT) k64_products(Geom g, int l, int mode, const double* __restrict__ ex_f,
                                                    const double* __restrict__ ex_p, const int* __restrict__ prev,
                                                    const int* __restrict__ next, const PairInfo* __restrict__ info,
                                                    const float2* __restrict__ flow_in, double* __restrict__ prod) {
    const int p = blockIdx.y;
    const int w = g.lw[l], h = g.lh[l];
    const long long i = (long long)blockIdx.x * kNT + threadIdx.x;
    if (i >= (long long)w * h) return;
    const int y = (int)(i / w), x = (int)(i - (long long)y * w);
    const size_t ls = g.lsum;
    const double* pe = ex_f + (size_t)prev[p] * 5 * ls + g.loff[l];
    const double* ne = (info[p].shifted ? ex_p + (size_t)p * 5 * ls : ex_f + (size_t)next[p] * 5 * ls) + g.loff[l];
    double du = 0.0, dv = 0.0;
    if (mode) {
        const float2 f = flow_in[(size_t)p * ls + g.loff[l] + i];
        du = (double)f.x;
        dv = (double)f.y;
    }
    const Prod5 o = products_at(w, h, ls, pe, ne, x, y, du, dv);
    const size_t n0 = (size_t)g.W * g.H;
    double* d = prod + (size_t)p * 5 * n0 + i;
#pragma unroll
    for (int q = 0; q < 5; ++q) d[q * n0] = o.v[q];
}

// acc / count for box_mean: the divisor is a small integer, so its refined reciprocal is
// computed once per count and the quotient takes the division's fast path (bit-identical to
// __ddiv_rn whenever its range test passes; the rare rest, e.g. acc == 0, redone exactly)
__device__ __forceinline__ double div_count(double acc, double m, double r2) {
    bool ok;
    const double q = ddiv_fast(acc, m, r2, ok);
    return ok ? q : ddiv(acc, m);
}

// box_mean's running sum (flow.hpp:171-195) along a line of n values, as the reference orders
// it: position 0 adds v[0..min(R, n-1)]; each later x adds v[x+R] (while x + R < n), then
// subtracts v[x-R-1] (once x - R > 0); the mean divides by the clipped window's count.
struct BoxWalk {
    int n, R;
    double r_int;  // reciprocal of the interior count 2R+1
    __device__ __forceinline__ int count(int x) const {
        const int lo = x - R > 0 ? x - R : 0, hi = x + R < n - 1 ? x + R : n - 1;
        return hi - lo + 1;
    }
    __device__ __forceinline__ double mean(double acc, int x) const {
        const int c = count(x);
        return c == 2 * R + 1 ? div_count(acc, (double)c, r_int) : ddiv(acc, (double)c);
    }
};

__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// box_mean's row pass, coalesced: a CTA takes RB rows of one (pair, plane) and walks them in
// chunks of CW columns, each staged with its CH-column history on either side (R < CH) into a
// shared tile by cp.async (every load of the chunk in flight at once; small tiles keep many CTAs
// per SM, which is what hides the latency).  One thread per row runs the sequential running sum,
// writing each mean in place over the input it no longer needs; the CW means then leave as whole
// row segments.
#ifndef FROI_K64_RB
#define FROI_K64_RB 32
#endif
#ifndef FROI_K64_CMINB
#define FROI_K64_CMINB 5
#endif
#ifndef FROI_K64_SB
#define FROI_K64_SB 8
#endif
constexpr int RB = FROI_K64_RB, CW = 32, CH = 8, SW = CW + 2 * CH, TWC = SW + 1;  // TWC: odd row stride
constexpr int SB = FROI_K64_SB;  // walk steps whose inputs are loaded together
static_assert(CW % SB == 0 && 16 % SB == 0, "walk blocks");

__global__ void __launch_bounds__(RB) k64_box_rows(Geom g, int l, int R, const double* __restrict__ in,
                                                   double* __restrict__ out) {
    extern __shared__ double sm[];  // two tiles [RB][TWC]
    const int w = g.lw[l], h = g.lh[l];
    const int y0 = blockIdx.x * RB, pl = blockIdx.y, p = blockIdx.z;
    const size_t n0 = (size_t)g.W * g.H;
    const double* src = in + ((size_t)p * 5 + pl) * n0 + (size_t)y0 * w;
    double* dst = out + ((size_t)p * 5 + pl) * n0 + (size_t)y0 * w;
    const int rows = min(RB, h - y0);
    const int r = threadIdx.x;
    FROI_DCHECK(R < CH && rows > 0);
    const BoxWalk bw{w, R, drcp_refined((double)(2 * R + 1))};
    static_assert(RB % 32 == 0 && SW <= 64 && CW == 32, "staging: a warp covers a tile row in two steps");
    const int lane = threadIdx.x & 31, wrp = threadIdx.x >> 5;
    // a warp stages whole tile rows (lane = column, then lane + 32): no index division per element
    auto stage = [&](int c0, double* tile) {
        const int xa = c0 - CH + lane, xb = xa + 32;
        const bool oka = xa >= 0 && xa < w, okb = lane + 32 < SW && xb < w;
        const double* s = src + (size_t)wrp * w;
        double* d = tile + wrp * TWC + lane;
        for (int rr = wrp; rr < rows; rr += RB / 32, s += (size_t)(RB / 32) * w, d += (RB / 32) * TWC) {
            if (oka) cp_async8(d, s + xa);
            if (okb) cp_async8(d + 32, s + xb);
        }
        cp_async_commit();
    };
    double acc = 0.0;
    for (int c0 = 0; c0 < w; c0 += CW) {
        double* tile = sm;
        stage(c0, tile);
        cp_async_wait<0>();
        __syncthreads();
        double* trow = tile + r * TWC;
        // in place: after step i, tile column i (x - CH) is never read again (its subtraction,
        // if any, was at step i - CH + R + 1 <= i), so the mean of x goes there
        // SB steps at a time: their 2 SB inputs are read before any of their means is written
        // (the compiler cannot prove the in-place writes never alias the reads), so one shared-
        // memory latency is paid per SB steps instead of per step
        if (r < rows && c0 >= R + 1 && c0 + CW + R <= w) {
            // interior chunk: every step adds and subtracts, and the window holds 2R+1 values
            const double m = (double)(2 * R + 1);
            for (int i0 = 0; i0 < CW; i0 += SB) {
                double va[SB], vs[SB];
#pragma unroll
                for (int k = 0; k < SB; ++k) {
                    va[k] = trow[i0 + k + R + CH];
                    vs[k] = trow[i0 + k - R - 1 + CH];
                }
#pragma unroll
                for (int k = 0; k < SB; ++k) {
                    acc = dsub(dadd(acc, va[k]), vs[k]);
                    trow[i0 + k] = div_count(acc, m, bw.r_int);
                }
            }
        } else if (r < rows) {
            for (int i0 = 0; i0 < CW; i0 += SB) {
                double va[SB], vs[SB];
#pragma unroll
                for (int k = 0; k < SB; ++k) {
                    va[k] = trow[i0 + k + R + CH];
                    vs[k] = trow[i0 + k - R - 1 + CH];
                }
#pragma unroll
                for (int k = 0; k < SB; ++k) {
                    const int i = i0 + k, x = c0 + i;
                    if (x < w) {
                        if (x == 0) {
                            for (int t = 0; t <= R && t < w; ++t) acc = dadd(acc, trow[t + CH]);
                        } else {
                            if (x + R <= w - 1) acc = dadd(acc, va[k]);
                            if (x - R >= 1) acc = dsub(acc, vs[k]);
                        }
                        trow[i] = bw.mean(acc, x);
                    }
                }
            }
        }
        __syncthreads();  // every row's means are in place
        if (c0 + lane < w)
            for (int rr = wrp; rr < rows; rr += RB / 32) dst[(size_t)rr * w + c0 + lane] = tile[rr * TWC + lane];
        __syncthreads();  // the tile is free for the next chunk
    }
}

// box_mean's column pass fused with the solve (flow.hpp:236-253): a CTA takes CC columns of one
// pair, one warp per plane (lane = column) runs the column's sequential running sum over chunks
// of CR rows, each staged with its CH-row history into a shared tile by cp.async; the five
// planes' means meet in the tile, and all five warps then solve its pixels and write their flow.
constexpr int CC = 32, CR = 16, TR = CR + 2 * CH;  // columns per CTA, rows per chunk, tile rows

__global__ void __launch_bounds__(5 * CC, FROI_K64_CMINB) k64_box_cols_solve(Geom g, int l, int R, int mode,
                                                             const double* __restrict__ rowm,
                                                             const float2* __restrict__ flow_in,
                                                             float2* __restrict__ flow_out) {
    extern __shared__ double sm[];  // two tiles [5][TR][CC]
    const int w = g.lw[l], h = g.lh[l];
    const int x0 = blockIdx.x * CC, p = blockIdx.y;
    const int q = threadIdx.x / CC, lane = threadIdx.x % CC;
    const size_t n0 = (size_t)g.W * g.H;
    const double* col = rowm + (size_t)p * 5 * n0 + x0;
    const size_t fo = (size_t)p * g.lsum + g.loff[l];
    const int cols = min(CC, w - x0);
    FROI_DCHECK(R < CH && cols > 0);
    const BoxWalk bw{h, R, drcp_refined((double)(2 * R + 1))};
    // warp q stages plane q's tile rows (lane = column): no index division per element
    auto stage = [&](int y0, double* tile) {
        if (lane < cols) {
            const double* s = col + q * n0 + lane;
            double* d = tile + q * TR * CC + lane;
            const int jb = max(0, CH - y0), je = min(TR, h - y0 + CH);
            for (int j = jb; j < je; ++j) cp_async8(d + j * CC, s + (size_t)(y0 - CH + j) * w);
        }
        cp_async_commit();
    };
    double acc = 0.0;
    for (int y0 = 0; y0 < h; y0 += CR) {
        double* tile = sm;
        stage(y0, tile);
        cp_async_wait<0>();
        __syncthreads();
        double* tq = tile + q * TR * CC + lane;
        // in place, as in k64_box_rows: the mean of row y0 + i goes to tile row i after step i
        if (lane < cols && y0 >= R + 1 && y0 + CR + R <= h) {  // interior chunk, as in k64_box_rows
            const double m = (double)(2 * R + 1);
            for (int i0 = 0; i0 < CR; i0 += SB) {
                double va[SB], vs[SB];
#pragma unroll
                for (int k = 0; k < SB; ++k) {
                    va[k] = tq[(i0 + k + R + CH) * CC];
                    vs[k] = tq[(i0 + k - R - 1 + CH) * CC];
                }
#pragma unroll
                for (int k = 0; k < SB; ++k) {
                    acc = dsub(dadd(acc, va[k]), vs[k]);
                    tq[(i0 + k) * CC] = div_count(acc, m, bw.r_int);
                }
            }
        } else if (lane < cols) {
            for (int i0 = 0; i0 < CR; i0 += SB) {  // SB steps' inputs first, as in k64_box_rows
                double va[SB], vs[SB];
#pragma unroll
                for (int k = 0; k < SB; ++k) {
                    va[k] = tq[(i0 + k + R + CH) * CC];
                    vs[k] = tq[(i0 + k - R - 1 + CH) * CC];
                }
#pragma unroll
                for (int k = 0; k < SB; ++k) {
                    const int i = i0 + k, y = y0 + i;
                    if (y < h) {
                        if (y == 0) {
                            for (int t = 0; t <= R && t < h; ++t) acc = dadd(acc, tq[(t + CH) * CC]);
                        } else {
                            if (y + R <= h - 1) acc = dadd(acc, va[k]);
                            if (y - R >= 1) acc = dsub(acc, vs[k]);
                        }
                        tq[i * CC] = bw.mean(acc, y);
                    }
                }
            }
        }
        __syncthreads();  // the chunk's five planes of means are in place
        for (int i = q; i < CR; i += 5) {  // warp = row of the chunk, lane = column
            const int c = lane, y = y0 + i, x = x0 + c;
            if (y >= h || c >= cols) continue;
            const double* mm = tile + i * CC + c;
            const double g11 = mm[0], g12 = mm[TR * CC], g22 = mm[2 * TR * CC], h1 = mm[3 * TR * CC],
                         h2 = mm[4 * TR * CC];
            const double det = dsub(dmul(g11, g22), dmul(g12, g12));
            const double frob2 = dadd(dadd(dmul(g11, g11), dmul(dmul(2.0, g12), g12)), dmul(g22, g22));
            const size_t o = fo + (size_t)y * w + x;
            float2 rr;
            if (!(det > dmul(1e-9, frob2))) {
                rr = mode ? flow_in[o] : make_float2(0.f, 0.f);  // keep the prior (zero on the first pass)
            } else {
                const double rd = drcp_refined(det);
                rr.x = __double2float_rn(div_count(dsub(dmul(g22, h1), dmul(g12, h2)), det, rd));
                rr.y = __double2float_rn(div_count(dadd(dmul(-g12, h1), dmul(g11, h2)), det, rd));
            }
            flow_out[o] = rr;
        }
        __syncthreads();  // the tile is free for the next chunk
    }
}

// coarse (level l + 1) -> fine (level l) prior, same buffer
__global__ void __launch_bounds__(kNT) k64_upsample(Geom g, int l, float2* __restrict__ flow) {
    const int p = blockIdx.y;
    const int aw = g.lw[l], ah = g.lh[l], fw = g.lw[l + 1], fh = g.lh[l + 1];
    const long long i = (long long)blockIdx.x * kNT + threadIdx.x;
    if (i >= (long long)aw * ah) return;
    const int y = (int)(i / aw), x = (int)(i - (long long)y * aw);
    const double fx = ddiv((double)aw, (double)fw), fy = ddiv((double)ah, (double)fh);
    const double sy = dsub(ddiv(dadd((double)y, 0.5), fy), 0.5);
    const double sx = dsub(ddiv(dadd((double)x, 0.5), fx), 0.5);
    const float2* c = flow + (size_t)p * g.lsum + g.loff[l + 1];
    Bl b;
    b.setup(fw, fh, sx, sy);
    const float2 c00 = c[b.i00], c01 = c[b.i01], c10 = c[b.i10], c11 = c[b.i11];
    auto interp = [&](double v00, double v01, double v10, double v11) {
        const double top = dadd(dmul(v00, b.ofx), dmul(v01, b.fx));
        const double bot = dadd(dmul(v10, b.ofx), dmul(v11, b.fx));
        return dadd(dmul(top, b.ofy), dmul(bot, b.fy));
    };
    const double u = interp(c00.x, c01.x, c10.x, c11.x), v = interp(c00.y, c01.y, c10.y, c11.y);
    flow[(size_t)p * g.lsum + g.loff[l] + i] = make_float2(__double2float_rn(dmul(u, fx)), __double2float_rn(dmul(v, fy)));
}

inline unsigned blocks(long long n) { return (unsigned)cdiv<long long>(n, kNT); }

constexpr size_t kRowSmem = sizeof(double) * RB * TWC, kColSmem = sizeof(double) * 5 * TR * CC;
static_assert(kRowSmem <= 48 * 1024 && kColSmem <= 48 * 1024, "box tiles fit the default shared memory");

// box_mean's two passes, the column pass fused with the solve
void box_pass(int R, const Geom& g, int l, int mode, int n_pairs, const Flow64Buffers& b, const float2* fin,
              float2* fout, cudaStream_t s) {
    k64_box_rows<<<dim3(cdiv(g.lh[l], RB), 5, n_pairs), RB, kRowSmem, s>>>(g, l, R, b.prod, b.rowm);
    FROI_LAUNCH_CHECK();
    k64_box_cols_solve<<<dim3(cdiv(g.lw[l], CC), n_pairs), 5 * CC, kColSmem, s>>>(g, l, R, mode, b.rowm, fin, fout);
    FROI_LAUNCH_CHECK();
}

// pyramid levels >= 1 and the expansions of every level, for frame slots (info == nullptr) or
// the shifted pair slots
int expand64(const Geom& g, const Flow64Const& C, double* img, double* ex, double* tmp, const PairInfo* info,
             int n_items, cudaStream_t s) {
    int launches = 0;
    for (int l = 0; l < g.L; ++l) {
        if (l > 0) {
            k64_blur_rows<<<dim3(blocks((long long)g.lw[l - 1] * g.lh[l - 1]), n_items), kNT, 0, s>>>(g, C, l - 1, img,
                                                                                                   info, tmp);
            FROI_LAUNCH_CHECK();
            k64_blur_cols_resize<<<dim3(blocks((long long)g.lw[l] * g.lh[l]), n_items), kNT, 0, s>>>(g, C, l - 1, tmp,
                                                                                                 info, img);
            FROI_LAUNCH_CHECK();
            launches += 2;
        }
        k64_polyexp<<<dim3(cdiv(g.lw[l], PEX), cdiv(g.lh[l], PEY), n_items), kNT, 0, s>>>(g, C, l, img, info, ex);
        FROI_LAUNCH_CHECK();
        ++launches;
    }
    return launches;
}

}  // namespace

int launch_expand_frames64(const Geom& g, const Flow64Const& C, const Flow64Buffers& b, const void* den,
                           int n_slots, cudaStream_t s) {
    if (n_slots <= 0) return 0;
    const double inv = 1.0 / (double)g.maxval;
    const dim3 grid(blocks((long long)g.W * g.H), n_slots);
    if (g.sample_bytes == 1) k64_norm0<uint8_t><<<grid, kNT, 0, s>>>(g, inv, (const uint8_t*)den, b.img_f);
    else k64_norm0<uint16_t><<<grid, kNT, 0, s>>>(g, inv, (const uint16_t*)den, b.img_f);
    FROI_LAUNCH_CHECK();
    return 1 + expand64(g, C, b.img_f, b.ex_f, b.tmp_f, nullptr, n_slots, s);
}

int launch_expand_shifted64(const Geom& g, const Flow64Const& C, const Flow64Buffers& b, const void* den,
                            const int* d_next, const PairInfo* d_info, int n_pairs, cudaStream_t s) {
    if (n_pairs <= 0) return 0;
    const double inv = 1.0 / (double)g.maxval;
    const dim3 grid(blocks((long long)g.W * g.H), n_pairs);
    if (g.sample_bytes == 1)
        k64_norm0_shifted<uint8_t><<<grid, kNT, 0, s>>>(g, inv, (const uint8_t*)den, d_next, d_info, b.img_p);
    else
        k64_norm0_shifted<uint16_t><<<grid, kNT, 0, s>>>(g, inv, (const uint16_t*)den, d_next, d_info, b.img_p);
    FROI_LAUNCH_CHECK();
    return 1 + expand64(g, C, b.img_p, b.ex_p, b.tmp_p, d_info, n_pairs, s);
}

int launch_flow64(const Geom& g, const DevParams& P, const Flow64Buffers& b, const int* d_prev, const int* d_next,
                  const PairInfo* d_info, int n_pairs, cudaStream_t s, int* cur_out) {
    if (n_pairs <= 0) return 0;
    if (P.window_radius > CH - 1) throw Error(1, "exact flow: window_size > 15 is not supported");
    const int R = P.window_radius;
    float2* buf[2] = {b.flow0, b.flow1};
    int cur = 0, launches = 0;
    for (int l = g.L - 1; l >= 0; --l) {
        const long long n = (long long)g.lw[l] * g.lh[l];
        for (int it = 0; it < P.iterations; ++it) {
            const int mode = (it == 0 && l == g.L - 1) ? 0 : 1;
            if (it == 0 && l < g.L - 1) {
                k64_upsample<<<dim3(blocks(n), n_pairs), kNT, 0, s>>>(g, l, buf[cur]);
                FROI_LAUNCH_CHECK();
                ++launches;
            }
            k64_products<<<dim3(blocks(n), n_pairs), kNT, 0, s>>>(g, l, mode, b.ex_f, b.ex_p, d_prev, d_next, d_info,
                                                                 buf[cur], b.prod);
            FROI_LAUNCH_CHECK();
            box_pass(R, g, l, mode, n_pairs, b, buf[cur], buf[1 - cur], s);
            launches += 3;
            cur = 1 - cur;
        }
    }
    *cur_out = cur;
    return launches;
}

}  // namespace froi
