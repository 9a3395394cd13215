// k_flow.cu — pyramid, polynomial expansion and the fused flow iteration
// (flow.hpp:118-345): fp32 storage and arithmetic, exact fp32 warp coordinates, compensated
// fp32 determinant in the 2x2 solve.
//
//   k_pyr_down   7-tap Gaussian (sigma 1, rows then columns, edge-replicated) fused with the
//                bilinear resample to floor(w*scale) x floor(h*scale)            (flow.hpp:259-298)
//   k_polyexp    5-tap separable Gaussian-weighted quadratic fit per pixel; writes the four
//                planes the warp gathers together as one float4 {a11,a12,a22,bx} plus {by};
//                the constant term c is only produced by the debug tap        (flow.hpp:118-153)
//   k_flow_iter  one launch per (level, iteration); one CTA (512 threads, 2 per SM) per strip of
//                nr vertically stacked 64x32 output tiles of one pair: phase 1 builds the five
//                normal-equation products G over the rows each tile adds (tile + 7 px halo; the
//                14 overlap rows stay in a 48-row shared ring), with the prior from the same level
//                (or upsampled by k_upsample) and the bilinear warp of the next frame's planes;
//                phases 2/3 take the 15x15 clipped box sums in place (vertical then horizontal
//                running sums); phase 4 solves the 2x2 system on the window sums in fp32 with a
//                compensated determinant and the reference's singularity test (flow.hpp:204-255)
//
// Level-0 images are read straight from the denoised u8/u16 frames (normalised on the fly, with
// the registration shift applied as a clamped gather, registration.hpp:100-107), so the fp32
// level-0 image is never materialised.
#include "kernels.cuh"

#include <algorithm>
#include <cstdlib>
#include <type_traits>

namespace froi {
namespace {

// ------------------------------------------------------------------ sources
template <typename T>
struct FrameSrc {  // normalize_frame(apply_shift(den, s)) at level 0
    const T* f;
    int W, H, dx, dy;
    double inv;        // 1.0 / maxval
    const float* lut;  // 8-bit frames: the 256 values (float)(v * inv), global (L1-resident)
    __device__ __forceinline__ float at(int x, int y) const {
        const int sx = clampi(clampi(x, 0, W - 1) + dx, 0, W - 1);
        const int sy = clampi(clampi(y, 0, H - 1) + dy, 0, H - 1);
        const int v = f[sy * W + sx];
        return sizeof(T) == 1 ? __ldg(lut + v) : (float)((double)v * inv);
    }
    // [x0, x1) x [y0, y1) needs no clamping (before or after the shift)
    __device__ __forceinline__ bool inside(int x0, int y0, int x1, int y1) const {
        return x0 >= 0 && y0 >= 0 && x1 <= W && y1 <= H && x0 + dx >= 0 && y0 + dy >= 0 && x1 + dx <= W &&
               y1 + dy <= H;
    }
    __device__ __forceinline__ const T* base(int x0, int y0) const { return f + (y0 + dy) * W + x0 + dx; }
    __device__ __forceinline__ float conv(T v) const {
        return sizeof(T) == 1 ? __ldg(lut + v) : (float)((double)v * inv);
    }
};

struct ImageSrc {
    const float* f;
    int W, H;
    __device__ __forceinline__ float at(int x, int y) const {
        return f[(size_t)clampi(y, 0, H - 1) * W + clampi(x, 0, W - 1)];
    }
    __device__ __forceinline__ bool inside(int x0, int y0, int x1, int y1) const {
        return x0 >= 0 && y0 >= 0 && x1 <= W && y1 <= H;
    }
    __device__ __forceinline__ const float* base(int x0, int y0) const { return f + (size_t)y0 * W + x0; }
    __device__ __forceinline__ float conv(float v) const { return v; }
};

// Stages an edge-clamped source block into shared memory with U elements per thread in flight:
// all U source reads (for 8-bit frames a byte load then its table lookup) are issued before any
// store, instead of one dependent load pair per element.
template <int NT, int U, typename At>
__device__ __forceinline__ void stage_block(float* dst, int n, int sw, At at) {
    for (int i0 = threadIdx.x; i0 < n; i0 += U * NT) {
        float v[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const int i = i0 + k * NT;
            if (i < n) {
                const int yy = i / sw, xx = i - yy * sw;
                v[k] = at(xx, yy);
            }
        }
#pragma unroll
        for (int k = 0; k < U; ++k)
            if (i0 + k * NT < n) dst[i0 + k * NT] = v[k];
    }
}

// The bw x bh source block at (bx0, by0), minus `sub`, into shared memory: without any clamping
// when the block lies inside the image.
template <int NT, int U, typename Src>
__device__ __forceinline__ void stage_src(const Src& src, float* dst, int bx0, int by0, int bw, int bh,
                                          float sub) {
    if (src.inside(bx0, by0, bx0 + bw, by0 + bh)) {
        const auto* b0 = src.base(bx0, by0);
        const int W = src.W;
        stage_block<NT, U>(dst, bw * bh, bw, [&](int xx, int yy) { return src.conv(b0[yy * W + xx]) - sub; });
    } else {
        stage_block<NT, U>(dst, bw * bh, bw, [&](int xx, int yy) { return src.at(bx0 + xx, by0 + yy) - sub; });
    }
}

// ------------------------------------------------------------------ polynomial expansion
constexpr int PX = 32, PY = 32, PNT = 256;

// RC > 0: compile-time radius (unrolled taps, weights as constant-bank operands); 0: runtime.
template <typename Src, bool kDebug, int RC = 0>
__device__ __forceinline__ void polyexp_tile(const Src& src, int w, int h, int r_rt,
                                             const DevParams& P, float4* outA, float* outB,
                                             float* dbg_planes, float* smem) {
    const int r = RC > 0 ? RC : r_rt;
    const int x0 = blockIdx.x * PX, y0 = blockIdx.y * PY;
    const int sw = PX + 2 * r, sh = PY + 2 * r;
    float* s_in = smem;               // sh * sw
    float* s_r = s_in + sh * sw;      // 3 * sh * PX
    const int tid = threadIdx.x;
    // constant offset: the fit of A and b is invariant to it and it removes cancellation
    const float c0 = src.at(x0, y0);
    stage_src<PNT, 3>(src, s_in, x0 - r, y0 - r, sw, sh, c0);
    __syncthreads();
    if (RC == 2 && !kDebug) {
        // radius 2: same arithmetic per output, loads shared between neighbours -- row pass two
        // adjacent columns from 6 loads, column pass two adjacent rows from 18 loads
        constexpr int SW = PX + 4, SH = PY + 4;
        float g0[5], g1[5], g2[5];
#pragma unroll
        for (int t = 0; t < 5; ++t) {
            g0[t] = P.g0[t];
            g1[t] = P.g1[t];
            g2[t] = P.g2[t];
        }
        for (int i = tid; i < SH * (PX / 2); i += PNT) {
            const int yy = i / (PX / 2), xx = 2 * (i - yy * (PX / 2));
            const float* row = s_in + yy * SW + xx;
            float v[6];
#pragma unroll
            for (int t = 0; t < 6; ++t) v[t] = row[t];
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                // (a0, a1) as one packed FFMA2 per tap: the same two roundings as two FFMAs
                float a0 = 0.f, a1 = 0.f, a2 = 0.f;
#pragma unroll
                for (int t = 0; t < 5; ++t) {
                    fma2(a0, a1, g0[t], g1[t], v[t + k], v[t + k], a0, a1);
                    a2 = fmaf(g2[t], v[t + k], a2);
                }
                s_r[yy * PX + xx + k] = a0;
                s_r[SH * PX + yy * PX + xx + k] = a1;
                s_r[2 * SH * PX + yy * PX + xx + k] = a2;
            }
        }
        __syncthreads();
        const float inv_m20 = P.poly_moments[0], inv_m22 = P.poly_moments[1];
        const float i01 = P.poly_moments[3], i11 = P.poly_moments[4], i12 = P.poly_moments[5];
        const int xx = tid & (PX - 1);
#pragma unroll 1
        for (int yb = (tid / PX) * 2; yb < PY; yb += 2 * (PNT / PX)) {
        float q0[6], q1[6], q2[6];
#pragma unroll
        for (int t = 0; t < 6; ++t) {
            q0[t] = s_r[(yb + t) * PX + xx];
            q1[t] = s_r[SH * PX + (yb + t) * PX + xx];
            q2[t] = s_r[2 * SH * PX + (yb + t) * PX + xx];
        }
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const int x = x0 + xx, y = y0 + yb + k;
            if (x >= w || y >= h) continue;
            float s1 = 0.f, sx = 0.f, sy = 0.f, sxx = 0.f, syy = 0.f, sxy = 0.f;
#pragma unroll
            for (int t = 0; t < 5; ++t) {  // packed pairs (FFMA2): same roundings as six FFMAs
                fma2(s1, sx, g0[t], g0[t], q0[t + k], q1[t + k], s1, sx);
                fma2(sy, sxy, g1[t], g1[t], q0[t + k], q1[t + k], sy, sxy);
                sxx = fmaf(g0[t], q2[t + k], sxx);
                syy = fmaf(g2[t], q0[t + k], syy);
            }
            const float bx = sx * inv_m20, by = sy * inv_m20;
            const float a12 = 0.5f * sxy * inv_m22;
            const float a11 = i01 * s1 + i11 * sxx + i12 * syy;
            const float a22 = i01 * s1 + i12 * sxx + i11 * syy;
            const int o = y * w + x;
            outA[o] = make_float4(a11, a12, a22, bx);
            outB[o] = by;
        }
        }
        return;
    }
    // correlate_rows with g0, g1, g2 (flow.hpp:55-70)
    for (int i = tid; i < sh * PX; i += PNT) {
        const int yy = i / PX, xx = i - yy * PX;
        const float* row = s_in + yy * sw + xx;
        float a0 = 0.f, a1 = 0.f, a2 = 0.f;
#pragma unroll
        for (int t = 0; t <= 2 * r; ++t) {
            const float v = row[t];
            a0 += P.g0[t] * v;
            a1 += P.g1[t] * v;
            a2 += P.g2[t] * v;
        }
        s_r[i] = a0;
        s_r[sh * PX + i] = a1;
        s_r[2 * sh * PX + i] = a2;
    }
    __syncthreads();
    // correlate_cols and the moment combination (flow.hpp:136-151)
    for (int i = tid; i < PY * PX; i += PNT) {
        const int yy = i / PX, xx = i - yy * PX;
        const int x = x0 + xx, y = y0 + yy;
        if (x >= w || y >= h) continue;
        float s1 = 0.f, sx = 0.f, sy = 0.f, sxx = 0.f, syy = 0.f, sxy = 0.f;
#pragma unroll
        for (int t = 0; t <= 2 * r; ++t) {
            const float r0 = s_r[(yy + t) * PX + xx];
            const float r1 = s_r[sh * PX + (yy + t) * PX + xx];
            const float r2 = s_r[2 * sh * PX + (yy + t) * PX + xx];
            s1 += P.g0[t] * r0;
            sx += P.g0[t] * r1;
            sy += P.g1[t] * r0;
            sxx += P.g0[t] * r2;
            syy += P.g2[t] * r0;
            sxy += P.g1[t] * r1;
        }
        const float inv_m20 = P.poly_moments[0], inv_m22 = P.poly_moments[1];
        const float i00 = P.poly_moments[2], i01 = P.poly_moments[3];
        const float i11 = P.poly_moments[4], i12 = P.poly_moments[5];
        const float bx = sx * inv_m20, by = sy * inv_m20;
        const float a12 = 0.5f * sxy * inv_m22;
        const float a11 = i01 * s1 + i11 * sxx + i12 * syy;
        const float a22 = i01 * s1 + i12 * sxx + i11 * syy;
        const size_t o = (size_t)y * w + x;
        if (kDebug) {
            const size_t n = (size_t)w * h;
            dbg_planes[o] = i00 * s1 + i01 * (sxx + syy) + c0;
            dbg_planes[n + o] = bx;
            dbg_planes[2 * n + o] = by;
            dbg_planes[3 * n + o] = a11;
            dbg_planes[4 * n + o] = a12;
            dbg_planes[5 * n + o] = a22;
        } else {
            outA[o] = make_float4(a11, a12, a22, bx);
            outB[o] = by;
        }
    }
}

// Frame slots: level-0 expansion from the denoised frame (unshifted).
template <typename T, int RC>
__global__ void __launch_bounds__(PNT) k_polyexp_frame(Geom g, DevParams P, const T* den,
                                                       float4* exA, float* exB) {
    extern __shared__ float smem_f[];
    const int slot = blockIdx.z;
    const double inv = 1.0 / g.maxval;
    FrameSrc<T> src{den + (size_t)slot * g.W * g.H, g.W, g.H, 0, 0, inv, P.norm_lut};
    polyexp_tile<FrameSrc<T>, false, RC>(src, g.W, g.H, P.poly_radius, P, exA + (size_t)slot * g.lsum,
                                         exB + (size_t)slot * g.lsum, nullptr, smem_f);
}

// Pair slots: level-0 expansion of apply_shift(den[t], s) when s != 0.
template <typename T, int RC>
__global__ void __launch_bounds__(PNT) k_polyexp_shifted(Geom g, DevParams P, const T* den,
                                                         const int* next, const PairInfo* info,
                                                         float4* exA, float* exB) {
    extern __shared__ float smem_f[];
    const int p = blockIdx.z;
    const PairInfo I = info[p];
    if (!I.shifted) return;
    const double inv = 1.0 / g.maxval;
    FrameSrc<T> src{den + (size_t)next[p] * g.W * g.H, g.W, g.H, I.dx, I.dy, inv, P.norm_lut};
    polyexp_tile<FrameSrc<T>, false, RC>(src, g.W, g.H, P.poly_radius, P, exA + (size_t)p * g.lsum,
                                         exB + (size_t)p * g.lsum, nullptr, smem_f);
}

// Levels >= 1 from a float pyramid image (frame slots if info == nullptr, else pair slots).
template <int RC>
__global__ void __launch_bounds__(PNT) k_polyexp_level(Geom g, DevParams P, int l,
                                                       const float* pyr, long long pyr_stride,
                                                       const PairInfo* info, float4* exA,
                                                       float* exB) {
    extern __shared__ float smem_f[];
    const int z = blockIdx.z;
    if (info && !info[z].shifted) return;
    const long long poff = g.loff[l] - g.loff[1];
    ImageSrc src{pyr + (size_t)z * pyr_stride + poff, g.lw[l], g.lh[l]};
    polyexp_tile<ImageSrc, false, RC>(src, g.lw[l], g.lh[l], P.poly_radius, P,
                                  exA + (size_t)z * g.lsum + g.loff[l],
                                  exB + (size_t)z * g.lsum + g.loff[l], nullptr, smem_f);
}

__global__ void __launch_bounds__(PNT) k_polyexp_debug(Geom g, DevParams P, const float* img,
                                                       float* planes) {
    extern __shared__ float smem_f[];
    ImageSrc src{img, g.W, g.H};
    polyexp_tile<ImageSrc, true>(src, g.W, g.H, P.poly_radius, P, nullptr, nullptr, planes, smem_f);
}

// ------------------------------------------------------------------ pyramid
constexpr int QX = 32, QY = 8, QNT = 256;

__device__ __forceinline__ void bl_index(double s, int n, int& i0, int& i1, double& f) {
    // bilinear() index rule (flow.hpp:157-168)
    s = s < 0.0 ? 0.0 : (s > (double)(n - 1) ? (double)(n - 1) : s);
    const int lim = n - 2 >= 0 ? n - 2 : 0;
    i0 = min((int)s, lim);
    i1 = min(i0 + 1, n - 1);
    f = s - i0;
}

template <typename Src>
__device__ __forceinline__ void pyr_tile(const Src& src, int w, int h, int tw, int th,
                                         const float* kblur, float* out, float* smem, int rwmax,
                                         int rhmax) {
    const int ox0 = blockIdx.x * QX, oy0 = blockIdx.y * QY;
    const double sx = (double)w / tw, sy = (double)h / th;
    int xa, xb, ya, yb, t0, t1;
    double f;
    bl_index((ox0 + 0.5) * sx - 0.5, w, xa, t1, f);
    bl_index((min(ox0 + QX - 1, tw - 1) + 0.5) * sx - 0.5, w, t0, xb, f);
    bl_index((oy0 + 0.5) * sy - 0.5, h, ya, t1, f);
    bl_index((min(oy0 + QY - 1, th - 1) + 0.5) * sy - 0.5, h, t0, yb, f);
    const int RW = xb - xa + 1, RH = yb - ya + 1;
    if (RW > rwmax || RH > rhmax) __trap();
    const int iw = RW + 6, ih = RH + 6;
    float* s_in = smem;             // ih * iw
    float* s_rb = s_in + ih * iw;   // ih * RW
    float* s_bl = s_rb + ih * RW;   // RH * RW
    // bilinear() taps of this tile's output columns and rows, computed once (same fp64 rule)
    __shared__ int s_ix0[QX], s_ix1[QX], s_iy0[QY], s_iy1[QY];
    __shared__ float s_fx[QX], s_fy[QY];
    if (threadIdx.x < QX) {
        double fd;
        bl_index((ox0 + threadIdx.x + 0.5) * sx - 0.5, w, s_ix0[threadIdx.x], s_ix1[threadIdx.x], fd);
        s_fx[threadIdx.x] = (float)fd;
    } else if (threadIdx.x < QX + QY) {
        const int t = threadIdx.x - QX;
        double fd;
        bl_index((oy0 + t + 0.5) * sy - 0.5, h, s_iy0[t], s_iy1[t], fd);
        s_fy[t] = (float)fd;
    }
    for (int i = threadIdx.x; i < ih * iw; i += QNT) {
        const int yy = i / iw, xx = i - yy * iw;
        s_in[i] = src.at(xa - 3 + xx, ya - 3 + yy);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < ih * RW; i += QNT) {
        const int yy = i / RW, xx = i - yy * RW;
        const float* row = s_in + yy * iw + xx;
        float acc = 0.f;
        for (int t = 0; t < 7; ++t) acc += kblur[t] * row[t];
        s_rb[i] = acc;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < RH * RW; i += QNT) {
        const int yy = i / RW, xx = i - yy * RW;
        float acc = 0.f;
        for (int t = 0; t < 7; ++t) acc += kblur[t] * s_rb[(yy + t) * RW + xx];
        s_bl[i] = acc;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < QX * QY; i += QNT) {
        const int yy = i / QX, xx = i - yy * QX;
        const int x = ox0 + xx, y = oy0 + yy;
        if (x >= tw || y >= th) continue;
        const int x0 = s_ix0[xx], x1 = s_ix1[xx], y0 = s_iy0[yy], y1 = s_iy1[yy];
        const float* r0 = s_bl + (y0 - ya) * RW;
        const float* r1 = s_bl + (y1 - ya) * RW;
        const float ffx = s_fx[xx], ffy = s_fy[yy];
        const float top = r0[x0 - xa] * (1.f - ffx) + r0[x1 - xa] * ffx;
        const float bot = r1[x0 - xa] * (1.f - ffx) + r1[x1 - xa] * ffx;
        out[(size_t)y * tw + x] = top * (1.f - ffy) + bot * ffy;
    }
}

// Exact 2:1 levels (w == 2 tw, h == 2 th; the default pyramid): bilinear() then always reads
// blurred pixels (2x, 2x+1) x (2y, 2y+1) with fraction 0.5, so the tile is fixed: a 32x16 output
// tile blurs a 64x32 block from a 70x38 input block.  Same blur order and resample expression as
// pyr_tile; loops and divisions are compile-time, the column blur walks 8 rows per thread.
constexpr int Q2X = 32, Q2Y = 16, Q2W = 2 * Q2X + 6, Q2H = 2 * Q2Y + 6;

// Even sizes: the 0.5 bilinear resample of the blurred image is the mean of each 2x2 block
// (SURVEY.md §8 a6), so blur + resample is one separable 8-tap filter c = (k * [1, 1]) / 2
// evaluated at stride 2: only the kept samples are computed (half the row-pass work, a quarter
// of the column-pass work of blurring every pixel first).  fp32, like the rest of the pyramid.
template <typename Src>
__device__ __forceinline__ void pyr2_tile(const Src& src, int tw, int th, const float* kblur,
                                          float* out, float* smem) {
    float* s_in = smem;              // Q2H x Q2W input (edge-clamped by the source)
    float* s_r = s_in + Q2H * Q2W;   // Q2H x Q2X row-filtered, stride 2
    const int ox0 = blockIdx.x * Q2X, oy0 = blockIdx.y * Q2Y;
    const int ix0 = 2 * ox0 - 3, iy0 = 2 * oy0 - 3;
    const int tid = threadIdx.x;
    stage_src<QNT, 4>(src, s_in, ix0, iy0, Q2W, Q2H, 0.f);
    float c[8];
    c[0] = 0.5f * kblur[0];
#pragma unroll
    for (int u = 1; u < 7; ++u) c[u] = 0.5f * (kblur[u - 1] + kblur[u]);
    c[7] = 0.5f * kblur[6];
    __syncthreads();
    // rows: output column ox of input row yy from 8 consecutive inputs (four 8-byte loads)
    for (int i = tid; i < Q2H * Q2X; i += QNT) {
        const int yy = i / Q2X, ox = i - yy * Q2X;
        const float2* row = (const float2*)(s_in + yy * Q2W + 2 * ox);
        float acc = 0.f;
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            const float2 v = row[m];
            acc = fmaf(c[2 * m], v.x, acc);
            acc = fmaf(c[2 * m + 1], v.y, acc);
        }
        s_r[i] = acc;
    }
    __syncthreads();
    // columns: two vertically adjacent outputs per thread share 6 of their 8 input rows
    {
        const int xx = tid & (Q2X - 1), yy = 2 * (tid >> 5);
        const int x = ox0 + xx;
        float v[10];
#pragma unroll
        for (int t = 0; t < 10; ++t) v[t] = s_r[(2 * yy + t) * Q2X + xx];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int y = oy0 + yy + r;
            float acc = 0.f;
#pragma unroll
            for (int t = 0; t < 8; ++t) acc = fmaf(c[t], v[2 * r + t], acc);
            if (x < tw && y < th) out[(size_t)y * tw + x] = acc;
        }
    }
}
constexpr size_t pyr2_smem() { return sizeof(float) * (Q2H * Q2W + Q2H * Q2X); }

template <typename T, bool HALF>
__global__ void __launch_bounds__(QNT) k_pyr0_frame(Geom g, DevParams P, const T* den, float* pyr,
                                                    int rwmax, int rhmax) {
    extern __shared__ float smem_f[];
    const int slot = blockIdx.z;
    const double inv = 1.0 / g.maxval;
    FrameSrc<T> src{den + (size_t)slot * g.W * g.H, g.W, g.H, 0, 0, inv, P.norm_lut};
    float* dst = pyr + (size_t)slot * (g.lsum - g.loff[1]);
    if (HALF) pyr2_tile(src, g.lw[1], g.lh[1], P.blur, dst, smem_f);
    else pyr_tile(src, g.W, g.H, g.lw[1], g.lh[1], P.blur, dst, smem_f, rwmax, rhmax);
}

template <typename T, bool HALF>
__global__ void __launch_bounds__(QNT) k_pyr0_shifted(Geom g, DevParams P, const T* den,
                                                      const int* next, const PairInfo* info,
                                                      float* pyr, int rwmax, int rhmax) {
    extern __shared__ float smem_f[];
    const int p = blockIdx.z;
    const PairInfo I = info[p];
    if (!I.shifted) return;
    const double inv = 1.0 / g.maxval;
    FrameSrc<T> src{den + (size_t)next[p] * g.W * g.H, g.W, g.H, I.dx, I.dy, inv, P.norm_lut};
    float* dst = pyr + (size_t)p * (g.lsum - g.loff[1]);
    if (HALF) pyr2_tile(src, g.lw[1], g.lh[1], P.blur, dst, smem_f);
    else pyr_tile(src, g.W, g.H, g.lw[1], g.lh[1], P.blur, dst, smem_f, rwmax, rhmax);
}

template <bool HALF>
__global__ void __launch_bounds__(QNT) k_pyr_level(Geom g, DevParams P, int l, float* pyr,
                                                   const PairInfo* info, int rwmax, int rhmax) {
    // level l -> l+1, l >= 1
    extern __shared__ float smem_f[];
    const int z = blockIdx.z;
    if (info && !info[z].shifted) return;
    float* base = pyr + (size_t)z * (g.lsum - g.loff[1]);
    ImageSrc src{base + (g.loff[l] - g.loff[1]), g.lw[l], g.lh[l]};
    float* dst = base + (g.loff[l + 1] - g.loff[1]);
    if (HALF) pyr2_tile(src, g.lw[l + 1], g.lh[l + 1], P.blur, dst, smem_f);
    else pyr_tile(src, g.lw[l], g.lh[l], g.lw[l + 1], g.lh[l + 1], P.blur, dst, smem_f, rwmax, rhmax);
}

// ------------------------------------------------------------------ flow iteration
constexpr int FX = 64, FY = 32, FNT = 512;
// timing diagnostics only (the last two give wrong results): no L1 prefetch of the
// prior / no box sums / gathers at the pixel itself
#ifndef FROI_FLOW_NOPF
#define FROI_FLOW_NOPF 0
#endif
#ifndef FROI_DIAG_NOBOX
#define FROI_DIAG_NOBOX 0
#endif
#ifndef FROI_DIAG_ZEROFLOW
#define FROI_DIAG_ZEROFLOW 0
#endif

struct IterArgs {
    int l;        // level
    int mode;     // 0 zero prior (coarsest level, first iteration), 1 prior = flow_in (same level)
    const float2* flow_in;
    float2* flow_out;
};

// floor(d) as (float, int) without the XU pipe: adding and removing 1.5*2^23 rounds to the
// nearest integer (exact for |d| < 2^22), a compare turns it into floor.
__device__ __forceinline__ float floor_split(float d, int& i) {
    const float M = 12582912.0f;
    d = fminf(fmaxf(d, -4194304.0f), 4194304.0f);
    float r = __fsub_rn(__fadd_rn(d, M), M);
    r = r > d ? r - 1.0f : r;
    i = __float_as_int(__fadd_rn(r, M)) - 0x4B400000;
    return r;
}

// bilinear() index rule (flow.hpp:157-168) for the coordinate i + d, computed exactly in fp32:
// the integer part goes to the index, d - floor(d) is exact, so (x0, fx) equal the reference's.
__device__ __forceinline__ void bl_split(int i, float d, int n, int& i0, float& f) {
    int fi;
    const float fl = floor_split(d, fi);
    i0 = i + fi;
    f = d - fl;
    if (i0 < 0) {
        i0 = 0;
        f = 0.f;
    } else if (i0 >= n - 1) {
        i0 = n - 2;
        f = 1.f;
    }
}

// One fine-pixel value of the coarse-to-fine prior (flow.hpp:318-337) in fp32, with explicit
// round-to-nearest operations in the reference's bilinear order (top row, bottom row, blend,
// scale): the same bits whichever kernel (k_upsample / k_upsample2) computes it.
__device__ __forceinline__ float up_ch(float a, float b, float d, float e, float ax, float ay, float s) {
    const float oax = __fsub_rn(1.f, ax), oay = __fsub_rn(1.f, ay);
    const float top = __fadd_rn(__fmul_rn(a, oax), __fmul_rn(b, ax));
    const float bot = __fadd_rn(__fmul_rn(d, oax), __fmul_rn(e, ax));
    return __fmul_rn(__fadd_rn(__fmul_rn(top, oay), __fmul_rn(bot, ay)), s);
}
__device__ __forceinline__ float2 up_px(float2 a, float2 b, float2 d, float2 e, float ax, float ay, float fx,
                                        float fy) {
    return make_float2(up_ch(a.x, b.x, d.x, e.x, ax, ay, fx), up_ch(a.y, b.y, d.y, e.y, ax, ay, fy));
}

// Coarse-to-fine upsampling of the prior (flow.hpp:318-337), fp32: one thread per fine pixel,
// run once per level before its first iteration.  rfx = 1/fx (exact for the default 0.5 scale).
__global__ void __launch_bounds__(256) k_upsample(Geom g, int l, const float2* __restrict__ coarse,
                                                  float2* __restrict__ fine, float fx, float fy,
                                                  float rfx, float rfy) {
    // 32 x 32 fine pixels per CTA, four rows per thread with all 16 coarse loads issued first
    constexpr int NY = 4;
    const int p = blockIdx.z;
    const int w = g.lw[l], h = g.lh[l], cw = g.lw[l + 1], ch = g.lh[l + 1];
    const int x = blockIdx.x * 32 + (threadIdx.x & 31);
    const float2* c = coarse + (size_t)p * g.lsum + g.loff[l + 1];
    float2* f = fine + (size_t)p * g.lsum + g.loff[l];
    const float sx = (x + 0.5f) * rfx - 0.5f;
    int x0;
    float ax;
    bl_split(0, sx, cw, x0, ax);
    float2 q[NY][4];
    float ay[NY];
#pragma unroll
    for (int k = 0; k < NY; ++k) {
        const int y = min(blockIdx.y * 32 + (threadIdx.x >> 5) + 8 * k, h - 1);
        const float sy = (y + 0.5f) * rfy - 0.5f;
        int y0;
        bl_split(0, sy, ch, y0, ay[k]);
        const float2* r0 = c + y0 * cw + x0;
        q[k][0] = __ldg(r0);
        q[k][1] = __ldg(r0 + 1);
        q[k][2] = __ldg(r0 + cw);
        q[k][3] = __ldg(r0 + cw + 1);
    }
#pragma unroll
    for (int k = 0; k < NY; ++k) {
        const int y = blockIdx.y * 32 + (threadIdx.x >> 5) + 8 * k;
        if (x >= w || y >= h) continue;
        f[y * w + x] = up_px(q[k][0], q[k][1], q[k][2], q[k][3], ax, ay[k], fx, fy);
    }
}

// The exact 2:1 case of k_upsample (fine size = 2 x coarse, the default pyramid): one thread per
// coarse pixel (i, j) writes the fine 2x2 block (2i..2i+1, 2j..2j+1) as two 16-byte stores.  Away
// from the border the bilinear corners are always coarse (i-1..i+1, j-1..j+1) with weights 0.75 /
// 0.25, so nine loads serve four outputs; border blocks take k_upsample's per-pixel index rule.
// Every output is up_px on the same operands as in k_upsample, so the two kernels agree bit for bit
// (FROI_UPSAMPLE2=0 in the environment selects k_upsample everywhere; tests compare the two).
__global__ void __launch_bounds__(256) k_upsample2(Geom g, int l, const float2* __restrict__ coarse,
                                                   float2* __restrict__ fine, float fx, float fy) {
    const int p = blockIdx.z;
    const int w = g.lw[l], cw = g.lw[l + 1], ch = g.lh[l + 1];
    const int i = blockIdx.x * 32 + (threadIdx.x & 31), j = blockIdx.y * 8 + (threadIdx.x >> 5);
    if (i >= cw || j >= ch) return;
    const float2* c = coarse + (size_t)p * g.lsum + g.loff[l + 1];
    float2* f = fine + (size_t)p * g.lsum + g.loff[l];
    float2 o[2][2];
    if (i >= 1 && i <= cw - 2 && j >= 1 && j <= ch - 2) {
        float2 v[3][3];
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int q = 0; q < 3; ++q) v[r][q] = __ldg(c + (j - 1 + r) * cw + (i - 1 + q));
#pragma unroll
        for (int yy = 0; yy < 2; ++yy)
#pragma unroll
            for (int xx = 0; xx < 2; ++xx)
                o[yy][xx] = up_px(v[yy][xx], v[yy][xx + 1], v[yy + 1][xx], v[yy + 1][xx + 1], xx ? 0.25f : 0.75f,
                                  yy ? 0.25f : 0.75f, fx, fy);
    } else {
#pragma unroll
        for (int yy = 0; yy < 2; ++yy) {
            const int y = 2 * j + yy;
            int y0;
            float ay;
            bl_split(0, (y + 0.5f) * 0.5f - 0.5f, ch, y0, ay);
#pragma unroll
            for (int xx = 0; xx < 2; ++xx) {
                const int x = 2 * i + xx;
                int x0;
                float ax;
                bl_split(0, (x + 0.5f) * 0.5f - 0.5f, cw, x0, ax);
                const float2* r0 = c + y0 * cw + x0;
                o[yy][xx] = up_px(__ldg(r0), __ldg(r0 + 1), __ldg(r0 + cw), __ldg(r0 + cw + 1), ax, ay, fx, fy);
            }
        }
    }
#pragma unroll
    for (int yy = 0; yy < 2; ++yy)
        *(float4*)(f + (size_t)(2 * j + yy) * w + 2 * i) = make_float4(o[yy][0].x, o[yy][0].y, o[yy][1].x, o[yy][1].y);
}

// Normal-equation products G of one pixel (flow.hpp:212-232).
struct GTerms {
    float g11, g12, g22, h1, h2;
};

// Streaming reads (the previous frame's coefficients at the pixel itself: read once per tile)
// bypass L1 allocation, leaving its capacity to the bilinear gathers that do reuse lines.
__device__ __forceinline__ float4 ld_stream(const float4* p) {
    float4 v;
    asm("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
        : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
        : "l"(p));
    return v;
}
__device__ __forceinline__ float ld_stream(const float* p) {
    float v;
    asm("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
}

// Gathered operands of one pixel's normal-equation products.
struct GLoad {
    float4 q00, q01, q10, q11, pa;
    float b00, b01, b10, b11, pb, fx, fy;
};

// Issue every gather of one pixel (no branches, so the loads of several pixels overlap).
__device__ __forceinline__ void g_load(GLoad& o, const float4* __restrict__ pA,
                                       const float* __restrict__ pB, const float4* __restrict__ nA,
                                       const float* __restrict__ nB, int w, int h, int gx, int gy,
                                       float du, float dv) {
    int xa, ya;
    bl_split(gx, du, w, xa, o.fx);
    bl_split(gy, dv, h, ya, o.fy);
    // unsigned 32-bit element offsets: one wide multiply-add per address, no sign extension
    const unsigned i0 = (unsigned)(ya * w + xa), i1 = i0 + (unsigned)w;
    const float4* r0 = nA + i0;
    const float4* r1 = nA + i1;
    const float* b0 = nB + i0;
    const float* b1 = nB + i1;
    o.q00 = __ldg(r0);
    o.q01 = __ldg(r0 + 1);
    o.q10 = __ldg(r1);
    o.q11 = __ldg(r1 + 1);
    o.b00 = __ldg(b0);
    o.b01 = __ldg(b0 + 1);
    o.b10 = __ldg(b1);
    o.b11 = __ldg(b1 + 1);
    const unsigned c = (unsigned)(gy * w + gx);
    o.pa = ld_stream(pA + c);
    o.pb = ld_stream(pB + c);
}

// Bilinear weights w00..w11 make every interpolated channel one FMUL + three FFMA (packed for the
// (a11,a12) and (a22,bx) channel pairs).  fx = fy = 0 (or 1 at the far border) keeps exactly the
// corner value, so identical frames still give exactly zero flow.
__device__ __forceinline__ GTerms g_terms(const GLoad& o, float du, float dv) {
    const float4 q00 = o.q00, q01 = o.q01, q10 = o.q10, q11 = o.q11, pa = o.pa;
    const float ofx = 1.f - o.fx, ofy = 1.f - o.fy;
    float w00, w01, w10, w11;
    mul2(w00, w01, ofx, o.fx, ofy, ofy);
    mul2(w10, w11, ofx, o.fx, o.fy, o.fy);
    float n11, n12, n22, nbx;
    mul2(n11, n12, q00.x, q00.y, w00, w00);
    fma2(n11, n12, q01.x, q01.y, w01, w01, n11, n12);
    fma2(n11, n12, q10.x, q10.y, w10, w10, n11, n12);
    fma2(n11, n12, q11.x, q11.y, w11, w11, n11, n12);
    mul2(n22, nbx, q00.z, q00.w, w00, w00);
    fma2(n22, nbx, q01.z, q01.w, w01, w01, n22, nbx);
    fma2(n22, nbx, q10.z, q10.w, w10, w10, n22, nbx);
    fma2(n22, nbx, q11.z, q11.w, w11, w11, n22, nbx);
    const float nby = fmaf(o.b11, w11, fmaf(o.b10, w10, fmaf(o.b01, w01, o.b00 * w00)));
    // A and delta-b at twice the reference's scale (the 1/2 of the averages dropped): every
    // product below is then exactly 4x, and the solve is scale-invariant, so the flow is unchanged
    float a11, a12, a22, e1;
    add2(a11, a12, pa.x, pa.y, n11, n12);          // 2 a11, 2 a12
    add2(a22, e1, pa.z, pa.w, n22, -nbx);          // 2 a22, -(nbx - bx_prev)
    const float e2 = o.pb - nby;
    float db1, db2;
    fma2(db1, db2, a11, a12, du, du, e1, e2);      // + A d (first column)
    fma2(db1, db2, a12, a22, dv, dv, db1, db2);    // + A d (second column)
    GTerms t;
    mul2(t.g11, t.g22, a11, a22, a11, a22);
    fma2(t.g11, t.g22, a12, a12, a12, a12, t.g11, t.g22);
    t.g12 = (a11 + a22) * a12;
    mul2(t.h1, t.h2, a11, a12, db1, db1);
    fma2(t.h1, t.h2, a12, a22, db2, db2, t.h1, t.h2);
    return t;
}

// One CTA per strip of `nr` vertically stacked FX x FY output tiles of one pair (FNT threads,
// 2 CTAs per SM).  The products G live in a ring of RG rows per plane: each tile computes only
// the FY rows its window adds (the first tile also the 2R rows above), the 2R overlap rows stay
// resident, so the halo overhead is (FX+2R)/FX x (FY*nr+2R)/(FY*nr) instead of
// (FX+2R)/FX x (FY+2R)/FY.  Ring slots: row r of the strip (relative to its first halo row) sits
// in slot r % RG; tile k's box sums overwrite slots of rows [FY*k, FY*k+FY), which no later tile
// reads.  RG = 48 >= FY + 2R keeps the footprint at ~76 KB, leaving the L1 room the gathers need.
constexpr int RG = 48;

// Ring row stride SW and plane stride PL (floats).  SW is odd, so phase 3 (a warp walks 32 rows
// of one column) is conflict-free.  PAD 2: PL == HW (mod 32), so the phase-2 warps that wrap from
// one plane to the next still address 32 consecutive banks.  PAD 1: also 2 SW == HW (mod 32), for
// the phase-1 warps that wrap from one pixel-pair row to the next (no faster, 7.5 KB larger).
constexpr int ring_sw(int hw, int pad) {
    int s = hw + 1;
    if (pad == 1 && ((hw / 2) & 1))
        while (((2 * s - hw) & 31) != 0 || !(s & 1)) ++s;
    return s;
}
constexpr int ring_pl(int hw, int pad) {
    int p = ring_sw(hw, pad) * RG;
    if (pad)
        while (((p - hw) & 31) != 0) ++p;
    return p;
}

// vertical (2R+1)-row running sums down one ring column (FY outputs, rows from slot BOFF on),
// written in place one step behind: a thread owns its column, and output j-1 overwrites row j-1
// only after row j-1 was subtracted for output j
template <int R, int BOFF, int SW>
__device__ __forceinline__ void vsum_inplace(float* col) {
    float acc = 0.f;
#pragma unroll
    for (int j = 0; j <= 2 * R; ++j) acc += col[((BOFF + j) % RG) * SW];
    float pv = acc;
#pragma unroll
    for (int j = 1; j < FY; ++j) {
        acc += col[((BOFF + j + 2 * R) % RG) * SW] - col[((BOFF + j - 1) % RG) * SW];
        col[((BOFF + j - 1) % RG) * SW] = pv;
        pv = acc;
    }
    col[((BOFF + FY - 1) % RG) * SW] = pv;
}

#ifndef FROI_FLOW_MINB
#define FROI_FLOW_MINB 2
#endif
template <int R, int PAD>
__global__ void __launch_bounds__(FNT, FROI_FLOW_MINB) k_flow_iter(Geom g, IterArgs a,
                                                      const float4* __restrict__ exA_f,
                                                      const float* __restrict__ exB_f,
                                                      const float4* __restrict__ exA_p,
                                                      const float* __restrict__ exB_p,
                                                      const int* __restrict__ prev,
                                                      const int* __restrict__ next,
                                                      const PairInfo* __restrict__ info, int nr) {
    extern __shared__ float smem_f[];
    // ring rows are SW = HW + 1 floats apart (odd stride: the row-wise box pass is conflict-free)
    constexpr int HW = FX + 2 * R, SW = ring_sw(HW, PAD), PL = ring_pl(HW, PAD);
    static_assert(FY + 2 * R <= RG && FY == 32 && RG == 48, "ring layout");
    const int p = blockIdx.z;
    const int l = a.l;
    const int w = g.lw[l], h = g.lh[l];
    const int x0 = blockIdx.x * FX, ys = blockIdx.y * FY * nr;
    float* G = smem_f;  // 5 planes [RG][SW]
    const size_t pair_off = (size_t)p * g.lsum;
    const size_t lo = g.loff[l];
    // opaque() keeps each plane base a single 64-bit value, so a gather address is one wide
    // multiply-add of its unsigned 32-bit element offset (no re-association with the level offset)
    const float4* pA = opaque(exA_f + (size_t)prev[p] * g.lsum + lo);
    const float* pB = opaque(exB_f + (size_t)prev[p] * g.lsum + lo);
    const bool sh = info[p].shifted != 0;
    const float4* nA = opaque((sh ? exA_p + pair_off : exA_f + (size_t)next[p] * g.lsum) + lo);
    const float* nB = opaque((sh ? exB_p + pair_off : exB_f + (size_t)next[p] * g.lsum) + lo);
    const float2* fin = opaque(a.flow_in + pair_off + lo);
    float2* out = opaque(a.flow_out + pair_off + lo);
    if (!FROI_FLOW_NOPF && a.mode) {
        // the first tile's prior rows (its later tiles' rows are prefetched during phase 2):
        // later pair rounds of the first tile then find them in L1
        const int xs = max(0, x0 - R), xe = min(w, x0 + FX + R);
        constexpr int NL = (HW * 8 + 127) / 128 + 1;
        for (int i = threadIdx.x; i < (FY + 2 * R) * NL; i += FNT) {
            const int row = i / NL, ln = i - row * NL;
            const int y = ys - R + row, x = xs + ln * 16;
            if (y >= 0 && y < h && x < xe) asm volatile("prefetch.global.L1 [%0];" ::"l"(fin + (size_t)y * w + x));
        }
    }
    for (int k = 0; k < nr; ++k) {
        const int y0 = ys + k * FY;
        if (y0 >= h) break;
        // phase 1: normal-equation products of the rows this tile adds; two independent pixels
        // per step so each thread keeps ~20 gathers in flight
        const int r0 = k == 0 ? 0 : FY * k + 2 * R;
        const int npx = (k == 0 ? FY + 2 * R : FY) * HW;
        // Each thread takes two vertically adjacent halo pixels (rows 2rp, 2rp+1 of the block).
        // When the lower pixel's bilinear top row is the upper pixel's bottom row (the common case
        // for a smooth flow) those four corners are reused from registers instead of re-gathered.
        auto phase1 = [&](auto in_tag) {
            constexpr bool IN = decltype(in_tag)::value;
            const int npp = npx / 2;
            // whole iterations of pixel pairs; the remainder goes out as single pixels over
            // twice as many threads (a shorter last step before the barrier)
            const int full = (npp / FNT) * FNT;
            for (int ip = threadIdx.x; ip < full; ip += FNT) {
                const int rp = ip / HW, hx = ip - rp * HW;
                const int ux = x0 - R + hx, uy = ys - R + r0 + 2 * rp;
                int gx, gyA, gyB;
                bool okA, okB;
                if (IN) {  // the whole block of rows and columns lies inside the image
                    gx = ux;
                    gyA = uy;
                    gyB = uy + 1;
                    okA = okB = true;
                } else {
                    const bool okx = ux >= 0 && ux < w;
                    okA = okx && uy >= 0 && uy < h;
                    okB = okx && uy + 1 >= 0 && uy + 1 < h;
                    gx = clampi(ux, 0, w - 1);
                    gyA = clampi(uy, 0, h - 1);
                    gyB = clampi(uy + 1, 0, h - 1);
                }
                const int siA = ((r0 + 2 * rp) % RG) * SW + hx, siB = ((r0 + 2 * rp + 1) % RG) * SW + hx;
                float2 prA = make_float2(0.f, 0.f), prB = make_float2(0.f, 0.f);
                if (a.mode)
                    asm volatile("ld.global.nc.v2.f32 {%0, %1}, [%4];\n\tld.global.nc.v2.f32 {%2, %3}, [%5];"
                                 : "=f"(prA.x), "=f"(prA.y), "=f"(prB.x), "=f"(prB.y)
                                 : "l"(fin + (unsigned)(gyA * w + gx)), "l"(fin + (unsigned)(gyB * w + gx)));
                GLoad lA, lB;
                int xaA, yaA, xaB, yaB;
                if (FROI_DIAG_ZEROFLOW) {  // diagnostic: gather at the pixel itself (coalesced)
                    prA.x = prA.x * 1e-30f;
                    prA.y = prA.y * 1e-30f;
                    prB.x = prB.x * 1e-30f;
                    prB.y = prB.y * 1e-30f;
                }
                bl_split(gx, prA.x, w, xaA, lA.fx);
                bl_split(gyA, prA.y, h, yaA, lA.fy);
                bl_split(gx, prB.x, w, xaB, lB.fx);
                bl_split(gyB, prB.y, h, yaB, lB.fy);
                const unsigned iA0 = (unsigned)(yaA * w + xaA), iA1 = iA0 + (unsigned)w;
                const unsigned iB0 = (unsigned)(yaB * w + xaB), iB1 = iB0 + (unsigned)w;
                FROI_DCHECK(iA1 + 1 < (unsigned)(w * h) && iB1 + 1 < (unsigned)(w * h));
                FROI_DCHECK(siA >= 0 && siA < RG * SW && siB >= 0 && siB < RG * SW);
                lA.q00 = __ldg(nA + iA0);
                lA.q01 = __ldg(nA + iA0 + 1);
                lA.q10 = __ldg(nA + iA1);
                lA.q11 = __ldg(nA + iA1 + 1);
                lA.b00 = __ldg(nB + iA0);
                lA.b01 = __ldg(nB + iA0 + 1);
                lA.b10 = __ldg(nB + iA1);
                lA.b11 = __ldg(nB + iA1 + 1);
                lB.q10 = __ldg(nA + iB1);
                lB.q11 = __ldg(nA + iB1 + 1);
                lB.b10 = __ldg(nB + iB1);
                lB.b11 = __ldg(nB + iB1 + 1);
                if (iB0 == iA1) {
                    lB.q00 = lA.q10;
                    lB.q01 = lA.q11;
                    lB.b00 = lA.b10;
                    lB.b01 = lA.b11;
                } else {
                    lB.q00 = __ldg(nA + iB0);
                    lB.q01 = __ldg(nA + iB0 + 1);
                    lB.b00 = __ldg(nB + iB0);
                    lB.b01 = __ldg(nB + iB0 + 1);
                }
                const unsigned cA = (unsigned)(gyA * w + gx), cB = (unsigned)(gyB * w + gx);
                lA.pa = ld_stream(pA + cA);
                lA.pb = ld_stream(pB + cA);
                lB.pa = ld_stream(pA + cB);
                lB.pb = ld_stream(pB + cB);
                GTerms tA = g_terms(lA, prA.x, prA.y), tB = g_terms(lB, prB.x, prB.y);
                if (!okA) tA = GTerms{0.f, 0.f, 0.f, 0.f, 0.f};
                if (!okB) tB = GTerms{0.f, 0.f, 0.f, 0.f, 0.f};
                G[siA] = tA.g11;
                G[PL + siA] = tA.g12;
                G[2 * PL + siA] = tA.g22;
                G[3 * PL + siA] = tA.h1;
                G[4 * PL + siA] = tA.h2;
                G[siB] = tB.g11;
                G[PL + siB] = tB.g12;
                G[2 * PL + siB] = tB.g22;
                G[3 * PL + siB] = tB.h1;
                G[4 * PL + siB] = tB.h2;
            }
            for (int q = threadIdx.x; q < 2 * (npp - full); q += FNT) {
                const int ip = full + (q >> 1);
                const int rp = ip / HW, hx = ip - rp * HW;
                const int ux = x0 - R + hx, uy = ys - R + r0 + 2 * rp + (q & 1);
                int gx, gy;
                bool ok;
                if (IN) {
                    gx = ux;
                    gy = uy;
                    ok = true;
                } else {
                    ok = ux >= 0 && ux < w && uy >= 0 && uy < h;
                    gx = clampi(ux, 0, w - 1);
                    gy = clampi(uy, 0, h - 1);
                }
                const float2 pr = a.mode ? __ldg(fin + (unsigned)(gy * w + gx)) : make_float2(0.f, 0.f);
                GLoad ld;
                g_load(ld, pA, pB, nA, nB, w, h, gx, gy, pr.x, pr.y);
                GTerms t = g_terms(ld, pr.x, pr.y);
                if (!ok) t = GTerms{0.f, 0.f, 0.f, 0.f, 0.f};
                const int si = ((r0 + 2 * rp + (q & 1)) % RG) * SW + hx;
                G[si] = t.g11;
                G[PL + si] = t.g12;
                G[2 * PL + si] = t.g22;
                G[3 * PL + si] = t.h1;
                G[4 * PL + si] = t.h2;
            }
        };
        const int ry0 = ys - R + r0, ry1 = ry0 + npx / HW;
        if (x0 - R >= 0 && x0 + FX + R <= w && ry0 >= 0 && ry1 <= h) phase1(std::true_type{});
        else phase1(std::false_type{});
        __syncthreads();
        // the threads phase 2 leaves idle pull the next tile's prior rows into L1, so its
        // gathers do not start behind an L2/DRAM round trip
        if (!FROI_FLOW_NOPF && a.mode && k + 1 < nr && threadIdx.x >= 5 * HW) {
            const int ny0 = ys + FY * (k + 1) + R;
            const int xs = max(0, x0 - R), xe = min(w, x0 + FX + R);
            constexpr int NL = (HW * 8 + 127) / 128 + 1;
            for (int i = threadIdx.x - 5 * HW; i < FY * NL; i += FNT - 5 * HW) {
                const int row = i / NL, ln = i - row * NL;
                const int y = ny0 + row, x = xs + ln * 16;
                if (y < h && x < xe) asm volatile("prefetch.global.L1 [%0];" ::"l"(fin + (size_t)y * w + x));
            }
        }
        // phase 2: vertical running sums down each of the 5*HW ring columns (FY outputs each),
        // in place over this tile's first FY ring rows
        const int b0 = (FY * k) % RG;  // 0, 32 or 16
        if (!FROI_DIAG_NOBOX && threadIdx.x < 5 * HW) {
            const int vc = threadIdx.x / HW, vx = threadIdx.x - vc * HW;
            float* col = G + vc * PL + vx;
            if (b0 == 0) vsum_inplace<R, 0, SW>(col);
            else if (b0 == 32) vsum_inplace<R, 32, SW>(col);
            else vsum_inplace<R, 16, SW>(col);
        }
        __syncthreads();
        // phase 3: horizontal running sums along each of the 5*FY rows in 32-wide segments, in
        // place one step behind; a segment first takes the 2R inputs it shares with the next
        // segment into registers, so after one barrier every thread owns what it overwrites
        constexpr int NSEG = FX / 32;
        const bool hact = !FROI_DIAG_NOBOX && threadIdx.x < 5 * FY * NSEG;
        const int hc = threadIdx.x / (FY * NSEG);
        const int hrem = threadIdx.x - hc * FY * NSEG;
        const int hsg = hrem / FY, hty = hrem - hsg * FY;  // a warp walks 32 rows of one segment
        float* hrow = G + hc * PL + ((b0 + hty) % RG) * SW + hsg * 32;
        float tail[2 * R];
        if (hact) {
#pragma unroll
            for (int j = 0; j < 2 * R; ++j) tail[j] = hrow[32 + j];
        }
        __syncthreads();
        if (hact) {
            float acc = 0.f;
#pragma unroll
            for (int j = 0; j <= 2 * R; ++j) acc += hrow[j];
            float pv = acc;
#pragma unroll
            for (int j = 1; j < 32; ++j) {
                const float in = j + 2 * R < 32 ? hrow[j + 2 * R] : tail[j + 2 * R - 32];
                acc += in - hrow[j - 1];
                hrow[j - 1] = pv;
                pv = acc;
            }
            hrow[31] = pv;
        }
        __syncthreads();
        // phase 4: the 2x2 solve of the clipped-window means (flow.hpp:242-253) on the window
        // sums: the solution and the det > 1e-9 ||G||^2 test are invariant to the common 1/count
        // scale, so it is never applied.  fp32 with a compensated determinant (Kahan: the g12^2
        // rounding error is carried exactly).
        const int tx = threadIdx.x % FX, x = x0 + tx;
        const int ty0 = threadIdx.x / FX;
        const float* Gs = G + tx;
#pragma unroll
        for (int j = 0; j < FY / (FNT / FX); ++j) {
            const int ty = ty0 + j * (FNT / FX), y = y0 + ty;
            const int rr = b0 + ty;
            const int sidx = (rr >= RG ? rr - RG : rr) * SW;
            FROI_DCHECK(sidx >= 0 && sidx + tx < RG * SW);
            const float g11 = Gs[sidx], g12 = Gs[PL + sidx], g22 = Gs[2 * PL + sidx];
            const float h1 = Gs[3 * PL + sidx], h2 = Gs[4 * PL + sidx];
            if (x >= w || y >= h) continue;
            const float q = g12 * g12;
            const float qe = fmaf(g12, g12, -q);
            const float det = fmaf(g11, g22, -q) - qe;
            const float frob2 = fmaf(g11, g11, fmaf(2.f * g12, g12, g22 * g22));
            const unsigned o = (unsigned)(y * w + x);
            float2 r;
            if (det > 1e-9f * frob2) {
                const float rd = __fdividef(1.f, det);
                r.x = (g22 * h1 - g12 * h2) * rd;
                r.y = (g11 * h2 - g12 * h1) * rd;
            } else {
                // singular: keep the prior (flow.hpp:245-246), zero on the coarsest first pass
                r = a.mode ? fin[o] : make_float2(0.f, 0.f);
            }
            out[o] = r;
        }
        __syncthreads();  // ring rows are rewritten by the next tile
    }
}

#ifndef FROI_NR_MAX
#define FROI_NR_MAX 32
#endif
// tiles per strip: the least (rounds of resident CTAs) x (rows each CTA computes, halo included)
// among strips of 1..32 tiles (powers of two) that still fill every CTA slot (2 per SM) once
int strip_tiles(const Geom& g, int l, int n_pairs, int R) {
    static const int sms = [] {
        int dev = 0, n = 148;
        if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        return n > 0 ? n : 148;
    }();
    const long long slots = 2LL * sms;
    const int tx = cdiv(g.lw[l], FX), ty = cdiv(g.lh[l], FY);
    int best = 1;
    long long best_cost = -1;
    for (int nr = 1; nr <= FROI_NR_MAX; nr *= 2) {
        const long long ctas = (long long)tx * cdiv(ty, nr) * n_pairs;
        if (nr > 1 && ctas < slots) break;
        const long long cost = cdiv(ctas, slots) * (long long)(FY * std::min(nr, ty) + 2 * R);
        if (best_cost < 0 || cost < best_cost) {
            best_cost = cost;
            best = nr;
        }
    }
    return best;
}

template <int R, int PAD>
void launch_iter_t(const Geom& g, const IterArgs& a, const FlowBuffers& b, const int* d_prev,
                   const int* d_next, const PairInfo* d_info, int n_pairs, cudaStream_t s) {
    size_t smem = sizeof(float) * 5 * (size_t)ring_pl(FX + 2 * R, PAD);
    // experiment knob: request at least this much shared memory (forces fewer CTAs per SM,
    // leaving room for the other lane's kernels)
    static const size_t smem_min = [] {
        const char* e = getenv("FROI_FLOW_SMEM_MIN");
        return e ? (size_t)atol(e) : (size_t)0;
    }();
    smem = std::max(smem, smem_min);
    // kernel attributes are per device: set on every call (one host thread may drive several)
    FROI_CUDA(cudaFuncSetAttribute(k_flow_iter<R, PAD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int nr = strip_tiles(g, a.l, n_pairs, R);
    dim3 grid(cdiv(g.lw[a.l], FX), cdiv(g.lh[a.l], FY * nr), n_pairs);
    k_flow_iter<R, PAD><<<grid, FNT, smem, s>>>(g, a, b.exA_f, b.exB_f, b.exA_p, b.exB_p, d_prev, d_next, d_info, nr);
    FROI_LAUNCH_CHECK();
}

template <int R>
void launch_iter(const Geom& g, const IterArgs& a, const FlowBuffers& b, const int* d_prev,
                 const int* d_next, const PairInfo* d_info, int n_pairs, cudaStream_t s) {
    // plane-padded ring (A/B on the C3 bench, k_flow_iter time: no padding 276.4 us, row and
    // plane padding 270.1 us, plane padding only 270.0 us with 7.5 KB less shared memory per CTA,
    // which keeps two CTAs inside the 164 KB carveout: L1 92 KB instead of 60 KB)
    launch_iter_t<R, 2>(g, a, b, d_prev, d_next, d_info, n_pairs, s);
}

template <typename K>
void set_smem(K kernel, size_t bytes) {
    if (bytes > 48 * 1024)
        FROI_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
}

size_t polyexp_smem(int r) { return sizeof(float) * ((PY + 2 * r) * (PX + 2 * r) + 3 * (PY + 2 * r) * PX); }

void pyr_bounds(const Geom& g, int l, int& rwmax, int& rhmax) {
    const double sx = (double)g.lw[l] / g.lw[l + 1], sy = (double)g.lh[l] / g.lh[l + 1];
    rwmax = (int)(QX * sx) + 4;
    rhmax = (int)(QY * sy) + 4;
}
size_t pyr_smem(int rwmax, int rhmax) {
    return sizeof(float) * ((rhmax + 6) * (rwmax + 6) + (rhmax + 6) * rwmax + rhmax * rwmax);
}

}  // namespace

// exact 2:1 pyramid step (the fixed-tile kernel), else the general resample
bool is_half(const Geom& g, int l) { return g.lw[l] == 2 * g.lw[l + 1] && g.lh[l] == 2 * g.lh[l + 1]; }
#define FROI_HALF(h, ...)        \
    if (h) {                     \
        constexpr bool HF = true;  \
        __VA_ARGS__;             \
    } else {                     \
        constexpr bool HF = false; \
        __VA_ARGS__;             \
    }

// the default poly_n = 5 (radius 2) runs fully unrolled; other radii take the runtime loops
#define FROI_POLY_RC(P, ...)            \
    if ((P).poly_radius == 2) {         \
        constexpr int RC = 2;           \
        __VA_ARGS__;                    \
    } else {                            \
        constexpr int RC = 0;           \
        __VA_ARGS__;                    \
    }

void launch_expand_frames(const Geom& g, const DevParams& P, const FlowBuffers& b, int n_slots,
                          cudaStream_t s) {
    if (n_slots <= 0) return;
    const size_t pe = polyexp_smem(P.poly_radius);
    // level 0 expansion straight from the denoised frame
    {
        dim3 grid(cdiv(g.W, PX), cdiv(g.H, PY), n_slots);
        if (g.sample_bytes == 1) {
            FROI_POLY_RC(P, set_smem(k_polyexp_frame<uint8_t, RC>, pe);
                         k_polyexp_frame<uint8_t, RC><<<grid, PNT, pe, s>>>(g, P, (const uint8_t*)b.den, b.exA_f, b.exB_f))
        } else {
            FROI_POLY_RC(P, set_smem(k_polyexp_frame<uint16_t, RC>, pe);
                         k_polyexp_frame<uint16_t, RC><<<grid, PNT, pe, s>>>(g, P, (const uint16_t*)b.den, b.exA_f, b.exB_f))
        }
        FROI_LAUNCH_CHECK();
    }
    for (int l = 0; l + 1 < g.L; ++l) {
        int rwmax, rhmax;
        pyr_bounds(g, l, rwmax, rhmax);
        const bool half = is_half(g, l);
        const size_t ps = half ? pyr2_smem() : pyr_smem(rwmax, rhmax);
        const dim3 grid = half ? dim3(cdiv(g.lw[l + 1], Q2X), cdiv(g.lh[l + 1], Q2Y), n_slots)
                               : dim3(cdiv(g.lw[l + 1], QX), cdiv(g.lh[l + 1], QY), n_slots);
        FROI_HALF(half,
            if (l == 0) {
                if (g.sample_bytes == 1) {
                    set_smem(k_pyr0_frame<uint8_t, HF>, ps);
                    k_pyr0_frame<uint8_t, HF><<<grid, QNT, ps, s>>>(g, P, (const uint8_t*)b.den, b.pyr_f, rwmax, rhmax);
                } else {
                    set_smem(k_pyr0_frame<uint16_t, HF>, ps);
                    k_pyr0_frame<uint16_t, HF><<<grid, QNT, ps, s>>>(g, P, (const uint16_t*)b.den, b.pyr_f, rwmax, rhmax);
                }
            } else {
                set_smem(k_pyr_level<HF>, ps);
                k_pyr_level<HF><<<grid, QNT, ps, s>>>(g, P, l, b.pyr_f, nullptr, rwmax, rhmax);
            })
        FROI_LAUNCH_CHECK();
        dim3 eg(cdiv(g.lw[l + 1], PX), cdiv(g.lh[l + 1], PY), n_slots);
        FROI_POLY_RC(P, set_smem(k_polyexp_level<RC>, pe);
                     k_polyexp_level<RC><<<eg, PNT, pe, s>>>(g, P, l + 1, b.pyr_f, g.lsum - g.loff[1],
                                                             nullptr, b.exA_f, b.exB_f))
        FROI_LAUNCH_CHECK();
    }
}

void launch_expand_shifted(const Geom& g, const DevParams& P, const FlowBuffers& b,
                           const int* d_next, const PairInfo* d_info, int n_pairs, cudaStream_t s) {
    if (n_pairs <= 0) return;
    const size_t pe = polyexp_smem(P.poly_radius);
    {
        dim3 grid(cdiv(g.W, PX), cdiv(g.H, PY), n_pairs);
        if (g.sample_bytes == 1) {
            FROI_POLY_RC(P, set_smem(k_polyexp_shifted<uint8_t, RC>, pe);
                         k_polyexp_shifted<uint8_t, RC><<<grid, PNT, pe, s>>>(g, P, (const uint8_t*)b.den, d_next,
                                                                              d_info, b.exA_p, b.exB_p))
        } else {
            FROI_POLY_RC(P, set_smem(k_polyexp_shifted<uint16_t, RC>, pe);
                         k_polyexp_shifted<uint16_t, RC><<<grid, PNT, pe, s>>>(g, P, (const uint16_t*)b.den, d_next,
                                                                               d_info, b.exA_p, b.exB_p))
        }
        FROI_LAUNCH_CHECK();
    }
    for (int l = 0; l + 1 < g.L; ++l) {
        int rwmax, rhmax;
        pyr_bounds(g, l, rwmax, rhmax);
        const bool half = is_half(g, l);
        const size_t ps = half ? pyr2_smem() : pyr_smem(rwmax, rhmax);
        const dim3 grid = half ? dim3(cdiv(g.lw[l + 1], Q2X), cdiv(g.lh[l + 1], Q2Y), n_pairs)
                               : dim3(cdiv(g.lw[l + 1], QX), cdiv(g.lh[l + 1], QY), n_pairs);
        FROI_HALF(half,
            if (l == 0) {
                if (g.sample_bytes == 1) {
                    set_smem(k_pyr0_shifted<uint8_t, HF>, ps);
                    k_pyr0_shifted<uint8_t, HF><<<grid, QNT, ps, s>>>(g, P, (const uint8_t*)b.den, d_next, d_info, b.pyr_p, rwmax, rhmax);
                } else {
                    set_smem(k_pyr0_shifted<uint16_t, HF>, ps);
                    k_pyr0_shifted<uint16_t, HF><<<grid, QNT, ps, s>>>(g, P, (const uint16_t*)b.den, d_next, d_info, b.pyr_p, rwmax, rhmax);
                }
            } else {
                set_smem(k_pyr_level<HF>, ps);
                k_pyr_level<HF><<<grid, QNT, ps, s>>>(g, P, l, b.pyr_p, d_info, rwmax, rhmax);
            })
        FROI_LAUNCH_CHECK();
        dim3 eg(cdiv(g.lw[l + 1], PX), cdiv(g.lh[l + 1], PY), n_pairs);
        FROI_POLY_RC(P, set_smem(k_polyexp_level<RC>, pe);
                     k_polyexp_level<RC><<<eg, PNT, pe, s>>>(g, P, l + 1, b.pyr_p, g.lsum - g.loff[1],
                                                             d_info, b.exA_p, b.exB_p))
        FROI_LAUNCH_CHECK();
    }
}

int launch_flow(const Geom& g, const DevParams& P, const FlowBuffers& b, const int* d_prev,
                const int* d_next, const PairInfo* d_info, int n_pairs, cudaStream_t s) {
    if (n_pairs <= 0) return 0;
    const int R = P.window_radius;
    float2* buf[2] = {b.flow0, b.flow1};
    int cur = 0;
    for (int l = g.L - 1; l >= 0; --l) {
        for (int it = 0; it < P.iterations; ++it) {
            IterArgs a;
            a.l = l;
            a.mode = (it == 0 && l == g.L - 1) ? 0 : 1;
            if (it == 0 && l < g.L - 1) {
                // upscale the coarser estimate into this level of the same buffer (flow.hpp:318-337)
                const float fx = (float)((double)g.lw[l] / g.lw[l + 1]);
                const float fy = (float)((double)g.lh[l] / g.lh[l + 1]);
                // (16-byte stores: the level's base and the per-pair stride must keep float2 pairs aligned)
                static const bool up2 = [] {
                    const char* e = getenv("FROI_UPSAMPLE2");
                    return !(e && atoi(e) == 0);
                }();
                if (up2 && g.lw[l] == 2 * g.lw[l + 1] && g.lh[l] == 2 * g.lh[l + 1] && g.lw[l + 1] >= 3 &&
                    g.lh[l + 1] >= 3 && g.lsum % 2 == 0 && g.loff[l] % 2 == 0) {
                    dim3 ug(cdiv(g.lw[l + 1], 32), cdiv(g.lh[l + 1], 8), n_pairs);
                    k_upsample2<<<ug, 256, 0, s>>>(g, l, buf[cur], buf[cur], fx, fy);
                } else {
                    dim3 ug(cdiv(g.lw[l], 32), cdiv(g.lh[l], 32), n_pairs);
                    k_upsample<<<ug, 256, 0, s>>>(g, l, buf[cur], buf[cur], fx, fy,
                                                  (float)(1.0 / ((double)g.lw[l] / g.lw[l + 1])),
                                                  (float)(1.0 / ((double)g.lh[l] / g.lh[l + 1])));
                }
                FROI_LAUNCH_CHECK();
            }
            a.flow_in = buf[cur];
            a.flow_out = buf[1 - cur];
            switch (R) {  // window_size 3..15 (the reference default is 15)
                case 1: launch_iter<1>(g, a, b, d_prev, d_next, d_info, n_pairs, s); break;
                case 2: launch_iter<2>(g, a, b, d_prev, d_next, d_info, n_pairs, s); break;
                case 3: launch_iter<3>(g, a, b, d_prev, d_next, d_info, n_pairs, s); break;
                case 4: launch_iter<4>(g, a, b, d_prev, d_next, d_info, n_pairs, s); break;
                case 5: launch_iter<5>(g, a, b, d_prev, d_next, d_info, n_pairs, s); break;
                case 6: launch_iter<6>(g, a, b, d_prev, d_next, d_info, n_pairs, s); break;
                case 7: launch_iter<7>(g, a, b, d_prev, d_next, d_info, n_pairs, s); break;
                default: throw Error(1, "flow: window_size > 15 is not supported by the GPU flow kernel");
            }
            cur = 1 - cur;
        }
    }
    return cur;
}

void launch_expand_image(const Geom& g, const DevParams& P, const float* d_img, float* d_planes,
                         cudaStream_t s) {
    const size_t pe = polyexp_smem(P.poly_radius);
    set_smem(k_polyexp_debug, pe);
    k_polyexp_debug<<<dim3(cdiv(g.W, PX), cdiv(g.H, PY), 1), PNT, pe, s>>>(g, P, d_img, d_planes);
    FROI_LAUNCH_CHECK();
}

}  // namespace froi
