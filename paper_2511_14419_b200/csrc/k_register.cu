// k_register.cu — phase-correlation registration (registration.hpp:26-97, fft.hpp:19-55),
// bit-exact with the reference.
//
// The reference transforms with an iterative radix-2 FFT whose twiddles come from the
// recurrence w *= wlen.  The host replays that recurrence once per context (same libm cos/sin,
// same complex product) into twiddle tables, and every butterfly here performs exactly the
// reference's arithmetic with explicit round-to-nearest fp64 operations, so the correlation
// surface, the selected shift and the confidence are bit-identical.  Work split per pair:
//   k_fft_rows_fwd  one CTA per (row, frame): windowed mean-removed input (host Hann tables),
//                   bit-reversed into shared memory, row FFT                    [per new frame]
//   k_fft_cols      one CTA per (column block, frame): column FFTs in shared memory
//   k_xpow_rows_inv one CTA per (row, pair): cross-power conj(Fa)Fb/|.| (glibc hypot
//                   restated), inverse row FFT, keeps only the 2M+1 columns the search reads
//   k_inv_cols      one CTA per (needed column, pair): inverse column FFT, keeps 2M+1 rows
//   k_argmax        one CTA per pair: first strict maximum in dy-major scan, second peak
//                   outside Chebyshev radius 2, confidence, 1.5 fallback (roi.hpp:333)
// Each frame's spectrum is computed once and shared by the two pairs that use it.
#include "kernels.cuh"

namespace froi {
namespace {

constexpr int NT = 256;

__device__ __forceinline__ int brev(int x, int log2n) {
    return log2n == 0 ? 0 : (int)(__brev((unsigned)x) >> (32 - log2n));
}

// (v * w) as GCC expands std::complex<double> multiplication, then u +- v (fft.hpp:32-35).
__device__ __forceinline__ void bfly(double2& u, double2& v, const double2 w) {
    const double vr = dsub(dmul(v.x, w.x), dmul(v.y, w.y));
    const double vi = dadd(dmul(v.x, w.y), dmul(v.y, w.x));
    const double2 nu = make_double2(dadd(u.x, vr), dadd(u.y, vi));
    v = make_double2(dsub(u.x, vr), dsub(u.y, vi));
    u = nu;
}

// Shared-memory slot of element i: pad slots every 16 and every 128 elements keep every radix-16
// pass and the bit-reversed scatter (interleave index fastest across lanes) at the 4-wavefront
// minimum for 16-byte elements, for rows and column blocks alike (checked offline for n = 2^8..2^12).
__device__ __forceinline__ int pd(int i) { return i + (i >> 4) + (i >> 7); }
__host__ __device__ constexpr int padded(int n) { return n + (n >> 4) + (n >> 7) + 1; }
struct PadStd {
    static __device__ __forceinline__ int at(int i) { return pd(i); }
};
// The cross-power kernel's layout (4 interleaved rows, radix-8 passes, bit-reversed scatter from
// row-major element order): pads every 8, 256 and 512 elements put every quarter-warp of a
// 128-bit access on 8 distinct bank groups (checked offline for n = 1024: the standard layout
// costs 2x the ideal wavefronts on the scatter and 1.25x on the passes).
struct PadX {
    static __device__ __forceinline__ int at(int i) { return i + (i >> 3) + (i >> 8) + (i >> 9); }
};
__host__ __device__ constexpr int padded_x(int n) { return n + (n >> 3) + (n >> 8) + (n >> 9) + 1; }

// Q consecutive radix-2 stages (half-lengths h, 2h, .., h*2^(Q-1), h = 2^s) over groups of
// 2^Q elements {i + m*h} held in registers, for `1 << lc` interleaved transforms of length n
// (element i of transform c at a[pd(i) << lc | c]).  Every butterfly is the reference's
// (fft.hpp:32-35) with its operands and twiddle tw[hq - 1 + k] (the w sequence for
// len = 2hq); only the number of shared-memory round trips changes.
//
// prune_m >= 0 (the inverse transforms of the registration, whose outputs are read only at
// positions [0, M] and [n-M, n)): after stage t the value at position p feeds exactly the final
// outputs q with q = p mod 2^(t+1), so a group whose positions k + m*h (m < 2^Q) hit no needed
// residue mod T = h*2^Q is skipped; every input of a computed group is then itself needed, so the
// outputs read are exactly the reference's.
template <int Q, typename Pad = PadStd>
__device__ __forceinline__ void fft_pass(double2* a, int n, int s, int lc,
                                         const double2* __restrict__ tw, int prune_m = -1) {
    constexpr int G = 1 << Q;
    const int h = 1 << s;
    const int ng = (n >> Q) << lc;
    const int T = h << Q;
    for (int j = threadIdx.x; j < ng; j += blockDim.x) {
        const int c = j & ((1 << lc) - 1), b = j >> lc;
        const int k = b & (h - 1);
        if (prune_m >= 0 && T > 2 * prune_m + 1 && k > prune_m && k + (G - 1) * h < T - prune_m) continue;
        const int i = ((b >> s) << (s + Q)) + k;
        double2 e[G];
#pragma unroll
        for (int m = 0; m < G; ++m) e[m] = a[(Pad::at(i + m * h) << lc) | c];
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const int hq = h << q;
#pragma unroll
            for (int m = 0; m < G; ++m) {
                if (m & (1 << q)) continue;
                const int kq = k + (m & ((1 << q) - 1)) * h;
                bfly(e[m], e[m | (1 << q)], tw[hq - 1 + kq]);
            }
        }
#pragma unroll
        for (int m = 0; m < G; ++m) a[(Pad::at(i + m * h) << lc) | c] = e[m];
    }
    __syncthreads();
}

// The n - 1 twiddles of a length-n transform into shared memory (dst, behind the data), so the
// butterflies read them without L1 tag lookups; the caller's barrier publishes them.  When data
// and twiddles together would exceed a CTA's shared memory (8192-point transforms), the
// butterflies read the twiddles from global memory instead (in_smem == 0).
__device__ __forceinline__ const double2* stage_tw(double2* dst, const double2* __restrict__ tw, int n,
                                                   int in_smem) {
    if (!in_smem) return tw;
    for (int i = threadIdx.x; i < n - 1; i += blockDim.x) dst[i] = __ldg(tw + i);
    return dst;
}
constexpr size_t kMaxCtaSmem = 227 * 1024;

// All log2n stages, QM per pass; input already bit-reversed.
template <int QM, typename Pad = PadStd>
__device__ __forceinline__ void fft_stages(double2* a, int n, int log2n, int lc,
                                           const double2* __restrict__ tw, int prune_m = -1) {
    int s = 0;
    for (; s + QM <= log2n; s += QM) fft_pass<QM, Pad>(a, n, s, lc, tw, prune_m);
    switch (log2n - s) {
        case 3: fft_pass<3, Pad>(a, n, s, lc, tw, prune_m); break;
        case 2: fft_pass<2, Pad>(a, n, s, lc, tw, prune_m); break;
        case 1: fft_pass<1, Pad>(a, n, s, lc, tw, prune_m); break;
        default: break;
    }
}
#ifndef FFT_Q_ROWS
#define FFT_Q_ROWS 4
#endif
#ifndef FFT_Q_COLS
#define FFT_Q_COLS 4
#endif
#ifndef FFT_Q_XPOW
#define FFT_Q_XPOW 3
#endif
// stages per shared-memory pass: radix-16 for the plain transforms; radix-8 (~70 registers,
// 3 CTAs per SM) where the cross-power prologue needs the occupancy
constexpr int kQRows = FFT_Q_ROWS, kQCols = FFT_Q_COLS, kQXpow = FFT_Q_XPOW;

// Rows per CTA for the row transforms: 256 threads, one radix-16 group per thread.
__host__ __device__ constexpr int rows_lc(int log2n) { return log2n >= 12 ? 0 : (log2n >= 8 ? 12 - log2n : 4); }

template <typename T>
__global__ void __launch_bounds__(NT) k_fft_rows_fwd(int W, int H, int pw, int ph, int log2pw, int tw_smem,
                                                     const T* __restrict__ den,
                                                     const unsigned long long* __restrict__ sums,
                                                     const double* __restrict__ wx,
                                                     const double* __restrict__ wy,
                                                     const double2* __restrict__ tw,
                                                     double2* __restrict__ spec) {
    extern __shared__ double2 sm[];
    double2* a = sm;
    const int lc = rows_lc(log2pw), R = 1 << lc;
    const int y0 = blockIdx.x * R, slot = blockIdx.y;
    const T* f = den + (size_t)slot * W * H;
    // windowed_spectrum_input (registration.hpp:26-42): exact integer sum, then one division
    const double mean = ddiv((double)sums[slot], (double)((long long)W * H));
    const double2* stw = stage_tw(a + ((size_t)padded(pw) << lc), tw, pw, tw_smem);
    if (sizeof(T) == 1 && W == pw && H == ph && (W & 15) == 0 && (R << log2pw) == 16 * NT) {
        // 8-bit frames without padding: each thread reads 16 consecutive samples of one row with
        // one 128-bit load, then converts and scatters them to their bit-reversed slots.  The
        // lowest lane bits pick the row, the next 3 - lc the top bits of x (the low bits of the
        // bit-reversed slot), so every 8-lane phase of a 128-bit store hits 8 distinct bank groups.
        const int hb = lc >= 3 ? 0 : 3 - lc;
        const int r = threadIdx.x & (R - 1), u = threadIdx.x >> lc;
        const int x0 = (u & ((1 << hb) - 1)) * (pw >> hb) + (u >> hb) * 16;
        const int y = y0 + r;
        if (y < ph) {
            const uint4 raw = __ldg((const uint4*)(f + (size_t)y * W + x0));
            const double wyv = __ldg(wy + y);
            const unsigned int wds[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                const int x = x0 + k;
                const double sv = (double)((wds[k >> 2] >> (8 * (k & 3))) & 0xffu);
                const double val = dmul(dmul(dsub(sv, mean), __ldg(wx + x)), wyv);
                a[(pd(brev(x, log2pw)) << lc) | r] = make_double2(val, 0.0);
            }
        }
    } else {
        for (int e = threadIdx.x; e < (R << log2pw); e += NT) {
            const int r = e & (R - 1), x = e >> lc;
            const int y = y0 + r;
            if (y >= ph) continue;
            const int sy = min(y, H - 1), sx = min(x, W - 1);
            const double v = dmul(dmul(dsub((double)f[(size_t)sy * W + sx], mean), wx[x]), wy[y]);
            a[(pd(brev(x, log2pw)) << lc) | r] = make_double2(v, 0.0);
        }
    }
    __syncthreads();
    fft_stages<kQRows>(a, pw, log2pw, lc, stw);
    for (int e = threadIdx.x; e < (R << log2pw); e += NT) {
        const int r = e & (R - 1), x = e >> lc;
        if (y0 + r < ph) spec[((size_t)slot * ph + y0 + r) * pw + x] = a[(pd(x) << lc) | r];
    }
}

// Warp-per-row forward transform for 1024-point rows (the 1024^2 geometries): one warp holds its
// row in registers, 32 elements per lane.  Layout B (lane l holds positions 32l..32l+31 of the
// bit-reversed array) makes the stages of half-length 1..16 lane-local with warp-uniform twiddles;
// one padded shared-memory transpose gives layout A (lane l holds positions l + 32m), where the
// stages of half-length 32..512 are lane-local.  Every butterfly is the reference's, with the same
// operands and twiddle as fft_pass; only two shared-memory round trips remain (vs eight).
constexpr int RW_WARPS = 4;

__device__ __forceinline__ int brev5(int x) { return (int)(__brev((unsigned)x) >> 27); }

template <typename T>
__global__ void __launch_bounds__(32 * RW_WARPS, 3) k_fft_rows_w1024(int W, int H, int ph,
                                                                     const T* __restrict__ den,
                                                                     const unsigned long long* __restrict__ sums,
                                                                     const double* __restrict__ wx,
                                                                     const double* __restrict__ wy,
                                                                     const double2* __restrict__ tw,
                                                                     double2* __restrict__ spec) {
    extern __shared__ double2 xs_dyn[];  // RW_WARPS x (33 * 32)
    const int warp = threadIdx.x >> 5, l = threadIdx.x & 31;
    const int y = blockIdx.x * RW_WARPS + warp, slot = blockIdx.y;
    if (y >= ph) return;  // warp-uniform
    const T* f = den + (size_t)slot * W * H;
    const double mean = ddiv((double)sums[slot], (double)((long long)W * H));
    const double wyv = __ldg(wy + y);
    const T* row = f + (size_t)min(y, H - 1) * W;
    const int bl = brev5(l);
    double2 e[32];
    // position 32l + m holds input x = brev10(32l + m) = 32 brev5(m) + brev5(l)
#pragma unroll
    for (int m = 0; m < 32; ++m) {
        const int x = 32 * ((int)(__brev((unsigned)m) >> 27)) + bl;
        const double sv = (double)row[min(x, W - 1)];
        e[m] = make_double2(dmul(dmul(dsub(sv, mean), __ldg(wx + x)), wyv), 0.0);
    }
#pragma unroll
    for (int s = 0; s < 5; ++s) {
        const int h = 1 << s;
#pragma unroll
        for (int m = 0; m < 32; ++m) {
            if (m & h) continue;
            if (s == 0 || (s == 1 && (m & 1) == 0)) {
                // real inputs (imaginary parts +0: the windowed samples, then stage 0's sums) and
                // the twiddle (1, 0) (every length's first w, fft.hpp:30): the reference's
                // butterfly reduces exactly to u + v, u - v on the real parts, imaginary parts +0
                const double a = e[m].x, b = e[m + h].x;
                e[m] = make_double2(dadd(a, b), 0.0);
                e[m + h] = make_double2(dsub(a, b), 0.0);
            } else {
                bfly(e[m], e[m + h], __ldg(tw + h - 1 + (m & (h - 1))));
            }
        }
    }
    double2* xw = xs_dyn + warp * (33 * 32);
#pragma unroll
    for (int m = 0; m < 32; ++m) xw[33 * l + m] = e[m];  // position p at p + p / 32
    __syncwarp();
#pragma unroll
    for (int m = 0; m < 32; ++m) e[m] = xw[l + 33 * m];
#pragma unroll
    for (int j = 0; j < 5; ++j) {
        const int hm = 1 << j, h = 32 << j;
#pragma unroll
        for (int m = 0; m < 32; ++m) {
            if (m & hm) continue;
            bfly(e[m], e[m + hm], __ldg(tw + h - 1 + l + 32 * (m & (hm - 1))));
        }
    }
    double2* out = spec + ((size_t)slot * ph + y) * 1024;
#pragma unroll
    for (int m = 0; m < 32; ++m) out[l + 32 * m] = e[m];
}

__global__ void __launch_bounds__(NT) k_fft_cols(int pw, int ph, int log2ph, int lcb, int tw_smem,
                                                 const double2* __restrict__ tw,
                                                 double2* __restrict__ spec) {
    extern __shared__ double2 sm[];
    double2* a = sm;
    const int cb = 1 << lcb;
    const int slot = blockIdx.y, c0 = blockIdx.x * cb;
    double2* base = spec + (size_t)slot * ph * pw + c0;
    const int n = ph << lcb;
    // element i -> (row, column): the lowest bits pick the column, the next 3 - lcb the top bits
    // of the row (= the low bits of its bit-reversed slot), so every 8-lane phase of the 128-bit
    // scatter hits 8 distinct bank groups; rows are 16*pw bytes apart, so no coalescing is lost
    const int hb = lcb >= 3 ? 0 : 3 - lcb;
    auto row_of = [&](int i) {
        const int u = i >> lcb;
        return (u & ((1 << hb) - 1)) * (ph >> hb) + (u >> hb);
    };
    // global -> shared without a register round trip (cp.async, 16 B per element): every element
    // of the column block is in flight at once
    for (int i = threadIdx.x; i < n; i += NT) {
        const double2* src = base + (size_t)row_of(i) * pw + (i & (cb - 1));
        const unsigned dst = (unsigned)__cvta_generic_to_shared(a + ((pd(brev(row_of(i), log2ph)) << lcb) | (i & (cb - 1))));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
    }
    const double2* stw = stage_tw(a + ((size_t)padded(ph) << lcb), tw, ph, tw_smem);
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    fft_stages<kQCols>(a, ph, log2ph, lcb, stw);
    for (int i = threadIdx.x; i < (ph << lcb); i += NT) {
        const int r = i >> lcb, c = i & (cb - 1);
        base[(size_t)r * pw + c] = a[(pd(r) << lcb) | c];
    }
}

__global__ void __launch_bounds__(NT, 3) k_xpow_rows_inv(int pw, int ph, int log2pw, int M,
                                                         const double2* __restrict__ spec,
                                                         const int* __restrict__ prev,
                                                         const int* __restrict__ next,
                                                         const double2* __restrict__ itw,
                                                         double2* __restrict__ cols) {
    extern __shared__ double2 sm[];
    double2* a = sm;
    const int lc = rows_lc(log2pw), R = 1 << lc;
    const int y0 = blockIdx.x * R, p = blockIdx.y;
    const double2* fa = spec + (size_t)prev[p] * ph * pw;
    const double2* fb = spec + (size_t)next[p] * ph * pw;
    // XU elements per thread per round, all four 16-byte loads issued before the math so the
    // spectrum reads overlap instead of each stalling its own cross-power
    constexpr int XU = 2;
    const int ne = R << log2pw;
    for (int e0 = threadIdx.x; e0 < ne; e0 += XU * NT) {
        double2 A[XU], B[XU];
#pragma unroll
        for (int u = 0; u < XU; ++u) {
            const int e = e0 + u * NT, y = y0 + (e & (R - 1)), x = e >> lc;
            A[u] = B[u] = make_double2(0.0, 0.0);
            if (e < ne && y < ph) {
                A[u] = fa[(size_t)y * pw + x];
                B[u] = fb[(size_t)y * pw + x];
            }
        }
        // c = conj(A) * B (registration.hpp:61-65); |c| = std::abs -> glibc hypot; c / |c|.
        // All XU elements go through the branch-free fast paths first (their fp64 chains
        // interleave); an element a fast path flags is redone with the intrinsics.
        double2 rr[XU];
        bool ok[XU];
#pragma unroll
        for (int u = 0; u < XU; ++u) {
            const double nai = -A[u].y;
            const double re = dsub(dmul(A[u].x, B[u].x), dmul(nai, B[u].y));
            const double im = dadd(dmul(A[u].x, B[u].y), dmul(nai, B[u].x));
            bool okh, okx, oky;
            const double m = hypot_glibc_fast(re, im, okh);
            const bool big = m > 1e-12;
            const double mm = big ? m : 1.0;
            const double r2 = drcp_refined(mm);
            const double qx = ddiv_fast(re, mm, r2, okx), qy = ddiv_fast(im, mm, r2, oky);
            rr[u] = big ? make_double2(qx, qy) : make_double2(0.0, 0.0);
            ok[u] = okh && (!big || (okx && oky));
        }
#pragma unroll
        for (int u = 0; u < XU; ++u) {
            const int e = e0 + u * NT, r = e & (R - 1), x = e >> lc;
            if (e >= ne || y0 + r >= ph) continue;
            if (!ok[u]) {
                const double nai = -A[u].y;
                const double re = dsub(dmul(A[u].x, B[u].x), dmul(nai, B[u].y));
                const double im = dadd(dmul(A[u].x, B[u].y), dmul(nai, B[u].x));
                const double m = hypot_glibc(re, im);
                rr[u] = m > 1e-12 ? make_double2(ddiv(re, m), ddiv(im, m)) : make_double2(0.0, 0.0);
            }
            a[(PadX::at(brev(x, log2pw)) << lc) | r] = rr[u];
        }
    }
    __syncthreads();
    fft_stages<kQXpow, PadX>(a, pw, log2pw, lc, itw, M);  // only the 2M+1 wrapped columns are read
    const double inv = ddiv(1.0, (double)pw);
    const int nc = 2 * M + 1;
    for (int e = threadIdx.x; e < nc * R; e += NT) {
        const int r = e % R, ci = e / R;
        const int y = y0 + r;
        if (y >= ph) continue;
        const int dx = ci - M;
        const int x = dx < 0 ? dx + pw : dx;
        const double2 v = a[(PadX::at(x) << lc) | r];
        cols[((size_t)p * nc + ci) * ph + y] = make_double2(dmul(v.x, inv), dmul(v.y, inv));
    }
}

__global__ void __launch_bounds__(NT) k_inv_cols(int ph, int log2ph, int M,
                                                 const double2* __restrict__ cols,
                                                 const double2* __restrict__ itw,
                                                 double* __restrict__ surf) {
    extern __shared__ double2 sm[];
    double2* a = sm;
    const int ci = blockIdx.x, p = blockIdx.y;
    const int nc = 2 * M + 1;
    const double2* src = cols + ((size_t)p * nc + ci) * ph;
    for (int y = threadIdx.x; y < ph; y += NT) a[pd(brev(y, log2ph))] = src[y];
    __syncthreads();
    fft_stages<3>(a, ph, log2ph, 0, itw, M);  // only the 2M+1 wrapped rows are read
    const double inv = ddiv(1.0, (double)ph);
    for (int r = threadIdx.x; r < nc; r += NT) {
        const int dy = r - M;
        const int y = dy < 0 ? dy + ph : dy;
        surf[(size_t)p * nc * nc + (size_t)r * nc + ci] = dmul(a[pd(y)].x, inv);
    }
}

__global__ void __launch_bounds__(NT) k_argmax(int M, const double* __restrict__ surf,
                                               PairInfo* __restrict__ info) {
    const int p = blockIdx.x;
    const int nc = 2 * M + 1, n = nc * nc;
    const double* S = surf + (size_t)p * n;
    __shared__ double sv[NT];
    __shared__ int si[NT];
    // first strict maximum in scan order == maximum value, smallest index
    double bv = -1e300;
    int bi = 0x7fffffff;
    for (int i = threadIdx.x; i < n; i += NT) {
        const double v = S[i];
        if (v > bv) { bv = v; bi = i; }
    }
    sv[threadIdx.x] = bv;
    si[threadIdx.x] = bi;
    __syncthreads();
    for (int o = NT / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            const double ov = sv[threadIdx.x + o];
            const int oi = si[threadIdx.x + o];
            if (ov > sv[threadIdx.x] || (ov == sv[threadIdx.x] && oi < si[threadIdx.x])) {
                sv[threadIdx.x] = ov;
                si[threadIdx.x] = oi;
            }
        }
        __syncthreads();
    }
    const double best = sv[0];
    const int bidx = si[0];
    const int bdx = bidx % nc - M, bdy = bidx / nc - M;
    __syncthreads();
    double second = 0.0;
    for (int i = threadIdx.x; i < n; i += NT) {
        const int dx = i % nc - M, dy = i / nc - M;
        if (max(abs(dx - bdx), abs(dy - bdy)) <= 2) continue;
        const double v = S[i];
        second = (second < v) ? v : second;
    }
    sv[threadIdx.x] = second;
    __syncthreads();
    for (int o = NT / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            const double ov = sv[threadIdx.x + o];
            sv[threadIdx.x] = (sv[threadIdx.x] < ov) ? ov : sv[threadIdx.x];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        second = sv[0];
        PairInfo& I = info[p];
        if (best <= 0.0) {
            I.est_dx = 0;
            I.est_dy = 0;
            I.confidence = 1.0;
        } else {
            I.est_dx = bdx;
            I.est_dy = bdy;
            I.confidence = ddiv(best, (second < 1e-12) ? 1e-12 : second);
        }
        // extract_roi falls back to (0,0) below kShiftConfidenceThreshold (roi.hpp:333)
        const bool keep = !(I.confidence < 1.5);
        I.dx = keep ? I.est_dx : 0;
        I.dy = keep ? I.est_dy : 0;
        I.shifted = (I.dx != 0 || I.dy != 0);
    }
}

template <typename K>
void set_smem(K kernel, size_t bytes) {
    if (bytes > 48 * 1024)
        FROI_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
}

// log2 of the columns per CTA: 4 for 1024-row spectra (~70 KB of padded column data)
int column_lcb(const Geom& g) {
    int lcb = 12 - g.log2ph;
    if (lcb < 0) lcb = 0;
    if (lcb > 4) lcb = 4;
    while (lcb > 0 && (1 << lcb) > g.pw) --lcb;
    return lcb;
}

}  // namespace

void launch_fft_forward(const Geom& g, const void* d_den, const unsigned long long* d_sums,
                        const double* d_wx, const double* d_wy, const double2* d_tw_row,
                        const double2* d_tw_col, double2* d_spec, int n_slots, cudaStream_t s) {
    if (n_slots <= 0) return;
    const int lr = rows_lc(g.log2pw);
    size_t smem_r = sizeof(double2) * (((size_t)padded(g.pw) << lr) + g.pw);
    const int tw_r = smem_r <= kMaxCtaSmem;
    if (!tw_r) smem_r -= sizeof(double2) * g.pw;
    const int row_blocks = cdiv(g.ph, 1 << lr);
    static const bool rows_w = [] {
        const char* e = getenv("FROI_FFT_ROWS_W");
        return !(e && atoi(e) == 0);
    }();
    if (rows_w && g.pw == 1024) {
        const dim3 grid(cdiv(g.ph, RW_WARPS), n_slots);
        const size_t sm = sizeof(double2) * RW_WARPS * 33 * 32;
        if (g.sample_bytes == 1) {
            set_smem(k_fft_rows_w1024<uint8_t>, sm);
            k_fft_rows_w1024<uint8_t><<<grid, 32 * RW_WARPS, sm, s>>>(g.W, g.H, g.ph, (const uint8_t*)d_den, d_sums,
                                                                     d_wx, d_wy, d_tw_row, d_spec);
        } else {
            set_smem(k_fft_rows_w1024<uint16_t>, sm);
            k_fft_rows_w1024<uint16_t><<<grid, 32 * RW_WARPS, sm, s>>>(g.W, g.H, g.ph, (const uint16_t*)d_den, d_sums,
                                                                      d_wx, d_wy, d_tw_row, d_spec);
        }
    } else if (g.sample_bytes == 1) {
        set_smem(k_fft_rows_fwd<uint8_t>, smem_r);
        k_fft_rows_fwd<uint8_t><<<dim3(row_blocks, n_slots), NT, smem_r, s>>>(
            g.W, g.H, g.pw, g.ph, g.log2pw, tw_r, (const uint8_t*)d_den, d_sums, d_wx, d_wy, d_tw_row, d_spec);
    } else {
        set_smem(k_fft_rows_fwd<uint16_t>, smem_r);
        k_fft_rows_fwd<uint16_t><<<dim3(row_blocks, n_slots), NT, smem_r, s>>>(
            g.W, g.H, g.pw, g.ph, g.log2pw, tw_r, (const uint16_t*)d_den, d_sums, d_wx, d_wy, d_tw_row, d_spec);
    }
    FROI_LAUNCH_CHECK();
    const int lcb = column_lcb(g);
    size_t smem_c = sizeof(double2) * (((size_t)padded(g.ph) << lcb) + g.ph);
    const int tw_c = smem_c <= kMaxCtaSmem;
    if (!tw_c) smem_c -= sizeof(double2) * g.ph;
    set_smem(k_fft_cols, smem_c);
    k_fft_cols<<<dim3(g.pw >> lcb, n_slots), NT, smem_c, s>>>(g.pw, g.ph, g.log2ph, lcb, tw_c, d_tw_col, d_spec);
    FROI_LAUNCH_CHECK();
}

void launch_register_pairs(const Geom& g, const DevParams& p, const double2* d_spec,
                           const int* d_prev, const int* d_next, const double2* d_itw_row,
                           const double2* d_itw_col, double2* d_cols, double* d_surf,
                           PairInfo* d_info, int n_pairs, cudaStream_t s) {
    if (n_pairs <= 0) return;
    const int M = p.max_shift;
    const int lr = rows_lc(g.log2pw);
    const size_t smem_r = sizeof(double2) * ((size_t)padded_x(g.pw) << lr);
    set_smem(k_xpow_rows_inv, smem_r);
    k_xpow_rows_inv<<<dim3(cdiv(g.ph, 1 << lr), n_pairs), NT, smem_r, s>>>(g.pw, g.ph, g.log2pw, M, d_spec,
                                                                         d_prev, d_next, d_itw_row, d_cols);
    FROI_LAUNCH_CHECK();
    const size_t smem_c = sizeof(double2) * (size_t)padded(g.ph);
    set_smem(k_inv_cols, smem_c);
    k_inv_cols<<<dim3(2 * M + 1, n_pairs), NT, smem_c, s>>>(g.ph, g.log2ph, M, d_cols, d_itw_col, d_surf);
    FROI_LAUNCH_CHECK();
    k_argmax<<<n_pairs, NT, 0, s>>>(M, d_surf, d_info);
    FROI_LAUNCH_CHECK();
}

}  // namespace froi
