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

// In-place radix-2 stages over `ncol` interleaved transforms of length n (element i of
// transform c at a[i*ncol + c]); input already bit-reversed.  tw: stage with half-length h
// uses tw[h-1 .. 2h-2] (the reference's w sequence for len = 2h).  Two consecutive stages are
// fused per pass on groups {i, i+h, i+2h, i+3h} held in registers: the butterflies and their
// operands are exactly the reference's, only the number of shared-memory round trips halves.
__device__ __forceinline__ void fft_stages(double2* a, int n, int log2n, int ncol,
                                           const double2* tw) {
    int s = 0;
    for (; s + 1 < log2n; s += 2) {
        const int h = 1 << s;
        const int ng = (n >> 2) * ncol;
        for (int j = threadIdx.x; j < ng; j += blockDim.x) {
            const int c = j % ncol;
            const int b = j / ncol;
            const int k = b & (h - 1);
            const int i = ((b >> s) << (s + 2)) + k;
            double2* p0 = a + i * ncol + c;
            double2 e0 = p0[0], e1 = p0[h * ncol], e2 = p0[2 * h * ncol], e3 = p0[3 * h * ncol];
            const double2 w1 = tw[h - 1 + k];
            bfly(e0, e1, w1);
            bfly(e2, e3, w1);
            bfly(e0, e2, tw[2 * h - 1 + k]);
            bfly(e1, e3, tw[2 * h - 1 + k + h]);
            p0[0] = e0;
            p0[h * ncol] = e1;
            p0[2 * h * ncol] = e2;
            p0[3 * h * ncol] = e3;
        }
        __syncthreads();
    }
    if (s < log2n) {  // odd log2n: one trailing radix-2 stage
        const int h = 1 << s;
        const int nb = (n >> 1) * ncol;
        for (int j = threadIdx.x; j < nb; j += blockDim.x) {
            const int c = j % ncol;
            const int b = j / ncol;
            const int k = b & (h - 1);
            const int i1 = ((b >> s) << (s + 1)) + k;
            double2 u = a[i1 * ncol + c], v = a[(i1 + h) * ncol + c];
            bfly(u, v, tw[h - 1 + k]);
            a[i1 * ncol + c] = u;
            a[(i1 + h) * ncol + c] = v;
        }
        __syncthreads();
    }
}

template <typename T>
__global__ void __launch_bounds__(NT) k_fft_rows_fwd(int W, int H, int pw, int ph, int log2pw,
                                                     const T* __restrict__ den,
                                                     const unsigned long long* __restrict__ sums,
                                                     const double* __restrict__ wx,
                                                     const double* __restrict__ wy,
                                                     const double2* __restrict__ tw,
                                                     double2* __restrict__ spec) {
    extern __shared__ double2 sm[];
    double2* a = sm;
    double2* tws = sm + pw;
    const int y = blockIdx.x, slot = blockIdx.y;
    const T* f = den + (size_t)slot * W * H;
    // windowed_spectrum_input (registration.hpp:26-42): exact integer sum, then one division
    const double mean = ddiv((double)sums[slot], (double)((long long)W * H));
    const int sy = min(y, H - 1);
    const double wyv = wy[y];
    for (int x = threadIdx.x; x < pw; x += NT) {
        const int sx = min(x, W - 1);
        const double v = dmul(dmul(dsub((double)f[(size_t)sy * W + sx], mean), wx[x]), wyv);
        a[brev(x, log2pw)] = make_double2(v, 0.0);
    }
    for (int i = threadIdx.x; i < pw - 1; i += NT) tws[i] = tw[i];
    __syncthreads();
    fft_stages(a, pw, log2pw, 1, tws);
    double2* out = spec + ((size_t)slot * ph + y) * pw;
    for (int x = threadIdx.x; x < pw; x += NT) out[x] = a[x];
}

__global__ void __launch_bounds__(NT) k_fft_cols(int pw, int ph, int log2ph, int cb,
                                                 const double2* __restrict__ tw,
                                                 double2* __restrict__ spec) {
    extern __shared__ double2 sm[];
    double2* a = sm;
    double2* tws = sm + (size_t)ph * cb;
    const int slot = blockIdx.y, c0 = blockIdx.x * cb;
    double2* base = spec + (size_t)slot * ph * pw + c0;
    for (int i = threadIdx.x; i < ph * cb; i += NT) {
        const int r = i / cb, c = i - r * cb;
        a[brev(r, log2ph) * cb + c] = base[(size_t)r * pw + c];
    }
    for (int i = threadIdx.x; i < ph - 1; i += NT) tws[i] = tw[i];
    __syncthreads();
    fft_stages(a, ph, log2ph, cb, tws);
    for (int i = threadIdx.x; i < ph * cb; i += NT) {
        const int r = i / cb, c = i - r * cb;
        base[(size_t)r * pw + c] = a[r * cb + c];
    }
}

__global__ void __launch_bounds__(NT) k_xpow_rows_inv(int pw, int ph, int log2pw, int M,
                                                      const double2* __restrict__ spec,
                                                      const int* __restrict__ prev,
                                                      const int* __restrict__ next,
                                                      const double2* __restrict__ itw,
                                                      double2* __restrict__ cols) {
    extern __shared__ double2 sm[];
    double2* a = sm;
    double2* tws = sm + pw;
    const int y = blockIdx.x, p = blockIdx.y;
    const double2* fa = spec + ((size_t)prev[p] * ph + y) * pw;
    const double2* fb = spec + ((size_t)next[p] * ph + y) * pw;
    for (int x = threadIdx.x; x < pw; x += NT) {
        const double2 A = fa[x], B = fb[x];
        // c = conj(A) * B (registration.hpp:61-65); |c| = std::abs -> glibc hypot
        const double nai = -A.y;
        const double re = dsub(dmul(A.x, B.x), dmul(nai, B.y));
        const double im = dadd(dmul(A.x, B.y), dmul(nai, B.x));
        const double m = hypot_glibc(re, im);
        double2 r = make_double2(0.0, 0.0);
        if (m > 1e-12) r = make_double2(ddiv(re, m), ddiv(im, m));
        a[brev(x, log2pw)] = r;
    }
    for (int i = threadIdx.x; i < pw - 1; i += NT) tws[i] = itw[i];
    __syncthreads();
    fft_stages(a, pw, log2pw, 1, tws);
    const double inv = ddiv(1.0, (double)pw);
    const int nc = 2 * M + 1;
    for (int ci = threadIdx.x; ci < nc; ci += NT) {
        const int dx = ci - M;
        const int x = dx < 0 ? dx + pw : dx;
        const double2 v = a[x];
        cols[((size_t)p * nc + ci) * ph + y] = make_double2(dmul(v.x, inv), dmul(v.y, inv));
    }
}

__global__ void __launch_bounds__(NT) k_inv_cols(int ph, int log2ph, int M,
                                                 const double2* __restrict__ cols,
                                                 const double2* __restrict__ itw,
                                                 double* __restrict__ surf) {
    extern __shared__ double2 sm[];
    double2* a = sm;
    double2* tws = sm + ph;
    const int ci = blockIdx.x, p = blockIdx.y;
    const int nc = 2 * M + 1;
    const double2* src = cols + ((size_t)p * nc + ci) * ph;
    for (int y = threadIdx.x; y < ph; y += NT) a[brev(y, log2ph)] = src[y];
    for (int i = threadIdx.x; i < ph - 1; i += NT) tws[i] = itw[i];
    __syncthreads();
    fft_stages(a, ph, log2ph, 1, tws);
    const double inv = ddiv(1.0, (double)ph);
    for (int r = threadIdx.x; r < nc; r += NT) {
        const int dy = r - M;
        const int y = dy < 0 ? dy + ph : dy;
        surf[(size_t)p * nc * nc + (size_t)r * nc + ci] = dmul(a[y].x, inv);
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

int column_block(const Geom& g) {
    int cb = 4096 / g.ph;  // 64 KB of column data per CTA
    if (cb < 1) cb = 1;
    if (cb > g.pw) cb = g.pw;
    return cb;
}

}  // namespace

void launch_fft_forward(const Geom& g, const void* d_den, const unsigned long long* d_sums,
                        const double* d_wx, const double* d_wy, const double2* d_tw_row,
                        const double2* d_tw_col, double2* d_spec, int n_slots, cudaStream_t s) {
    if (n_slots <= 0) return;
    const size_t smem_r = sizeof(double2) * (2 * (size_t)g.pw);
    if (g.sample_bytes == 1) {
        set_smem(k_fft_rows_fwd<uint8_t>, smem_r);
        k_fft_rows_fwd<uint8_t><<<dim3(g.ph, n_slots), NT, smem_r, s>>>(
            g.W, g.H, g.pw, g.ph, g.log2pw, (const uint8_t*)d_den, d_sums, d_wx, d_wy, d_tw_row, d_spec);
    } else {
        set_smem(k_fft_rows_fwd<uint16_t>, smem_r);
        k_fft_rows_fwd<uint16_t><<<dim3(g.ph, n_slots), NT, smem_r, s>>>(
            g.W, g.H, g.pw, g.ph, g.log2pw, (const uint16_t*)d_den, d_sums, d_wx, d_wy, d_tw_row, d_spec);
    }
    FROI_LAUNCH_CHECK();
    const int cb = column_block(g);
    const size_t smem_c = sizeof(double2) * ((size_t)g.ph * cb + g.ph);
    set_smem(k_fft_cols, smem_c);
    k_fft_cols<<<dim3(g.pw / cb, n_slots), NT, smem_c, s>>>(g.pw, g.ph, g.log2ph, cb, d_tw_col, d_spec);
    FROI_LAUNCH_CHECK();
}

void launch_register_pairs(const Geom& g, const DevParams& p, const double2* d_spec,
                           const int* d_prev, const int* d_next, const double2* d_itw_row,
                           const double2* d_itw_col, double2* d_cols, double* d_surf,
                           PairInfo* d_info, int n_pairs, cudaStream_t s) {
    if (n_pairs <= 0) return;
    const int M = p.max_shift;
    const size_t smem_r = sizeof(double2) * (2 * (size_t)g.pw);
    set_smem(k_xpow_rows_inv, smem_r);
    k_xpow_rows_inv<<<dim3(g.ph, n_pairs), NT, smem_r, s>>>(g.pw, g.ph, g.log2pw, M, d_spec, d_prev,
                                                            d_next, d_itw_row, d_cols);
    FROI_LAUNCH_CHECK();
    const size_t smem_c = sizeof(double2) * (2 * (size_t)g.ph);
    set_smem(k_inv_cols, smem_c);
    k_inv_cols<<<dim3(2 * M + 1, n_pairs), NT, smem_c, s>>>(g.ph, g.log2ph, M, d_cols, d_itw_col, d_surf);
    FROI_LAUNCH_CHECK();
    k_argmax<<<n_pairs, NT, 0, s>>>(M, d_surf, d_info);
    FROI_LAUNCH_CHECK();
}

}  // namespace froi
