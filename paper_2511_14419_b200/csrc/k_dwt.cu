// k_dwt.cu — the codec side's first bandwidth-bound step on the GPU:
// reversible 5/3 DWT (dwt.hpp:113-171, canonical in-place layout, DC-shifted int32) and the RoI
// coefficient masks (map_mask_to_subbands, codec.hpp:152-171).  Integer lifting with
// whole-sample symmetric extension; `>>` on negative int32 is the arithmetic (floor) shift the
// reference relies on, so the coefficients are bit-identical.
//
//   k_dwt_dc      frame samples - 2^(depth-1) -> int32 grid (n frames)
//   k_dwt_rows    one CTA per row of the level's w x h region: line in shared memory, predict
//                 (odd samples) / update (even samples) in parallel, de-interleave on write-back
//   k_dwt_cols    one CTA per block of columns: the column block in shared memory, same lifting
//   k_dwt_*_inv   interleave, then the inverse lifting, levels coarse to fine
//   k_mask_level  one level of map_mask_to_subbands: 2x2 OR down-sampling fused with the square
//                 dilation (radius 2, clipped windows = outside unset)
#include "kernels.cuh"

namespace froi {
namespace {

constexpr int DNT = 256;

__device__ __forceinline__ int dwt_r(int i, int n) { return i + 1 < n ? i + 1 : n - 2; }
__device__ __forceinline__ int dwt_l(int i) { return i > 0 ? i - 1 : 1; }

// `ncol` interleaved lines of length n in shared memory, element i of line c at x[i*ncol + c]
__device__ __forceinline__ void lift_lines(int32_t* x, int n, int ncol, bool inverse) {
    if (n < 2) return;
    const int nodd = n / 2, neven = (n + 1) / 2;
    auto predict = [&](int sgn) {
        for (int t = threadIdx.x; t < nodd * ncol; t += blockDim.x) {
            const int c = t % ncol, i = 2 * (t / ncol) + 1;
            const int v = (x[(i - 1) * ncol + c] + x[dwt_r(i, n) * ncol + c]) >> 1;
            x[i * ncol + c] += sgn * v;
        }
        __syncthreads();
    };
    auto update = [&](int sgn) {
        for (int t = threadIdx.x; t < neven * ncol; t += blockDim.x) {
            const int c = t % ncol, i = 2 * (t / ncol);
            const int v = (x[dwt_l(i) * ncol + c] + x[dwt_r(i, n) * ncol + c] + 2) >> 2;
            x[i * ncol + c] += sgn * v;
        }
        __syncthreads();
    };
    if (!inverse) {
        predict(-1);
        update(1);
    } else {
        update(-1);
        predict(1);
    }
}

// position of element i after de-interleaving (evens to the front ceil(n/2), odds behind)
__device__ __forceinline__ int deint(int i, int n) { return (i & 1) ? (n + 1) / 2 + i / 2 : i / 2; }

template <typename T>
__global__ void __launch_bounds__(DNT) k_dwt_dc(const T* __restrict__ in, int32_t* __restrict__ g,
                                                long long n, int32_t dc) {
    const long long base = (long long)blockIdx.y * n;
    for (long long i = blockIdx.x * (long long)DNT + threadIdx.x; i < n; i += (long long)gridDim.x * DNT)
        g[base + i] = (int32_t)in[base + i] - dc;
}

__global__ void __launch_bounds__(DNT) k_dwt_rows(int32_t* g, int W, int H, int w, bool inverse) {
    extern __shared__ int32_t sline[];
    int32_t* row = g + (size_t)blockIdx.y * W * H + (size_t)blockIdx.x * W;
    for (int i = threadIdx.x; i < w; i += DNT) {
        if (!inverse) sline[i] = row[i];
        else sline[i] = row[deint(i, w)];  // interleave
    }
    __syncthreads();
    lift_lines(sline, w, 1, inverse);
    for (int i = threadIdx.x; i < w; i += DNT) {
        if (!inverse) row[deint(i, w)] = sline[i];
        else row[i] = sline[i];
    }
}

__global__ void __launch_bounds__(DNT) k_dwt_cols(int32_t* g, int W, int H, int w, int h, int cb,
                                                  bool inverse) {
    extern __shared__ int32_t scol[];  // [h][cb]
    int32_t* base = g + (size_t)blockIdx.y * W * H;
    const int c0 = blockIdx.x * cb, nc = min(cb, w - c0);
    for (int t = threadIdx.x; t < h * cb; t += DNT) {
        const int y = t / cb, c = t - y * cb;
        if (c < nc) scol[y * cb + c] = base[(size_t)(inverse ? deint(y, h) : y) * W + c0 + c];
    }
    __syncthreads();
    lift_lines(scol, h, cb, inverse);
    for (int t = threadIdx.x; t < h * cb; t += DNT) {
        const int y = t / cb, c = t - y * cb;
        if (c < nc) base[(size_t)(inverse ? y : deint(y, h)) * W + c0 + c] = scol[y * cb + c];
    }
}

template <typename T>
__global__ void __launch_bounds__(DNT) k_dwt_out(const int32_t* __restrict__ g, T* __restrict__ out,
                                                 long long n, int32_t dc, int32_t mx) {
    const long long base = (long long)blockIdx.y * n;
    for (long long i = blockIdx.x * (long long)DNT + threadIdx.x; i < n; i += (long long)gridDim.x * DNT) {
        const int32_t v = g[base + i] + dc;  // clamp_to_depth of an integer
        out[base + i] = (T)(v < 0 ? 0 : (v > mx ? mx : v));
    }
}

__global__ void __launch_bounds__(DNT) k_mask_level(const uint8_t* __restrict__ cur, int cw, int ch,
                                                    uint8_t* __restrict__ out, int nw, int nh, int dilate) {
    const int x = blockIdx.x * 32 + (threadIdx.x & 31), y = blockIdx.y * 8 + (threadIdx.x >> 5);
    if (x >= nw || y >= nh) return;
    const int r = dilate ? 2 : 0;
    uint8_t v = 0;
    for (int yy = max(0, y - r); yy <= min(nh - 1, y + r) && !v; ++yy)
        for (int xx = max(0, x - r); xx <= min(nw - 1, x + r) && !v; ++xx)
            for (int b = 0; b < 2; ++b)
                for (int a = 0; a < 2; ++a) {
                    const int sx = 2 * xx + a, sy = 2 * yy + b;
                    if (sx < cw && sy < ch && cur[(size_t)sy * cw + sx]) v = 1;
                }
    out[(size_t)y * nw + x] = v;
}

int dwt_extent(int n, int level) {
    for (int l = 0; l < level; ++l) n = (n + 1) / 2;
    return n;
}

int col_block(int h) {
    int cb = 32;
    while (cb > 1 && (size_t)h * cb * sizeof(int32_t) > 96 * 1024) cb >>= 1;
    return cb;
}

void set_dwt_smem(int W, int H) {
    const size_t rs = sizeof(int32_t) * (size_t)W, cs = sizeof(int32_t) * (size_t)H * col_block(H);
    if (rs > 48 * 1024) FROI_CUDA(cudaFuncSetAttribute(k_dwt_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rs));
    if (cs > 48 * 1024) FROI_CUDA(cudaFuncSetAttribute(k_dwt_cols, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cs));
}

void dwt_levels_run(int32_t* g, int W, int H, int levels, int n, bool inverse, cudaStream_t s) {
    set_dwt_smem(W, H);
    for (int k = 0; k < levels; ++k) {
        const int l = inverse ? levels - 1 - k : k;
        const int w = dwt_extent(W, l), h = dwt_extent(H, l), cb = col_block(h);
        const dim3 rg(h, n), cg(cdiv(w, cb), n);
        if (!inverse) {
            k_dwt_rows<<<rg, DNT, sizeof(int32_t) * w, s>>>(g, W, H, w, false);
            k_dwt_cols<<<cg, DNT, sizeof(int32_t) * h * cb, s>>>(g, W, H, w, h, cb, false);
        } else {
            k_dwt_cols<<<cg, DNT, sizeof(int32_t) * h * cb, s>>>(g, W, H, w, h, cb, true);
            k_dwt_rows<<<rg, DNT, sizeof(int32_t) * w, s>>>(g, W, H, w, true);
        }
        FROI_LAUNCH_CHECK();
    }
}

}  // namespace

void launch_dwt_forward(const void* d_frames, int sample_bytes, int W, int H, int depth, int n,
                        int levels, int32_t* d_coeffs, cudaStream_t s) {
    const long long px = (long long)W * H;
    const dim3 eg((unsigned)std::min<long long>(cdiv<long long>(px, DNT), 1024), n);
    if (sample_bytes == 1)
        k_dwt_dc<uint8_t><<<eg, DNT, 0, s>>>((const uint8_t*)d_frames, d_coeffs, px, 1 << (depth - 1));
    else
        k_dwt_dc<uint16_t><<<eg, DNT, 0, s>>>((const uint16_t*)d_frames, d_coeffs, px, 1 << (depth - 1));
    FROI_LAUNCH_CHECK();
    dwt_levels_run(d_coeffs, W, H, levels, n, false, s);
}

void launch_dwt_inverse(int32_t* d_coeffs, int W, int H, int depth, int n, int levels,
                        uint16_t* d_frames, cudaStream_t s) {
    dwt_levels_run(d_coeffs, W, H, levels, n, true, s);
    const long long px = (long long)W * H;
    const dim3 eg((unsigned)std::min<long long>(cdiv<long long>(px, DNT), 1024), n);
    k_dwt_out<uint16_t><<<eg, DNT, 0, s>>>(d_coeffs, d_frames, px, 1 << (depth - 1),
                                           (int32_t)((1u << depth) - 1u));
    FROI_LAUNCH_CHECK();
}

size_t launch_map_mask_to_subbands(const uint8_t* d_mask, int W, int H, int levels, bool any,
                                   uint8_t* d_out, cudaStream_t s) {
    const uint8_t* cur = d_mask;
    int cw = W, ch = H;
    size_t off = 0;
    for (int l = 1; l <= levels; ++l) {
        const int nw = (cw + 1) / 2, nh = (ch + 1) / 2;
        k_mask_level<<<dim3(cdiv(nw, 32), cdiv(nh, 8)), DNT, 0, s>>>(cur, cw, ch, d_out + off, nw, nh,
                                                                   any ? 1 : 0);
        FROI_LAUNCH_CHECK();
        cur = d_out + off;
        cw = nw;
        ch = nh;
        off += (size_t)nw * nh;
    }
    return off;
}

}  // namespace froi
