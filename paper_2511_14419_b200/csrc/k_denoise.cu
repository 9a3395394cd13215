// k_denoise.cu — fused median + bilateral denoise (denoise.hpp:28-90), bit-exact.
//
// k_denoise_u8_m1b2 (the default radii on 8-bit frames): persistent CTAs over 32x32 tiles, the
// next tile's raw pixels in flight; medians from sorted row triples; the 5x5 bilateral window in
// registers.  k_denoise (other radii, 16-bit): one CTA per 32x16 output tile, raw tile (halo =
// median radius + bilateral radius, edge-replicated) and median tile (halo = bilateral radius)
// in shared memory.  Both: bilateral sums in fp64 in the reference's dy-major / dx-minor order
// with explicit round-to-nearest operations (no FMA), the host-computed libm range LUT and
// spatial weights, rounding as std::lround (half away from zero); the CTA also reduces the
// integer sum of its denoised pixels for the registration mean (registration.hpp:27-29), exact
// in integers.
//
// Bound: the fp64 pipe, not HBM.  The byte model (SURVEY.md App. C row "D") is 2 B/px, which
// the kernel moves at ~70 GB/s; its ~118 fp64 instructions per pixel (4 per bilateral tap: the
// weight product, two sums and the weighted sample) run at ~44 % of the measured fp64 peak
// (profiles/fp64_work.json, profiles/r02_fp64.md).
#include "kernels.cuh"

namespace froi {
namespace {

constexpr int TX = 32, TY = 16, NT = 256;  // 2 output rows per thread

__device__ __forceinline__ void cswap(int& a, int& b) {
    const int t = min(a, b);
    b = max(a, b);
    a = t;
}

// Median of 9 by the classic 19-exchange selection network (exact for integers).
__device__ __forceinline__ int median9(int p0, int p1, int p2, int p3, int p4, int p5, int p6,
                                       int p7, int p8) {
    cswap(p1, p2); cswap(p4, p5); cswap(p7, p8); cswap(p0, p1); cswap(p3, p4); cswap(p6, p7);
    cswap(p1, p2); cswap(p4, p5); cswap(p7, p8); cswap(p0, p3); cswap(p5, p8); cswap(p4, p7);
    cswap(p3, p6); cswap(p1, p4); cswap(p2, p5); cswap(p4, p7); cswap(p4, p2); cswap(p6, p4);
    cswap(p4, p2);
    return p4;
}

struct Spatial {
    double w[225];  // (2*7+1)^2 spatial weights, host-computed libm values
};

// MR/BR > 0: compile-time radii (the default 1/2 path); 0: runtime radii.
template <typename T, int MR, int BR>
__global__ void __launch_bounds__(NT) k_denoise(int W, int H, int maxval, int enabled, int mr_rt,
                                                 int br_rt, const void* const* frame_raw, T* den,
                                                 unsigned long long* sums, const __grid_constant__ Spatial sp_w,
                                                 const double* lut_g) {
    const int mr = MR > 0 ? MR : mr_rt;
    const int br = BR > 0 ? BR : br_rt;
    extern __shared__ __align__(16) unsigned char smem[];
    const int slot = blockIdx.z;
    const T* src = (const T*)frame_raw[slot];
    T* dst = den + (size_t)slot * W * H;
    const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
    const int tid = threadIdx.y * TX + threadIdx.x;
    const int R1 = mr + br;
    const int rw = TX + 2 * R1, rh = TY + 2 * R1;
    const int mw = TX + 2 * br, mh = TY + 2 * br;
    const int side = 2 * br + 1;
    double* spat_s = (double*)smem;                 // side*side
    double* lut_s = spat_s + side * side;           // 256 (u8 only)
    const bool lut_in_smem = sizeof(T) == 1;
    double* medd_s = lut_s + (lut_in_smem ? 256 : 0);  // median tile as double (converted once)
    int* raw_s = (int*)(medd_s + mw * mh);
    int* med_s = raw_s + rw * rh;

    unsigned long long sum = 0;
    if (!enabled) {
        for (int r = 0; r < TY; r += NT / TX) {
            const int x = x0 + threadIdx.x, y = y0 + threadIdx.y + r;
            if (x < W && y < H) {
                const int v = src[(size_t)y * W + x];
                dst[(size_t)y * W + x] = (T)v;
                sum += (unsigned long long)v;
            }
        }
    } else {
        for (int i = tid; i < side * side; i += NT) spat_s[i] = sp_w.w[i];
        if (lut_in_smem)
            for (int i = tid; i < 256; i += NT) lut_s[i] = lut_g[i];
        for (int i = tid; i < rw * rh; i += NT) {
            const int ry = i / rw, rx = i - ry * rw;
            const int gy = clampi(y0 - R1 + ry, 0, H - 1), gx = clampi(x0 - R1 + rx, 0, W - 1);
            raw_s[i] = src[(size_t)gy * W + gx];
        }
        __syncthreads();
        // median at clamped coordinates: med_s[X - (x0-br)] = median(clamp(X)) (denoise.hpp:32-43)
        for (int i = tid; i < mw * mh; i += NT) {
            const int my = i / mw, mx = i - my * mw;
            const int cx = clampi(x0 - br + mx, 0, W - 1), cy = clampi(y0 - br + my, 0, H - 1);
            const int rx = cx - (x0 - R1), ry = cy - (y0 - R1);
            int m;
            if (mr == 1) {
                const int* r0 = raw_s + (ry - 1) * rw + rx;
                const int* r1 = r0 + rw;
                const int* r2 = r1 + rw;
                m = median9(r0[-1], r0[0], r0[1], r1[-1], r1[0], r1[1], r2[-1], r2[0], r2[1]);
            } else {
                // order statistic n/2 by rank counting (exact, any radius)
                const int n = (2 * mr + 1) * (2 * mr + 1), k = n / 2;
                m = 0;
                for (int a = 0; a < n; ++a) {
                    const int va = raw_s[(ry + a / (2 * mr + 1) - mr) * rw + rx + a % (2 * mr + 1) - mr];
                    int lt = 0, le = 0;
                    for (int b = 0; b < n; ++b) {
                        const int vb = raw_s[(ry + b / (2 * mr + 1) - mr) * rw + rx + b % (2 * mr + 1) - mr];
                        lt += vb < va;
                        le += vb <= va;
                    }
                    if (lt <= k && k < le) { m = va; break; }
                }
            }
            med_s[i] = m;
            medd_s[i] = (double)m;
        }
        __syncthreads();
        for (int r = 0; r < TY; r += NT / TX) {
            const int ty = threadIdx.y + r;
            const int x = x0 + threadIdx.x, y = y0 + ty;
            if (x < W && y < H) {
                // bilateral_filter (denoise.hpp:63-79): fp64, dy-major / dx-minor, no FMA
                const int c = med_s[(ty + br) * mw + threadIdx.x + br];
                double num = 0.0, dn = 0.0;
                if (BR > 0) {
#pragma unroll
                    for (int dy = -BR; dy <= BR; ++dy) {
                        const int* row = med_s + (ty + BR + dy) * mw + threadIdx.x + BR;
                        const double* rowd = medd_s + (ty + BR + dy) * mw + threadIdx.x + BR;
#pragma unroll
                        for (int dx = -BR; dx <= BR; ++dx) {
                            const int d = abs(row[dx] - c);
                            const double lw = lut_in_smem ? lut_s[d] : __ldg(lut_g + d);
                            const double wgt = dmul(sp_w.w[(dy + BR) * (2 * BR + 1) + dx + BR], lw);
                            num = dadd(num, dmul(wgt, rowd[dx]));
                            dn = dadd(dn, wgt);
                        }
                    }
                } else {
                    for (int dy = -br; dy <= br; ++dy) {
                        const int* row = med_s + (ty + br + dy) * mw + threadIdx.x + br;
                        const double* rowd = medd_s + (ty + br + dy) * mw + threadIdx.x + br;
                        const double* sp = spat_s + (dy + br) * side + br;
                        for (int dx = -br; dx <= br; ++dx) {
                            const int d = abs(row[dx] - c);
                            const double lw = lut_in_smem ? lut_s[d] : __ldg(lut_g + d);
                            const double wgt = dmul(sp[dx], lw);
                            num = dadd(num, dmul(wgt, rowd[dx]));
                            dn = dadd(dn, wgt);
                        }
                    }
                }
                double q = ddiv(num, dn);
                q = (q < 0.0) ? 0.0 : q;
                q = ((double)maxval < q) ? (double)maxval : q;
                const int outv = (int)round(q);
                dst[(size_t)y * W + x] = (T)outv;
                sum += (unsigned long long)outv;
            }
        }
    }
    // integer sum of the denoised tile for the registration mean
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_down_sync(0xffffffffu, sum, o);
    if ((tid & 31) == 0 && sum) atomicAdd(sums + slot, sum);
}

// 8-bit frames, median radius 1, bilateral radius 2 (the defaults).  A persistent CTA walks
// 32x32 tiles with the next tile's raw pixels in flight in registers.
//   median     each thread walks a column of the median tile: every raw row triple is sorted
//              once (min3 / max3 / sum) and the 3x3 median is med3(max of lows, med3 of mids,
//              min of highs) over the last three sorted triples (exact for integers).
//   bilateral  each thread filters 4 consecutive rows of one column from a 5x5 register window
//              (circular, 5 new medians per output), with the range weights in a 16-way
//              replicated table indexed by the signed difference (lane & 15 picks the copy, so a
//              warp's 64-bit lookups never bank-conflict beyond the 2-wavefront minimum).
// Same fp64 operations in the same order as k_denoise.
constexpr int QX = 32, QY = 32, QNT = 256, QRPT = QY / (QNT / QX), QREP = 16;
constexpr int QRW = QX + 6, QRH = QY + 6, QMW = QX + 4, QMH = QY + 4;

size_t qsmem_bytes() {
    return sizeof(double) * (511 * QREP) + sizeof(int) * QMW * QMH + sizeof(uint8_t) * QRW * QRH;
}

__device__ __forceinline__ int med3i(int a, int b, int c) {
    return a + b + c - min(min(a, b), c) - max(max(a, b), c);
}

__global__ void __launch_bounds__(QNT, 3) k_denoise_u8_m1b2(int W, int H, int maxval, int n_slots,
                                                            const void* const* frame_raw, uint8_t* den,
                                                            unsigned long long* sums,
                                                            const __grid_constant__ Spatial sp_w,
                                                            const double* lut_g) {
    constexpr int R1 = 3;
    extern __shared__ __align__(16) unsigned char smem[];
    double* lut_s = (double*)smem;                  // [511][QREP], index d + 255
    int* med_s = (int*)(lut_s + 511 * QREP);        // QMH * QMW medians * (QREP * 8)
    uint8_t* raw_s = (uint8_t*)(med_s + QMW * QMH); // QRH * QRW samples
    const int tid = threadIdx.y * QX + threadIdx.x;
    for (int i = tid; i < 511 * QREP; i += QNT) lut_s[i] = lut_g[min(abs(i / QREP - 255), maxval)];
    // byte address of this lane's copy of entry d = 0; + (m_n - m_c) * QREP * 8 selects d
    const char* lut0 = (const char*)(lut_s + 255 * QREP + (threadIdx.x & (QREP - 1)));
    const int tiles_x = (W + QX - 1) / QX, tiles_y = (H + QY - 1) / QY;
    const int per_slot = tiles_x * tiles_y;
    const double B52 = 4503599627370496.0;
    const int n_tiles = per_slot * n_slots;
    constexpr int NRAW = (QRW * QRH + QNT - 1) / QNT;
    // this thread's raw-tile positions are the same for every tile: (ry, rx) packed once
    int rpos[NRAW], roff[NRAW];
#pragma unroll
    for (int k = 0; k < NRAW; ++k) {
        const int i = tid + k * QNT, ry = i / QRW;
        rpos[k] = i < QRW * QRH ? (ry << 16) | (i - ry * QRW) : -1;
        roff[k] = ry * W + (i - ry * QRW);
    }
    auto fetch = [&](int t, int* v) {
        const int slot = t / per_slot, tr = t - slot * per_slot;
        const int by = tr / tiles_x, bx = tr - by * tiles_x;
        const uint8_t* src = (const uint8_t*)frame_raw[slot];
        const int gy0 = by * QY - R1, gx0 = bx * QX - R1;
        if (gx0 >= 0 && gy0 >= 0 && gx0 + QRW <= W && gy0 + QRH <= H) {  // no clamping
            const uint8_t* s0 = src + gy0 * W + gx0;
#pragma unroll
            for (int k = 0; k < NRAW; ++k) v[k] = rpos[k] >= 0 ? __ldg(s0 + roff[k]) : 0;
            return;
        }
#pragma unroll
        for (int k = 0; k < NRAW; ++k) {
            v[k] = 0;
            if (rpos[k] >= 0) {
                const int gy = clampi(gy0 + (rpos[k] >> 16), 0, H - 1);
                const int gx = clampi(gx0 + (rpos[k] & 0xffff), 0, W - 1);
                v[k] = __ldg(src + gy * W + gx);
            }
        }
    };
    int rv[NRAW];
    if (blockIdx.x < n_tiles) fetch(blockIdx.x, rv);
    const int lane = threadIdx.x, grp = threadIdx.y;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const int slot = t / per_slot, tr = t - slot * per_slot;
        const int by = tr / tiles_x, bx = tr - by * tiles_x;
        const int x0 = bx * QX, y0 = by * QY;
        __syncthreads();  // previous tile's bilateral is done with med_s
#pragma unroll
        for (int k = 0; k < NRAW; ++k)
            if (tid + k * QNT < QRW * QRH) raw_s[tid + k * QNT] = (uint8_t)rv[k];
        __syncthreads();
        if (t + (int)gridDim.x < n_tiles) fetch(t + gridDim.x, rv);  // in flight during this tile
        // medians at clamped centres (denoise.hpp:32-43): thread -> (column tid % QMW, run of
        // rows (tid / QMW) * QMH / 7 ..), one sliding window of sorted row triples per run
        if (tid < 7 * QMW) {
            const int mx = tid % QMW, mg = tid / QMW;
            const int cx = clampi(x0 - 2 + mx, 0, W - 1) - (x0 - R1);  // raw_s column of the centre
            const int rb = mg * QMH / 7, re = (mg + 1) * QMH / 7;
            // sorted triple of raw_s row r around the centre column
            auto tri = [&](int r, int& l, int& md, int& h) {
                const uint8_t* q = raw_s + r * QRW + cx;
                const int a = q[-1], b = q[0], c = q[1];
                l = min(min(a, b), c);
                h = max(max(a, b), c);
                md = a + b + c - l - h;
            };
            if (y0 - 2 >= 0 && y0 + QY + 2 <= H) {
                // interior band: median row my is centred on raw row my + 1, so the window slides
                // by exactly one raw row per output -- straight-line, constant row offsets
                const uint8_t* q = raw_s + rb * QRW + cx;
                int l0, m0, h0, l1, m1, h1;
                auto tq = [&](const uint8_t* r, int& l, int& md, int& h) {
                    const int a = r[-1], b = r[0], c = r[1];
                    l = min(min(a, b), c);
                    h = max(max(a, b), c);
                    md = a + b + c - l - h;
                };
                tq(q, l0, m0, h0);
                tq(q + QRW, l1, m1, h1);
                int* out = med_s + rb * QMW + mx;
                const int nrow = re - rb;  // 5 or 6
#pragma unroll
                for (int k = 0; k < 6; ++k) {
                    if (k < nrow) {
                        int l2, m2, h2;
                        tq(q + (k + 2) * QRW, l2, m2, h2);
                        const int m = med3i(max(max(l0, l1), l2), med3i(m0, m1, m2), min(min(h0, h1), h2));
                        out[k * QMW] = m * (QREP * 8);
                        l0 = l1; m0 = m1; h0 = h1;
                        l1 = l2; m1 = m2; h1 = h2;
                    }
                }
            } else {
            // the clamped centre row advances by 0 or 1 per median row
            int prev = clampi(y0 - 2 + rb, 0, H - 1) - (y0 - R1);
            int l0, m0, h0, l1, m1, h1, l2, m2, h2;
            tri(prev - 1, l0, m0, h0);
            tri(prev, l1, m1, h1);
            tri(prev + 1, l2, m2, h2);
            int m = med3i(max(max(l0, l1), l2), med3i(m0, m1, m2), min(min(h0, h1), h2));
            for (int my = rb; my < re; ++my) {
                const int cy = clampi(y0 - 2 + my, 0, H - 1) - (y0 - R1);
                if (cy != prev) {
                    l0 = l1; m0 = m1; h0 = h1;
                    l1 = l2; m1 = m2; h1 = h2;
                    tri(cy + 1, l2, m2, h2);
                    m = med3i(max(max(l0, l1), l2), med3i(m0, m1, m2), min(min(h0, h1), h2));
                    prev = cy;
                }
                med_s[my * QMW + mx] = m * (QREP * 8);
            }
            }
        }
        __syncthreads();
        const int ty0 = grp * QRPT;
        // NR output rows per pass, their 2*NR accumulation chains interleaved: window rows
        // ty0+r .. ty0+r+NR+3 are walked once; output row r+k takes j = k..k+4, each in the
        // reference's dy-major / dx-minor order, and each median is converted to double once
        // for all of them (2^52 bias, one DADD).
        constexpr int NR = 4;
        unsigned long long sum = 0;
        const double dmax = (double)maxval;
#pragma unroll
        for (int r = 0; r < QRPT; r += NR) {
            int mw[NR + 4][5];
#pragma unroll
            for (int j = 0; j < NR + 4; ++j)
#pragma unroll
                for (int dx = 0; dx < 5; ++dx) mw[j][dx] = med_s[(ty0 + r + j) * QMW + lane + dx];
            const char* lc[NR];
            double num[NR], dn[NR];
#pragma unroll
            for (int k = 0; k < NR; ++k) {
                lc[k] = lut0 - mw[k + 2][2];
                num[k] = 0.0;
                dn[k] = 0.0;
            }
#pragma unroll
            for (int j = 0; j < NR + 4; ++j)
#pragma unroll
                for (int dx = 0; dx < 5; ++dx) {
                    // 128 * median (the stored table offset) as a double: every product and sum
                    // below is then exactly 128x the reference's (power-of-two scaling commutes
                    // with round-to-nearest while nothing is subnormal), undone after the division
                    const double v = dsub(__hiloint2double(0x43300000, mw[j][dx]), B52);
#pragma unroll
                    for (int k = 0; k < NR; ++k) {
                        if (j < k || j > k + 4) continue;
                        const double w = dmul(sp_w.w[(j - k) * 5 + dx], *(const double*)(lc[k] + mw[j][dx]));
                        num[k] = dadd(num[k], dmul(w, v));
                        dn[k] = dadd(dn[k], w);
                    }
                }
#pragma unroll
            for (int k = 0; k < NR; ++k) {
                double q = dmul(ddiv(num[k], dn[k]), 1.0 / (QREP * 8));
                q = (q < 0.0) ? 0.0 : q;
                q = (dmax < q) ? dmax : q;
                const int outv = (int)round(q);
                const int x = x0 + lane, y = y0 + ty0 + r + k;
                if (x < W && y < H) {
                    den[(size_t)slot * W * H + (size_t)y * W + x] = (uint8_t)outv;
                    sum += (unsigned long long)outv;
                }
            }
        }
        for (int o = 16; o > 0; o >>= 1) sum += __shfl_down_sync(0xffffffffu, sum, o);
        if ((tid & 31) == 0 && sum) atomicAdd(sums + slot, sum);
    }
}

}  // namespace

void launch_denoise(const Geom& g, const DevParams& p, const void** d_frame_raw, void* d_den,
                    unsigned long long* d_sums, const double* h_spatial, const double* d_lut,
                    int n_slots, cudaStream_t s) {
    if (n_slots <= 0) return;
    const int mr = p.median_radius, br = p.bilateral_radius;
    const int R1 = mr + br, side = 2 * br + 1;
    const size_t smem = sizeof(double) * (side * side + (g.sample_bytes == 1 ? 256 : 0) +
                                          (TX + 2 * br) * (TY + 2 * br)) +
                        sizeof(int) * ((TX + 2 * R1) * (TY + 2 * R1) + (TX + 2 * br) * (TY + 2 * br));
    dim3 grid(cdiv(g.W, TX), cdiv(g.H, TY), n_slots), block(TX, NT / TX);
    Spatial sp{};
    for (int i = 0; i < side * side; ++i) sp.w[i] = h_spatial[i];
    const bool fast = mr == 1 && br == 2;
    if (fast && p.denoise_enabled && g.sample_bytes == 1 && g.maxval <= 255) {
        const size_t qsmem = qsmem_bytes();
        // kernel attributes are per device: set on every call (one host thread may drive several)
        FROI_CUDA(cudaFuncSetAttribute(k_denoise_u8_m1b2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)qsmem));
        const long long tiles = (long long)cdiv(g.W, QX) * cdiv(g.H, QY) * n_slots;
        const int blocks = (int)std::min<long long>(tiles, 148 * 3);
        k_denoise_u8_m1b2<<<blocks, dim3(QX, QNT / QX), qsmem, s>>>(g.W, g.H, g.maxval, n_slots, d_frame_raw,
                                                                   (uint8_t*)d_den, d_sums, sp, d_lut);
        FROI_LAUNCH_CHECK();
        return;
    }
    if (g.sample_bytes == 1) {
        auto k = fast ? k_denoise<uint8_t, 1, 2> : k_denoise<uint8_t, 0, 0>;
        if (smem > 48 * 1024)
            FROI_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k<<<grid, block, smem, s>>>(g.W, g.H, g.maxval, p.denoise_enabled, mr, br, d_frame_raw,
                                    (uint8_t*)d_den, d_sums, sp, d_lut);
    } else {
        auto k = fast ? k_denoise<uint16_t, 1, 2> : k_denoise<uint16_t, 0, 0>;
        if (smem > 48 * 1024)
            FROI_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k<<<grid, block, smem, s>>>(g.W, g.H, g.maxval, p.denoise_enabled, mr, br, d_frame_raw,
                                    (uint16_t*)d_den, d_sums, sp, d_lut);
    }
    FROI_LAUNCH_CHECK();
}

}  // namespace froi
