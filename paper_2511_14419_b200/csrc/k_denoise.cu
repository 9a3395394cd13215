// k_denoise.cu — fused median + bilateral denoise (denoise.hpp:28-90), bit-exact.
//
// One CTA produces a 32x16 output tile of one frame slot.  The raw tile (halo = median radius +
// bilateral radius, edge-replicated) and the median tile (halo = bilateral radius) live in
// shared memory; the bilateral sums run in fp64 in the reference's dy-major / dx-minor order
// with explicit round-to-nearest operations (no FMA), the range LUT and spatial weights are the
// host-computed libm values, and rounding is std::lround (half away from zero).  The CTA also
// reduces the integer sum of its denoised pixels for the registration mean
// (registration.hpp:27-29), which is exact in integers.
//
// Roofline: HBM-bound at 2 B/px for u8 (read raw, write den) — SURVEY.md App. C row "D".
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
