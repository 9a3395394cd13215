// Microbenchmark: a per-thread 15-deep x 5-plane ring kept in TMEM (tcgen05.ld/st 32x32b) versus
// the same ring in shared memory, alone and next to extra shared-memory traffic, to see whether
// TMEM traffic competes with the LSU/shared-memory data pipe.  nvcc -arch=sm_100a tmem_ring.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int NT = 384, COLS = 256, PER_WARP = 80;  // 12 warps: 3 per lane quarter x 80 columns

__device__ __forceinline__ void tst5(uint32_t a, float v0, float v1, float v2, float v3, float v4) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(v0), "f"(v1), "f"(v2), "f"(v3));
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(a + 4), "f"(v4));
}
__device__ __forceinline__ void tld5(uint32_t a, float& v0, float& v1, float& v2, float& v3, float& v4) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];" : "=f"(v0), "=f"(v1), "=f"(v2), "=f"(v3) : "r"(a));
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=f"(v4) : "r"(a + 4));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

template <int MODE, int EXTRA>
__global__ void __launch_bounds__(NT, 2) k(float* out, int iters) {
    extern __shared__ float sm[];  // [15*5][NT] ring (mode 1) + [EXTRA scratch]
    __shared__ uint32_t taddr_s;
    const int warp = threadIdx.x >> 5, tid = threadIdx.x;
    if (MODE == 0) {
        if (warp == 0) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(&taddr_s)), "n"(COLS));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;");
    }
    const uint32_t base = taddr_s + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * PER_WARP;
    float* ring = sm;
    float* xs = sm + 75 * NT;
    float a0 = 0, a1 = 0, a2 = 0, a3 = 0, a4 = 0, x = 0;
    float g0 = tid * 1e-3f, g1 = 1.f, g2 = 2.f, g3 = 3.f, g4 = 4.f;
    for (int it = 0; it < iters; ++it) {
        const int s = it % 15;
        float o0, o1, o2, o3, o4;
        if (MODE == 0) {
            tld5(base + s * 5, o0, o1, o2, o3, o4);
            tst5(base + s * 5, g0, g1, g2, g3, g4);
        } else if (MODE == 1) {
            float* r = ring + s * 5 * NT + tid;
            o0 = r[0]; o1 = r[NT]; o2 = r[2 * NT]; o3 = r[3 * NT]; o4 = r[4 * NT];
            r[0] = g0; r[NT] = g1; r[2 * NT] = g2; r[3 * NT] = g3; r[4 * NT] = g4;
        } else {
            o0 = o1 = o2 = o3 = o4 = 0.f;
        }
        a0 += g0 - o0; a1 += g1 - o1; a2 += g2 - o2; a3 += g3 - o3; a4 += g4 - o4;
#pragma unroll
        for (int e = 0; e < EXTRA; ++e) {
            x += xs[((it * 7 + e * 33) & 1023) * 0 + e * NT + tid];
            xs[e * NT + tid] = x;
        }
        g0 = a0 * 0.5f + 1.f; g1 = a1 * 0.25f; g2 = a2 + g0; g3 = g1 - a3; g4 = a4 * g2;
    }
    out[blockIdx.x * NT + tid] = a0 + a1 + a2 + a3 + a4 + x;
    if (MODE == 0) {
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncthreads();
        if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr_s), "n"(COLS));
    }
}

template <int MODE, int EXTRA>
void run(const char* name, float* d, int iters) {
    const int smem = (75 + 8) * NT * 4;
    cudaFuncSetAttribute(k<MODE, EXTRA>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int blocks = 148 * 2;
    k<MODE, EXTRA><<<blocks, NT, smem>>>(d, 100);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    k<MODE, EXTRA><<<blocks, NT, smem>>>(d, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    cudaError_t e = cudaGetLastError();
    const double cyc = ms * 1e-3 * 1.9e9 / iters;  // SM cycles per iteration (2 CTAs / SM)
    printf("%-28s %8.3f ms  %6.1f cycles/iter/SM  (%5.2f per warp-iter) %s\n", name, ms, cyc, cyc / 24, cudaGetErrorString(e));
}

int main() {
    float* d;
    cudaMalloc(&d, 148 * 2 * NT * 4);
    const int it = 20000;
    run<2, 0>("none", d, it);
    run<0, 0>("tmem ring", d, it);
    run<1, 0>("smem ring", d, it);
    run<2, 8>("8 extra lds/sts", d, it);
    run<0, 8>("tmem ring + 8 extra", d, it);
    run<1, 8>("smem ring + 8 extra", d, it);
    return 0;
}
