// Random check of the branch-free fast paths in csrc/common.cuh against the CUDA intrinsics
// (tests/test_gpu_fastpath.py).  Prints "<name> <mode> <operands> <mismatches>" per line.
#include <cstdio>
#include "../../paper_2511_14419_b200/csrc/common.cuh"

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdull;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ull;
    x ^= x >> 33;
    return x;
}

__device__ __forceinline__ bool same(double a, double b) { return __double_as_longlong(a) == __double_as_longlong(b); }

// mode 0: operands in the path's range (unit-scale spectra, [0, 0.5] gradients, squares of both);
// mode 1: any finite bit pattern
__device__ __forceinline__ double operand(uint64_t u, int mode, int kind) {
    if (mode == 1) return __longlong_as_double(u & 0x7fefffffffffffffull);
    const double v = (double)(u >> 11) * 0x1p-53;  // [0, 1)
    if (kind == 0) return v * 0x1p+20 * (u & 1 ? 1e-6 : 1.0);
    return v * 0.5;
}

__global__ void check(unsigned long long seed, int iters, int mode, unsigned long long* bad) {
    uint64_t s = seed * 0x9E3779B97F4A7C15ull + blockIdx.x * 1024ull + threadIdx.x;
    for (int i = 0; i < iters; ++i) {
        const uint64_t u = mix(s += 0x9E3779B97F4A7C15ull), v = mix(u + 1), w = mix(v + 7);
        // sqrt
        {
            const double x = operand(u, mode, 0);
            bool ok;
            const double r = froi::dsqrt_fast(x, ok);
            if (ok && !same(r, __dsqrt_rn(x))) atomicAdd(bad + 0, 1ull);
        }
        // division a / m and b / m through one reciprocal
        {
            const double a = operand(u, mode, 0), b = operand(v, mode, 0), m = operand(w, mode, 0);
            if (m > 0.0) {
                const double r2 = froi::drcp_refined(m);
                bool oka, okb;
                const double qa = froi::ddiv_fast(a, m, r2, oka), qb = froi::ddiv_fast(b, m, r2, okb);
                if ((oka && !same(qa, __ddiv_rn(a, m))) || (okb && !same(qb, __ddiv_rn(b, m))))
                    atomicAdd(bad + 1, 1ull);
            }
        }
        // hypot
        {
            const double x = operand(v, mode, 1) - 0.25 * (mode == 0), y = operand(w, mode, 1);
            bool ok;
            const double h = froi::hypot_glibc_fast(x, y, ok);
            if (ok && !same(h, froi::hypot_glibc(x, y))) atomicAdd(bad + 2, 1ull);
            if (!ok) atomicAdd(bad + 3, 1ull);  // how often the caller's redo runs
        }
    }
}

int main(int argc, char** argv) {
    const int iters = argc > 1 ? atoi(argv[1]) : 1000;
    unsigned long long* d;
    cudaMalloc(&d, 32);
    for (int mode = 0; mode < 2; ++mode) {
        cudaMemset(d, 0, 32);
        check<<<148 * 8, 1024>>>(777 + mode, iters, mode, d);
        unsigned long long h[4];
        if (cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost) != cudaSuccess) return 1;
        const double n = 148.0 * 8 * 1024 * iters;
        printf("sqrt %d %.0f %llu\n", mode, n, h[0]);
        printf("div %d %.0f %llu\n", mode, 2 * n, h[1]);
        printf("hypot %d %.0f %llu\n", mode, n, h[2]);
        printf("redo %d %.0f %llu\n", mode, n, h[3]);
    }
    return 0;
}
