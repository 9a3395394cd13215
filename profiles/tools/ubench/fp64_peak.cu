// fp64_peak.cu — measured fp64 throughput of this B200 (the denominator for the fp64 stages:
// denoise and registration are exact-fp64 by construction, so HBM is not their bound).
//
// DFMA: 8 independent chains per thread, 256 threads per CTA, 8 CTAs per SM, timed with CUDA
// events after a warm-up; DADD / DMUL likewise (same pipe, one flop each).  Prints one JSON line:
// TFLOP/s for DFMA (2 flops per instruction) and Gop/s for DADD and DMUL.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak.bin fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CH = 8, IT = 4096;

template <int OP>
__global__ void __launch_bounds__(256) k_fp64(double* out, double a, double b) {
    double x[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-7 + c;
    for (int i = 0; i < IT; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            if (OP == 0) x[c] = __fma_rn(x[c], a, b);
            else if (OP == 1) x[c] = __dadd_rn(x[c], b);
            else x[c] = __dmul_rn(x[c], a);
        }
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += x[c];
    if (s == 12345.678) out[threadIdx.x] = s;  // keeps the chains alive
}

template <int OP>
double run(int sms) {
    double* d;
    cudaMalloc(&d, 1024 * sizeof(double));
    const dim3 grid(sms * 8), block(256);
    k_fp64<OP><<<grid, block>>>(d, 0.999999, 1e-9);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        k_fp64<OP><<<grid, block>>>(d, 0.999999, 1e-9);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    cudaFree(d);
    const double ops = (double)grid.x * block.x * CH * IT;
    return ops / (best * 1e-3);
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    const double fma = run<0>(sms), add = run<1>(sms), mul = run<2>(sms);
    std::printf("{\"dfma_tflops\": %.3f, \"dadd_gops\": %.1f, \"dmul_gops\": %.1f, \"dfma_per_clk_per_sm\": %.2f, "
                "\"sms\": %d, \"clock_mhz\": %.0f, \"how\": \"8 independent chains x 256 thr x 8 CTAs/SM, best of 5\"}\n",
                2.0 * fma / 1e12, add / 1e9, mul / 1e9, fma / (sms * clk * 1e3), sms, clk / 1e3);
    return 0;
}
