// fp32_peak.cu — sustained FP32 FFMA throughput of this B200 (the "alu" roofline
// denominator of the projectors: "the builder measures a sustained
// FMA microbenchmark").
//
// Every thread runs NCH independent FFMA chains (enough ILP to cover the 4-cycle
// FFMA latency at any occupancy) for ITER iterations; grid = 148 SMs x BPS blocks
// of 256 threads.  FLOP = 2 per FFMA.  Timed with CUDA events: "burst" = best of
// 10 single launches (~10 ms each), "sustained" = back-to-back launches for ~4 s
// (the clocks a long solve sees).  Output: one JSON line on stdout.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp32_peak scripts/fp32_peak.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

constexpr int NCH = 8;

__global__ void __launch_bounds__(256) k_ffma(float* out, int iters, float a, float b) {
    float r[NCH];
#pragma unroll
    for (int c = 0; c < NCH; c++) r[c] = (float)(threadIdx.x + c) * 1e-3f;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int u = 0; u < 16; u++) {
#pragma unroll
            for (int c = 0; c < NCH; c++) r[c] = fmaf(r[c], a, b);
        }
    }
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < NCH; c++) s += r[c];
    if (s == 12345.678f) out[blockIdx.x] = s;  // keeps the chains live
}

// packed FP32 (sm_100a FFMA2: fma.rn.f32x2, two FMAs per lane per instruction)
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b, unsigned long long c) {
    unsigned long long d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__global__ void __launch_bounds__(256) k_ffma2(float* out, int iters, float a, float b) {
    unsigned long long r[NCH / 2];
    const float2 a2 = make_float2(a, a), b2 = make_float2(b, b);
    const unsigned long long A = *reinterpret_cast<const unsigned long long*>(&a2);
    const unsigned long long B = *reinterpret_cast<const unsigned long long*>(&b2);
#pragma unroll
    for (int c = 0; c < NCH / 2; c++) {
        const float2 v = make_float2((float)(threadIdx.x + c) * 1e-3f, (float)(threadIdx.x - c) * 1e-3f);
        r[c] = *reinterpret_cast<const unsigned long long*>(&v);
    }
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int u = 0; u < 16; u++) {
#pragma unroll
            for (int c = 0; c < NCH / 2; c++) r[c] = ffma2(r[c], A, B);
        }
    }
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < NCH / 2; c++) {
        const float2 v = *reinterpret_cast<const float2*>(&r[c]);
        s += v.x + v.y;
    }
    if (s == 12345.678f) out[blockIdx.x] = s;
}

int main() {
    int dev = 0, nsm = 0, clk_khz = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
    float* out;
    cudaMalloc(&out, 1 << 20);
    const int bps = 8, threads = 256, iters = 4096;
    const int blocks = nsm * bps;
    const double flop = 2.0 * NCH * 16.0 * iters * (double)threads * blocks;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_ffma<<<blocks, threads>>>(out, iters, 0.999f, 1e-4f);  // warm-up
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 10; r++) {
        cudaEventRecord(e0);
        k_ffma<<<blocks, threads>>>(out, iters, 0.999f, 1e-4f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    // sustained: back to back for ~4 s
    const int nrep = (int)(4000.0f / best) + 1;
    cudaEventRecord(e0);
    for (int r = 0; r < nrep; r++) k_ffma<<<blocks, threads>>>(out, iters, 0.999f, 1e-4f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float tot;
    cudaEventElapsedTime(&tot, e0, e1);
    // FFMA2: the same FLOP count per launch in half the instructions
    float best2 = 1e30f;
    for (int r = 0; r < 10; r++) {
        cudaEventRecord(e0);
        k_ffma2<<<blocks, threads>>>(out, iters, 0.999f, 1e-4f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best2) best2 = ms;
    }
    const double burst2 = flop / (best2 * 1e-3) / 1e12;
    const double burst = flop / (best * 1e-3) / 1e12;
    const double sus = flop * nrep / (tot * 1e-3) / 1e12;
    cudaError_t err = cudaGetLastError();
    printf("{\"fp32_ffma2_tflops\": %.3f, \"fp32_tflops\": %.3f, \"fp32_tflops_sustained\": %.3f, \"sms\": %d, \"clock_attr_mhz\": %.0f, "
           "\"nominal_tflops_at_attr_clock\": %.3f, \"launch_ms\": %.4f, \"sustained_s\": %.3f, \"reps\": %d, "
           "\"how\": \"%d FFMA chains x 16 x %d per thread, %d blocks x %d threads, CUDA events; burst = best of 10, "
           "sustained = back-to-back for ~4 s\", \"cuda\": \"%s\"}\n",
           burst2, burst, sus, nsm, clk_khz / 1e3, nsm * 128.0 * 2.0 * clk_khz * 1e3 / 1e12, best, tot / 1e3, nrep, NCH,
           iters, blocks, threads, cudaGetErrorString(err));
    return err == cudaSuccess ? 0 : 1;
}
