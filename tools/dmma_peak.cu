// Measured FP64 tensor-pipe (DMMA) peak of this GPU, for K1's roofline.
//
// Every warp issues kChains independent accumulator chains of
// mma.sync.aligned.m8n8k4.row.col.f64 (SASS DMMA.8x8x4, 512 FLOP per warp
// instruction) on register operands only — no memory traffic — for kIters
// rounds; grid = SMs × blocks_per_sm.  FLOP/s = warps·kIters·kChains·512 / time
// (CUDA events, best of 5 after a warm-up).  Also times the m16n8k8 shape.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/dmma_peak tools/dmma_peak.cu
//   tools/bin/dmma_peak      # prints one JSON line
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;
constexpr int kChains = 8;

__global__ void k_dmma_884(double* out, double seed) {
    double a = seed + threadIdx.x * 1e-3, b = seed - threadIdx.x * 1e-3;
    double c[kChains][2];
#pragma unroll
    for (int j = 0; j < kChains; ++j) c[j][0] = c[j][1] = 0.0;
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int j = 0; j < kChains; ++j)
            asm volatile(
                "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                : "+d"(c[j][0]), "+d"(c[j][1])
                : "d"(a), "d"(b));
    }
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < kChains; ++j) s += c[j][0] + c[j][1];
    if (s == 12345.678) out[threadIdx.x] = s;  // keep the chains live
}

__global__ void k_dmma_1688(double* out, double seed) {
    double a0 = seed, a1 = seed * 0.5, a2 = seed * 0.25, a3 = seed * 0.125;
    double b0 = seed - 1.0, b1 = seed - 0.5;
    double c[kChains][4];
#pragma unroll
    for (int j = 0; j < kChains; ++j) c[j][0] = c[j][1] = c[j][2] = c[j][3] = 0.0;
    for (int it = 0; it < kIters / 4; ++it) {
#pragma unroll
        for (int j = 0; j < kChains; ++j)
            asm volatile(
                "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
                "{%8,%9}, {%0,%1,%2,%3};"
                : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3])
                : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
    }
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < kChains; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
    if (s == 12345.678) out[threadIdx.x] = s;
}

template <class K>
double best_tflops(K kern, int blocks, int threads, double flop_per_warp_iter, int iters) {
    double* out = nullptr;
    cudaMalloc(&out, 1024 * sizeof(double));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    kern<<<blocks, threads>>>(out, 1.0);
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        kern<<<blocks, threads>>>(out, 1.0 + r);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaFree(out);
    const double warps = (double)blocks * threads / 32.0;
    return warps * iters * kChains * flop_per_warp_iter / (best * 1e-3) / 1e12;
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    double best884 = 0.0, best1688 = 0.0;
    int cfg884 = 0, cfg1688 = 0;
    for (int bps : {1, 2, 4}) {
        for (int threads : {128, 256}) {
            const double t = best_tflops(k_dmma_884, sms * bps, threads, 512.0, kIters);
            if (t > best884) best884 = t, cfg884 = bps * 1000 + threads;
            const double u = best_tflops(k_dmma_1688, sms * bps, threads, 2048.0, kIters / 4);
            if (u > best1688) best1688 = u, cfg1688 = bps * 1000 + threads;
        }
    }
    std::printf("{\"fp64_dmma_tflops\": %.2f, \"shape\": \"m8n8k4\", \"config\": \"%d CTA/SM x %d thr\", "
                "\"fp64_dmma_m16n8k8_tflops\": %.2f, \"config_m16n8k8\": \"%d CTA/SM x %d thr\", "
                "\"sms\": %d, \"max_clock_mhz\": %d}\n",
                best884, cfg884 / 1000, cfg884 % 1000, best1688, cfg1688 / 1000, cfg1688 % 1000,
                sms, clk / 1000);
    return 0;
}
