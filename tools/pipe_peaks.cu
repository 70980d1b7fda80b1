// pipe_peaks.cu — measures the sm_100a issue rates that bound the fused LOP
// kernel: MUFU.EX2, MUFU.RSQ, FFMA (3-register), FFMA2 (packed fp32x2), per SM
// per clock.  Writes one JSON object to stdout (see profiles/pipe_peaks.json).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/pipe_peaks tools/pipe_peaks.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int ITERS = 65536;
constexpr int CHAINS = 8;

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float rsq(float x) {
    float y;
    asm volatile("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

template <int KIND>
__global__ void bench(float* out, float seed, long long* cycles) {
    float v[CHAINS];
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) v[c] = seed + threadIdx.x * 1e-7f + c * 1e-3f;
    unsigned long long a2[CHAINS / 2];
#pragma unroll
    for (int c = 0; c < CHAINS / 2; ++c) {
        float2 f = make_float2(v[2 * c], v[2 * c + 1]);
        a2[c] = *reinterpret_cast<unsigned long long*>(&f);
    }
    const float2 mulv = make_float2(0.9999f, 0.9998f), addv = make_float2(1e-6f, 2e-6f);
    const unsigned long long m2 = *reinterpret_cast<const unsigned long long*>(&mulv);
    const unsigned long long ad2 = *reinterpret_cast<const unsigned long long*>(&addv);
    __syncthreads();
    const long long t0 = clock64();
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) {
            if (KIND == 0) v[c] = ex2(v[c]) - 1.0f;      // MUFU.EX2 (+FADD)
            if (KIND == 1) v[c] = rsq(v[c] + 1.0f);      // MUFU.RSQ (+FADD)
            if (KIND == 2) v[c] = fmaf(v[c], 0.9999f, 1e-6f);
        }
        if (KIND == 3) {
#pragma unroll
            for (int c = 0; c < CHAINS / 2; ++c)
                asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a2[c]) : "l"(m2), "l"(ad2));
        }
    }
    const long long t1 = clock64();
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) s += v[c];
#pragma unroll
    for (int c = 0; c < CHAINS / 2; ++c) {
        float2 f = *reinterpret_cast<float2*>(&a2[c]);
        s += f.x + f.y;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

double g_last_ops_per_s = 0, g_last_ms = 0;

template <int KIND>
double rate_per_sm_clk(int blocks_per_sm, int threads) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * blocks_per_sm;
    float* out;
    long long* cyc;
    cudaMalloc(&out, sizeof(float) * blocks * threads);
    cudaMalloc(&cyc, sizeof(long long) * blocks);
    bench<KIND><<<blocks, threads>>>(out, 0.5f, cyc);  // warm-up
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    bench<KIND><<<blocks, threads>>>(out, 0.5f, cyc);
    cudaEventRecord(e1);
    cudaDeviceSynchronize();
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    g_last_ops_per_s = (double)blocks * threads * ITERS * CHAINS / (ms * 1e-3);
    g_last_ms = ms;
    long long* h = new long long[blocks];
    cudaMemcpy(h, cyc, sizeof(long long) * blocks, cudaMemcpyDeviceToHost);
    double mean = 0;
    for (int b = 0; b < blocks; ++b) mean += (double)h[b];
    mean /= blocks;
    delete[] h;
    cudaFree(out);
    cudaFree(cyc);
    // ops per SM during the measured window (all blocks of an SM are co-resident)
    const double ops = (double)blocks_per_sm * threads * ITERS * CHAINS;
    return ops / mean;
}

int main() {
    const int bps = 4, thr = 512;  // 64 warps per SM
    const double ex2r = rate_per_sm_clk<0>(bps, thr);
    const double ex2s = g_last_ops_per_s, ex2ms = g_last_ms;
    const double rsqr = rate_per_sm_clk<1>(bps, thr);
    const double rsqs = g_last_ops_per_s;
    const double ffma = rate_per_sm_clk<2>(bps, thr);
    const double ffmas = g_last_ops_per_s;
    const double ffma2 = rate_per_sm_clk<3>(bps, thr);  // fp32 FMAs (2 per instruction)
    const double ffma2s = g_last_ops_per_s;
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    printf("{\"ex2_per_s\": %.4e, \"rsqrt_per_s\": %.4e, \"ffma_per_s\": %.4e, \"ffma2_fma_per_s\": %.4e, \"ex2_run_ms\": %.2f, ",
           ex2s, rsqs, ffmas, ffma2s, ex2ms);
    printf("\"device\": \"%s\", \"sms\": %d, \"ex2_per_sm_clk64\": %.3f, \"rsqrt_per_sm_clk64\": %.3f, "
           "\"mufu_per_sm_clk64\": %.3f, \"ffma_per_sm_clk64\": %.3f, \"ffma2_fma_per_sm_clk64\": %.3f, "
           "\"method\": \"clock64 over %d dependent-chain iterations x %d chains, %d warps/SM; "
           "ex2/rsqrt loops carry one FADD per MUFU\"}\n",
           p.name, p.multiProcessorCount, ex2r, rsqr, (ex2r + rsqr) / 2, ffma, ffma2, ITERS, CHAINS,
           bps * thr / 32);
    return 0;
}
