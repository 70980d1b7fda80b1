// mix_bench.cu — co-issue of MUFU (ex2/rsqrt) with packed fp32x2 FMA-pipe
// instructions on sm_100a: per "pair" 4 MUFU + NF FFMA2, independent chains,
// 48 warps/SM.  Prints MUFU and FFMA2 warp-instruction rates per SM per ns, so
// the fused LOP kernel's eval mix (4 MUFU : ~14 packed) can be compared with
// the pure-MUFU ceiling.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/mix_bench tools/mix_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 16384;
constexpr int CHAINS = 4;

template <int NF, int NL>
__global__ void mix(float* out, float seed) {
    __shared__ float4 sm[8 * 64];
    for (int i = threadIdx.x; i < 8 * 64; i += blockDim.x) sm[i] = make_float4(seed, seed, seed, seed);
    __syncthreads();
    const int warp = threadIdx.x >> 5, sub = threadIdx.x & 3;
    const float4* wb = sm + (warp & 7) * 64;
    float lsum = 0.f;
    float e[CHAINS], r[CHAINS];
    unsigned long long a[CHAINS];
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
        e[c] = seed * 1e-3f * (c + 1) - 1.0f;
        r[c] = seed + c;
        float2 f = make_float2(seed + c, seed - c);
        a[c] = *reinterpret_cast<unsigned long long*>(&f);
    }
    const float2 mv = make_float2(0.9999f, 0.9998f), av = make_float2(1e-6f, 2e-6f);
    const unsigned long long m2 = *reinterpret_cast<const unsigned long long*>(&mv);
    const unsigned long long a2 = *reinterpret_cast<const unsigned long long*>(&av);
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) {
            float t0, t1, t2, t3;
            asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(t0) : "f"(e[c]));
            asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(t1) : "f"(e[c] + 0.5f));
            asm volatile("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(t2) : "f"(r[c]));
            asm volatile("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(t3) : "f"(r[c] + 0.5f));
            e[c] = fminf(t0 + t1, 0.f) - 1.0f;
            r[c] = t2 + t3 + 1.0f;
#pragma unroll
            for (int k = 0; k < NF; ++k)
                asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[c]) : "l"(m2), "l"(a2));
            // NL shared loads per "record": lanes sub = 0..3 read 4 consecutive
            // 32-byte records (the kernel's pattern, 8-way broadcast)
            if (NL >= 1) {
                float4 v;
                asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                             : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                             : "r"((unsigned)__cvta_generic_to_shared(wb + 2 * ((i * 4 + c * 16 + sub) & 31))));
                lsum += v.x;
            }
            if (NL >= 2) {
                float2 v;
                asm volatile("ld.shared.v2.f32 {%0,%1}, [%2];"
                             : "=f"(v.x), "=f"(v.y)
                             : "r"((unsigned)__cvta_generic_to_shared(wb + 2 * ((i * 4 + c * 16 + sub) & 31) + 1)));
                lsum += v.y;
            }
        }
    }
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
        float2 f = *reinterpret_cast<float2*>(&a[c]);
        s += e[c] + r[c] + f.x + f.y;
    }
    s += lsum;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int NF, int NL>
void run(int sms) {
    const int bps = 6, thr = 256;  // 48 warps per SM
    const int blocks = sms * bps;
    float* out;
    cudaMalloc(&out, sizeof(float) * blocks * thr);
    mix<NF, NL><<<blocks, thr>>>(out, 0.5f);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    mix<NF, NL><<<blocks, thr>>>(out, 0.5f);
    cudaEventRecord(e1);
    cudaDeviceSynchronize();
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double warps = (double)blocks * thr / 32;
    const double iters = warps * ITERS * CHAINS;  // "pairs" per warp
    const double ns = ms * 1e6;
    printf("{\"nf\": %d, \"nl\": %d, \"ms\": %.3f, \"mufu_warp_inst_per_sm_ns\": %.3f, "
           "\"ffma2_warp_inst_per_sm_ns\": %.3f, \"ns_per_pair_per_smsp\": %.3f}\n",
           NF, NL, ms, iters * 4 / sms / ns, iters * NF / sms / ns, ns * sms * 4 / iters);
    cudaFree(out);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<0, 0>(sms);
    run<12, 0>(sms);
    run<12, 1>(sms);
    run<12, 2>(sms);
    run<14, 0>(sms);
    run<16, 0>(sms);
    run<0, 2>(sms);
    return 0;
}
