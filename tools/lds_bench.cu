// lds_bench.cu — shared-memory wavefront cost of LDS.128 address patterns
// (developer microbenchmark behind the per-query candidate lists of
// lop_fast.cu).  Each pattern is a per-lane float4 index into a 16 KB
// per-warp window; the kernel issues 8 independent LDS.128 per iteration and
// reports SM cycles per warp-LDS (= wavefronts when the crossbar is the limit).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/lds_bench tools/lds_bench.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

constexpr int WARPS = 8, ITERS = 4096, WIN = 256;  // float4 per warp window

__global__ void lds_kernel(const int* __restrict__ pat, int npat_steps, float* out, int zero) {
    __shared__ float4 sm[WARPS * WIN];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < WARPS * WIN; i += blockDim.x)
        sm[i] = make_float4(i * 1e-3f, 1.f, 2.f, 3.f);
    __syncthreads();
    int idx[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) idx[k] = pat[(k % npat_steps) * 32 + lane];
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm + warp * WIN);
    float acc = 0.f;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            float4 v;
            asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                         : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                         : "r"(base + (uint32_t)((idx[k] + (it & zero)) * 16)) : "memory");
            acc += (v.x + v.y) + (v.z + v.w);
        }
    }
    if (acc == 12345.f) out[0] = acc;
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    printf("SMs %d, clock %d kHz\n", sms, clk);
    srand(1);
    struct P { const char* name; std::vector<int> v; };
    std::vector<P> pats;
    auto add = [&](const char* n, auto f) {
        P p{n, std::vector<int>(8 * 32)};
        for (int s = 0; s < 8; ++s) for (int l = 0; l < 32; ++l) p.v[s * 32 + l] = f(s, l) & (WIN - 1);
        pats.push_back(p);
    };
    // AoS records of 2 float4: record r first half at float4 2r
    add("bcast L4 (current: 8 queries share records sub..sub+3)", [](int s, int l) { return 2 * (s * 4 + (l & 3)); });
    add("bcast L2 (16 queries share 2 records)", [](int s, int l) { return 2 * (s * 2 + (l & 1)); });
    add("distinct AoS 32B stride, lane l -> rec l", [](int s, int l) { return 2 * (s * 32 + l); });
    add("distinct contiguous 16B stride", [](int s, int l) { return s * 32 + l; });
    add("L4 per-query random rec base, AoS", [](int s, int l) { return 2 * (((rand() % 100) * 7 + 0) + (l & 3)); });
    static int qb[8][8];
    for (int s = 0; s < 8; ++s) for (int q = 0; q < 8; ++q) qb[s][q] = rand() % 120;
    add("L4 per-query random rec base, AoS (consistent)", [](int s, int l) { return 2 * (qb[s][l >> 2] + (l & 3)); });
    add("L4 per-query random base, SoA 16B", [](int s, int l) { return qb[s][l >> 2] + (l & 3); });
    add("L8 per-query random 128B-aligned base, SoA", [](int s, int l) { return (qb[s][l >> 3] & ~7) + (l & 7); });
    add("L8 per-query random base (unaligned), SoA", [](int s, int l) { return qb[s][l >> 3] + (l & 7); });
    add("quarter pairs bcast: 4 groups x 4 recs, SoA", [](int s, int l) { return qb[s][l >> 3] + (l & 3); });
    add("quarter pairs bcast aligned 64B, SoA", [](int s, int l) { return (qb[s][l >> 3] & ~3) + (l & 3); });
    add("all lanes same address", [](int s, int l) { return s; });
    int* dpat; float* dout;
    cudaMalloc(&dpat, 8 * 32 * sizeof(int));
    cudaMalloc(&dout, 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    const int blocks = sms * 2;  // 16 warps per SM
    for (auto& p : pats) {
        cudaMemcpy(dpat, p.v.data(), 8 * 32 * sizeof(int), cudaMemcpyHostToDevice);
        lds_kernel<<<blocks, WARPS * 32>>>(dpat, 8, dout, 0);
        cudaEventRecord(a);
        lds_kernel<<<blocks, WARPS * 32>>>(dpat, 8, dout, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (cudaGetLastError() != cudaSuccess) { printf("launch error\n"); return 1; }
        const double warp_lds_per_sm = (double)blocks * WARPS * ITERS * 8 / sms;
        const double cyc = ms * 1e-3 * clk * 1e3;
        printf("%-55s %6.2f SM-cycles per warp LDS.128\n", p.name, cyc / warp_lds_per_sm);
    }
    return 0;
}
