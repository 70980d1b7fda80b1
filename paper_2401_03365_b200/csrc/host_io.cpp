// host_io.cpp — host->device transfer of the caller's (pageable) clouds.
//
// A pageable cudaMemcpy runs at ~10 GB/s on the B200 hosts (the driver stages
// through its own pinned buffer with one thread).  Here the copy goes through a
// process-wide pool of two pinned 16 MB chunks filled by OpenMP threads while
// the DMA of the previous chunk runs: ~24 GB/s measured (tools/h2d_probe.cu).
#include "dev_knobs.h"
#include "host_io.h"

#include <omp.h>

#include <algorithm>
#include <array>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

namespace pcsb {

void cuda_check(cudaError_t e, const char* what);  // plan.cu: throws Failure
#define PCSB_CUDA(x) ::pcsb::cuda_check((x), #x)

namespace {
constexpr size_t kChunk = 16u << 20;

struct Staging {
    std::mutex mu;
    char* buf[2] = {nullptr, nullptr};
    cudaEvent_t done[2] = {nullptr, nullptr};
    bool ready = false;
};

// host threads filling / draining the pinned chunks (developer knob PCSB_IO_THREADS)
int staging_threads() {
    static const int t = [] {
        const char* e = dev_knob("PCSB_IO_THREADS");
        const int v = e ? std::atoi(e) : 16;  // e2e (config 3): 8 -> 16 threads +3%
        return std::max(1, std::min(v, omp_get_num_procs()));
    }();
    return t;
}

Staging& staging() {
    static Staging s;  // never freed: pinned memory lives as long as the process
    return s;
}
}  // namespace

void h2d_staged(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    if (!bytes) return;
    if (bytes < (2u << 20)) {  // small: the driver's path is as fast
        PCSB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
        return;
    }
    Staging& st = staging();
    std::lock_guard<std::mutex> lock(st.mu);
    if (!st.ready) {
        for (int i = 0; i < 2; ++i) {
            PCSB_CUDA(cudaHostAlloc((void**)&st.buf[i], kChunk, cudaHostAllocPortable));
            PCSB_CUDA(cudaEventCreateWithFlags(&st.done[i], cudaEventDisableTiming));
        }
        st.ready = true;
    }
    const int threads = staging_threads();
    const char* in = static_cast<const char*>(src);
    char* out = static_cast<char*>(dst);
    size_t k = 0;
    for (size_t off = 0; off < bytes; off += kChunk, ++k) {
        const size_t n = std::min(kChunk, bytes - off);
        char* b = st.buf[k & 1];
        // the chunk's previous DMA (two chunks ago) must have drained
        PCSB_CUDA(cudaEventSynchronize(st.done[k & 1]));
        const size_t per = (n + threads - 1) / threads;
#pragma omp parallel for num_threads(threads) schedule(static)
        for (int t = 0; t < threads; ++t) {
            const size_t a = (size_t)t * per;
            const size_t e = std::min(n, a + per);
            if (a < e) std::memcpy(b + a, in + off + a, e - a);
        }
        PCSB_CUDA(cudaMemcpyAsync(out + off, b, n, cudaMemcpyHostToDevice, s));
        PCSB_CUDA(cudaEventRecord(st.done[k & 1], s));
    }
    // the pool is reused by the next call: drain before releasing it
    PCSB_CUDA(cudaEventSynchronize(st.done[(k - 1) & 1]));
}

// device-side landing chunks of h2d_staged_f32x4 (packed fp32 xyz), per device
float* device_chunk(int k) {
    static std::mutex mu;
    static std::vector<std::array<float*, 2>> per_dev;
    int dev = 0;
    PCSB_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(mu);
    if ((int)per_dev.size() <= dev) per_dev.resize(dev + 1, {nullptr, nullptr});
    float*& p = per_dev[dev][k & 1];
    if (!p) PCSB_CUDA(cudaMalloc((void**)&p, kChunk));  // lives as long as the process
    return p;
}

void h2d_staged_f32x4(void* dst_float4, const double* xyz, size_t n, float w, cudaStream_t s) {
    if (!n) return;
    Staging& st = staging();
    std::lock_guard<std::mutex> lock(st.mu);
    if (!st.ready) {
        for (int i = 0; i < 2; ++i) {
            PCSB_CUDA(cudaHostAlloc((void**)&st.buf[i], kChunk, cudaHostAllocPortable));
            PCSB_CUDA(cudaEventCreateWithFlags(&st.done[i], cudaEventDisableTiming));
        }
        st.ready = true;
    }
    const int threads = staging_threads();
    // 12 bytes per point cross PCIe (packed fp32 xyz); a kernel widens each
    // landed chunk to float4 {x, y, z, w} in place in the destination
    const size_t per_chunk = kChunk / (3 * sizeof(float));
    float4* out = static_cast<float4*>(dst_float4);
    size_t k = 0;
    for (size_t p0 = 0; p0 < n; p0 += per_chunk, ++k) {
        const size_t np = std::min(per_chunk, n - p0);
        float* b = reinterpret_cast<float*>(st.buf[k & 1]);
        float* d = device_chunk((int)k);
        // the chunk's previous DMA and widening (two chunks ago) must have drained
        PCSB_CUDA(cudaEventSynchronize(st.done[k & 1]));
        const double* q = xyz + 3 * p0;
#pragma omp parallel for num_threads(threads) schedule(static)
        for (long long i = 0; i < (long long)(3 * np); ++i) b[i] = (float)q[i];
        PCSB_CUDA(cudaMemcpyAsync(d, b, np * 12, cudaMemcpyHostToDevice, s));
        launch_widen_f32x3(d, out + p0, np, w, s);
        PCSB_CUDA(cudaEventRecord(st.done[k & 1], s));
    }
    PCSB_CUDA(cudaEventSynchronize(st.done[(k - 1) & 1]));
}

void d2h_staged(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    if (!bytes) return;
    if (bytes < (2u << 20)) {
        PCSB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
        PCSB_CUDA(cudaStreamSynchronize(s));
        return;
    }
    Staging& st = staging();
    std::lock_guard<std::mutex> lock(st.mu);
    if (!st.ready) {
        for (int i = 0; i < 2; ++i) {
            PCSB_CUDA(cudaHostAlloc((void**)&st.buf[i], kChunk, cudaHostAllocPortable));
            PCSB_CUDA(cudaEventCreateWithFlags(&st.done[i], cudaEventDisableTiming));
        }
        st.ready = true;
    }
    const int threads = staging_threads();
    const char* in = static_cast<const char*>(src);
    char* out = static_cast<char*>(dst);
    // DMA chunk k+1 while the threads drain chunk k; 4 MB chunks (of the 16 MB
    // buffers) keep the first DMA and the last drain short
    constexpr size_t kD2H = 4u << 20;
    const size_t nchunks = (bytes + kD2H - 1) / kD2H;
    PCSB_CUDA(cudaMemcpyAsync(st.buf[0], in, std::min(kD2H, bytes), cudaMemcpyDeviceToHost, s));
    PCSB_CUDA(cudaEventRecord(st.done[0], s));
    for (size_t k = 0; k < nchunks; ++k) {
        const size_t off = k * kD2H, n = std::min(kD2H, bytes - off);
        if (k + 1 < nchunks) {
            const size_t off1 = off + kD2H, n1 = std::min(kD2H, bytes - off1);
            PCSB_CUDA(cudaMemcpyAsync(st.buf[(k + 1) & 1], in + off1, n1, cudaMemcpyDeviceToHost, s));
            PCSB_CUDA(cudaEventRecord(st.done[(k + 1) & 1], s));
        }
        PCSB_CUDA(cudaEventSynchronize(st.done[k & 1]));
        const char* b = st.buf[k & 1];
        const size_t per = (n + threads - 1) / threads;
#pragma omp parallel for num_threads(threads) schedule(static)
        for (int t = 0; t < threads; ++t) {
            const size_t a = (size_t)t * per;
            const size_t e = std::min(n, a + per);
            if (a < e) std::memcpy(out + off + a, b + a, e - a);
        }
    }
}

}  // namespace pcsb
