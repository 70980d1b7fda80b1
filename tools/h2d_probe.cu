// h2d_probe.cu — host->device strategies for a pageable user buffer (the
// pcs_lop_run upload): plain cudaMemcpy, cudaHostRegister + async copy, and a
// pinned double-buffered staging pipeline fed by T host threads.
//
//   nvcc -O3 -std=c++17 -o tools/bin/h2d_probe tools/h2d_probe.cu -lpthread
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

static double now_ms() {
    return std::chrono::duration<double, std::milli>(
               std::chrono::steady_clock::now().time_since_epoch())
        .count();
}

int main() {
    const size_t bytes = 240ull << 20;
    std::vector<char> host(bytes);
    for (size_t i = 0; i < bytes; i += 4096) host[i] = (char)i;
    void* dev = nullptr;
    cudaMalloc(&dev, bytes);
    cudaFree(0);
    cudaStream_t s;
    cudaStreamCreate(&s);
    for (int rep = 0; rep < 2; ++rep) {
        double t = now_ms();
        cudaMemcpy(dev, host.data(), bytes, cudaMemcpyHostToDevice);
        printf("pageable cudaMemcpy: %.2f ms (%.1f GB/s)\n", now_ms() - t, bytes / (now_ms() - t) / 1e6);

        t = now_ms();
        cudaHostRegister(host.data(), bytes, cudaHostRegisterDefault);
        const double t_reg = now_ms() - t;
        cudaMemcpyAsync(dev, host.data(), bytes, cudaMemcpyHostToDevice, s);
        cudaStreamSynchronize(s);
        const double t_cp = now_ms() - t - t_reg;
        const double t2 = now_ms();
        cudaHostUnregister(host.data());
        printf("register %.2f + copy %.2f + unregister %.2f ms\n", t_reg, t_cp, now_ms() - t2);

        for (int threads : {1, 4, 8, 16}) {
            const size_t chunk = 16ull << 20;
            char* pin[2];
            cudaHostAlloc((void**)&pin[0], chunk, cudaHostAllocDefault);
            cudaHostAlloc((void**)&pin[1], chunk, cudaHostAllocDefault);
            cudaEvent_t ev[2];
            cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming);
            cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming);
            t = now_ms();
            int k = 0;
            for (size_t off = 0; off < bytes; off += chunk, ++k) {
                const size_t n = std::min(chunk, bytes - off);
                char* b = pin[k & 1];
                if (k >= 2) cudaEventSynchronize(ev[k & 1]);
                std::vector<std::thread> th;
                const size_t per = (n + threads - 1) / threads;
                for (int i = 0; i < threads; ++i) {
                    const size_t a = i * per, e = std::min(n, a + per);
                    if (a < e) th.emplace_back([=, &host] { memcpy(b + a, host.data() + off + a, e - a); });
                }
                for (auto& x : th) x.join();
                cudaMemcpyAsync((char*)dev + off, b, n, cudaMemcpyHostToDevice, s);
                cudaEventRecord(ev[k & 1], s);
            }
            cudaStreamSynchronize(s);
            printf("pinned staging, %d threads: %.2f ms\n", threads, now_ms() - t);
            cudaFreeHost(pin[0]);
            cudaFreeHost(pin[1]);
        }
        t = now_ms();
        char* big;
        cudaHostAlloc((void**)&big, bytes, cudaHostAllocDefault);
        printf("cudaHostAlloc 240 MB: %.2f ms\n", now_ms() - t);
        t = now_ms();
        cudaMemcpyAsync(dev, big, bytes, cudaMemcpyHostToDevice, s);
        cudaStreamSynchronize(s);
        printf("pinned->device 240 MB: %.2f ms\n", now_ms() - t);
        cudaFreeHost(big);
    }
    printf("hardware threads: %u\n", std::thread::hardware_concurrency());
    return 0;
}
