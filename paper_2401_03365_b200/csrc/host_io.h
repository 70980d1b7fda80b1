// host_io.h — staged host->device copies of caller buffers (host_io.cpp).
#pragma once

#include <cstddef>

#include <cuda_runtime.h>

namespace pcsb {

// Copies `bytes` from pageable host memory to device memory on stream s; returns
// when the host buffer may be reused (the copy itself is complete too).
void h2d_staged(void* dst, const void* src, size_t bytes, cudaStream_t s);
// n points of xyz (3 doubles each, pageable) to float4 {x, y, z, w} on the device,
// rounded to fp32 by the host threads that fill the pinned chunks (half the
// bytes of an fp64 copy cross PCIe; round-to-nearest like __double2float_rn).
void h2d_staged_f32x4(void* dst_float4, const double* xyz, size_t n, float w, cudaStream_t s);
// grid_sort.cu: dst[i] = {src[3i], src[3i+1], src[3i+2], w}, i < n
void launch_widen_f32x3(const float* src, float4* dst, size_t n, float w, cudaStream_t s);
// Device -> pageable host after the work already queued on s; returns when dst is filled.
void d2h_staged(void* dst, const void* src, size_t bytes, cudaStream_t s);

}  // namespace pcsb
