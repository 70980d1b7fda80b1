// shard.cpp — multi-GPU ownership layout of the projected set (host logic).
//
// The reference updates every point of X in one OpenMP loop
// (proj/src/lop.cpp:41-100; Jacobi, so the update of point i depends only on
// X^k).  Across G GPUs, X is split into G contiguous ranges of its initial
// cell-sorted order (spatially compact shards).  Every rank keeps the whole X
// (repulsion needs neighbours of other shards) in an INTERNAL order in which
// shard r occupies slots [r*chunk, r*chunk + count_r): after each sweep a rank
// has updated only its own slots and one in-place all-gather of `chunk`
// float4 per rank rebuilds X^{k+1} everywhere.  Padding slots (count_r < chunk)
// map to no point.
#include <algorithm>
#include <cstdint>
#include <vector>

#include "../../include/pcs_lop.h"

extern "C" pcs_status pcs_shard_layout(const uint32_t* sorted_order, uint64_t m, int32_t nranks,
                                       uint32_t* orig_of_internal, uint32_t* internal_of_orig,
                                       uint32_t* chunk_out, uint32_t* counts) {
    if (nranks < 1 || (m && !sorted_order)) return PCS_ERR_INVALID_PARAM;
    if (m >= 0xFFFFFFF0ull) return PCS_ERR_INVALID_PARAM;
    const uint32_t chunk = (uint32_t)((m + (uint64_t)nranks - 1) / (uint64_t)nranks);
    if (chunk_out) *chunk_out = chunk;
    const uint64_t mpad = (uint64_t)chunk * (uint64_t)nranks;
    if (orig_of_internal)
        for (uint64_t i = 0; i < mpad; ++i) orig_of_internal[i] = 0xFFFFFFFFu;
    for (int32_t r = 0; r < nranks; ++r) {
        const uint64_t lo = m * (uint64_t)r / (uint64_t)nranks;
        const uint64_t hi = m * (uint64_t)(r + 1) / (uint64_t)nranks;
        if (counts) counts[r] = (uint32_t)(hi - lo);
        for (uint64_t p = lo; p < hi; ++p) {
            const uint32_t slot = (uint32_t)r * chunk + (uint32_t)(p - lo);
            const uint32_t o = sorted_order[p];
            if (o >= m) return PCS_ERR_INVALID_PARAM;
            if (orig_of_internal) orig_of_internal[slot] = o;
            if (internal_of_orig) internal_of_orig[o] = slot;
        }
    }
    return PCS_OK;
}

// Work-weighted variant: the cuts fall where the cumulative
// work of the cell-sorted order crosses r/nranks of the total, so dense regions
// (config 4's e^{3.9z} pole) are spread over more ranks.  weights[o] is the
// estimated work of original point o (NULL = 1 each); chunk = the largest shard.
extern "C" pcs_status pcs_shard_layout_weighted(const uint32_t* sorted_order, const float* weights,
                                                uint64_t m, int32_t nranks,
                                                uint32_t* orig_of_internal,
                                                uint32_t* internal_of_orig, uint32_t* chunk_out,
                                                uint32_t* counts) {
    if (nranks < 1 || (m && !sorted_order)) return PCS_ERR_INVALID_PARAM;
    if (m >= 0xFFFFFFF0ull) return PCS_ERR_INVALID_PARAM;
    std::vector<double> cum(m + 1, 0.0);
    for (uint64_t p = 0; p < m; ++p) {
        const uint32_t o = sorted_order[p];
        if (o >= m) return PCS_ERR_INVALID_PARAM;
        const double w = weights ? (double)weights[o] : 1.0;
        if (!(w >= 0.0)) return PCS_ERR_INVALID_PARAM;
        cum[p + 1] = cum[p] + w;
    }
    const double total = cum[m];
    std::vector<uint64_t> cut(nranks + 1, 0);
    cut[nranks] = m;
    for (int32_t r = 1; r < nranks; ++r) {
        const double target = total * (double)r / (double)nranks;
        uint64_t p = cut[r - 1];
        while (p < m && cum[p] < target) ++p;  // first p with cum[p] >= target
        cut[r] = p;
    }
    uint32_t chunk = 0;
    for (int32_t r = 0; r < nranks; ++r) chunk = std::max<uint32_t>(chunk, (uint32_t)(cut[r + 1] - cut[r]));
    if (m && !chunk) chunk = 1;
    if (chunk_out) *chunk_out = chunk;
    const uint64_t mpad = (uint64_t)chunk * (uint64_t)nranks;
    if (orig_of_internal)
        for (uint64_t i = 0; i < mpad; ++i) orig_of_internal[i] = 0xFFFFFFFFu;
    for (int32_t r = 0; r < nranks; ++r) {
        if (counts) counts[r] = (uint32_t)(cut[r + 1] - cut[r]);
        for (uint64_t p = cut[r]; p < cut[r + 1]; ++p) {
            const uint32_t slot = (uint32_t)r * chunk + (uint32_t)(p - cut[r]);
            const uint32_t o = sorted_order[p];
            if (orig_of_internal) orig_of_internal[slot] = o;
            if (internal_of_orig) internal_of_orig[o] = slot;
        }
    }
    return PCS_OK;
}
