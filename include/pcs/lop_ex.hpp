// lop_ex.hpp — extensions of the drop-in entry point (not in the reference).
#pragma once

#include "pcs/lop.hpp"

namespace pcs {

enum class EtaKind { InvCube, NegLinear };   // 1/(3r^3) (reference) | -r (WLOP convention)
enum class Precision { Fp64, Fp32 };

struct LopOptions {
    EtaKind eta = EtaKind::InvCube;
    bool density_weights = false;            // WLOP: v_j on the data, w_i per sweep
    Precision precision = Precision::Fp64;
    int device = -1;                         // CUDA ordinal, -1 = current
};

struct LopStats {
    std::uint64_t interactions_attr = 0, interactions_rep = 0, density_pairs = 0;
    std::uint64_t careful_points = 0;
    double setup_ms = 0, sweeps_ms = 0, kernel_ms = 0, sort_ms = 0, last_max_disp = 0;
};

std::pair<PointCloud, LopSummary> lop_project_ex(const PointCloud& data, const PointCloud& initial,
                                                 const LopParams& params, const LopOptions& options,
                                                 LopStats* stats = nullptr);

}  // namespace pcs
