// noise.hpp — seeded isotropic noise (proj/include/pcs/noise.hpp semantics:
// mt19937_64(seed), Box-Muller normals, x then y then z per point).
#pragma once

#include <cstdint>

#include "pcs/core.hpp"

namespace pcs {

struct NoiseParams {
    double sigma = 0.0;
    std::uint64_t seed = 0;
};

PointCloud add_noise(const PointCloud& cloud, const NoiseParams& params);

}  // namespace pcs
