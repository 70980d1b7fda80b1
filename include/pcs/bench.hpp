// bench.hpp — seeded synthetic surfaces (proj/include/pcs/bench.hpp:13-30 semantics).
// Only the generators are provided: the reference's MLS timing harness is off
// the LOP path.
#pragma once

#include <cstdint>

#include "pcs/core.hpp"

namespace pcs {

enum class SurfaceKind { Plane, Sphere, Torus, GaussianBump };

struct SyntheticSurface {
    SurfaceKind kind = SurfaceKind::Sphere;
    std::size_t n = 0;
    std::uint64_t seed = 0;
};

PointCloud generate_surface(const SyntheticSurface& surface);

}  // namespace pcs
