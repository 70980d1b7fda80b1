// spatial.hpp — exact radius / nearest queries of the drop-in C++ API.
// Same public declarations and meaning as the reference
// (proj/include/pcs/spatial.hpp): inclusive ball test d2 <= r*r on
// norm2(p - c), hits sorted by original index, distance = sqrt(d2); nearest
// breaks exact ties toward the smaller index.  The reference builds a kd-tree
// on the host; here the index holds a device copy of the cloud (pcs_mls_index,
// built on first use) with a uniform grid per query radius.
#pragma once

#include <cstdint>
#include <memory>
#include <vector>

#include "pcs/core.hpp"

struct pcs_mls_index;

namespace pcs {

class SpatialIndex {
public:
    struct Hit {
        std::size_t index;   ///< original position in the indexed cloud
        double distance;     ///< Euclidean distance to the query point
    };

    /// The index references the cloud; the cloud must outlive it.  leaf_size
    /// (the reference's kd-tree leaf size) is validated (>= 1) and otherwise
    /// unused by the device grid.
    explicit SpatialIndex(const PointCloud& cloud, int leaf_size = 16);

    /// All points with ||p - center|| <= r, sorted by original index.
    std::vector<Hit> radius_query(Point3 center, double r) const;

    /// Buffer-reusing variant. `out` is cleared first.
    void radius_query(Point3 center, double r, std::vector<Hit>& out) const;

    /// Globally nearest point; ties broken toward the smallest index.
    Hit nearest(Point3 query) const;

    std::size_t size() const { return cloud_->size(); }
    const PointCloud& cloud() const { return *cloud_; }

    /// The device index of the cloud (created on first use; shared by copies).
    pcs_mls_index* device_index() const;

private:
    struct Device;
    const PointCloud* cloud_;
    int leaf_size_;
    std::shared_ptr<Device> dev_;
};

}  // namespace pcs
