// dev_knobs.h — developer experiment knobs (environment variables).
//
// The shipped library reads NO environment variables: dev_knob() returns
// nullptr unless the library was compiled with -DPCSB_DEV_KNOBS, which only
// tools/build_variant.sh does (variants live under tools/bin/, selected with
// PCS_LOP_LIB for A/B runs).  The knobs and their measured defaults are listed
// in DESIGN.md §5b.
#pragma once

#include <cstdlib>

namespace pcsb {

inline const char* dev_knob(const char* name) {
#ifdef PCSB_DEV_KNOBS
    return std::getenv(name);
#else
    (void)name;
    return nullptr;
#endif
}

}  // namespace pcsb
