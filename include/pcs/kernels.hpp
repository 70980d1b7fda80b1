// kernels.hpp — weight-function parameters and the scalar weight functions.
// Semantics of proj/include/pcs/kernels.hpp:12-34 / proj/src/kernels.cpp:8-29:
// theta(d) = exp(-(d/h)^2), exactly 0 for d > h*cutoff_multiple;
// eta(d) = 1/(3 d^3); |eta'(d)| = 1/d^4.  The device kernels evaluate the same
// functions (lop_exact.cu in fp64, lop_fast.cu as 2^(...) on MUFU.EX2).
#pragma once

#include "pcs/errors.hpp"

namespace pcs {

struct KernelParams {
    double h = 1.0;
    double cutoff_multiple = 3.0;

    double support() const { return h * cutoff_multiple; }

    void validate() const {
        if (!(h > 0.0)) throw InvalidParam("kernel bandwidth h must be positive");
        if (!(cutoff_multiple > 0.0)) throw InvalidParam("kernel cutoff_multiple must be positive");
    }
};

double theta(double d, const KernelParams& params);
double eta(double d);
double eta_derivative_magnitude(double d);

}  // namespace pcs
