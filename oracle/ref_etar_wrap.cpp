// ref_etar_wrap.cpp — the reference's LOP with eta(r) = -r (|eta'| = 1).
//
// TEST INFRASTRUCTURE ONLY.  oracle/Makefile links the UNMODIFIED reference
// objects (proj/src/lop.cpp etc.) into oracle/_ref/libpcs_ref_etar.so with
//   -Wl,--wrap=_ZN3pcs24eta_derivative_magnitudeEd
// so that lop.cpp's one call of pcs::eta_derivative_magnitude
// (proj/src/lop.cpp:90-91, the repulsion weight theta(d)*|eta'(d)|/d) resolves
// to the function below instead of 1/d^4 (proj/src/kernels.cpp:23-29).
// Everything else — neighbour queries, anchor/isolation rules, Jacobi update,
// summary — is the reference's own code.  This pins the benchmark configs'
// eta = -r variant (configs 2-4) to the reference's control flow rather than
// to a restatement only.
#include <stdexcept>

#include "pcs/errors.hpp"

extern "C" double __wrap__ZN3pcs24eta_derivative_magnitudeEd(double d) {
    // same domain check as the reference's |eta'| (kernels.cpp:24-25)
    if (!(d > 0.0)) throw pcs::InvalidParam("eta_derivative_magnitude requires d > 0");
    return 1.0;
}
