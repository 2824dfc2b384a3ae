// Drop-in replacement header for the reference's specproj/qdwh.hpp (qdwh.hpp:1-305).
//
// Put  -I <repo>/include/specproj_b200/dropin  AHEAD of the reference's include
// directory and link libspecproj_b200.so: every  #include "specproj/qdwh.hpp"  then
// resolves here, and an unchanged call  specproj::hqdwh(A, n_min, eps, delta)
// (qdwh.hpp:196) runs the B200 projector.  Everything else of qdwh.hpp (QdwhParams,
// qdwh_params, l_update, dense_qdwh, dense_spectral_projector, error_metrics,
// ProjectorResult, IterationDiag, ...) is the reference's own code, included through
// #include_next; the reference's CPU hqdwh stays available as hqdwh_cpu_reference.
// Errors are the reference's exception types (NotPositiveDefiniteError, ...).
#pragma once

#define hqdwh hqdwh_cpu_reference
#include_next "specproj/qdwh.hpp"
#undef hqdwh

#ifndef SPECPROJ_B200_USE_REFERENCE_TYPES
#define SPECPROJ_B200_USE_REFERENCE_TYPES 1
#endif
#include "../../specproj.hpp"

namespace specproj {

// hqdwh (qdwh.hpp:196-241) on the B200
inline ProjectorResult hqdwh(const BandedSymmetric& A, int n_min, double eps, double delta) {
    return b200::hqdwh(A, n_min, eps, delta);
}

}  // namespace specproj
