// Smallest-eigenvalue driver on the GPU determinant: the reference's secant
// root finder on P(x) = det(M - xI) (/root/reference/proj/src/secant.cpp:27-117),
// restated over a DetEvaluator that calls the B200 LDL^T engine with the
// bit-exact determinant fold.  Same iterates, same stopping rule (top `digits`
// significant decimals of successive iterates agree; the reference uses 15),
// same error protocol (NoProgress / SignViolation / RootHitAtPrecision).
#pragma once
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

#include "bigz.h"

namespace hgpu {

// Errors of the secant protocol (errors.hpp:60-80, secant.hpp:30-38).
struct SecantError : std::runtime_error {
  enum Kind { NoProgress, SignViolation, RootHitAtPrecision, ZeroPivot } kind;
  Z probe;          // RootHitAtPrecision
  long pivot = -1;  // ZeroPivot
  SecantError(Kind k, const std::string& w) : std::runtime_error(w), kind(k) {}
};

struct SecantIterate {
  Z x, det;  // mantissas at K bits
};

struct SecantTrace {
  std::vector<SecantIterate> iterates;
  bool converged = false, exact_root_hit = false;
  long iterations = 0;
  const Z& eigenvalue() const { return iterates.back().x; }
};

// det(M - xI) mantissa at K bits; throws SecantError{ZeroPivot} with the
// pivot index on a zero pivot.
using DetFn = std::function<Z(const Z& x)>;

// initial_points (secant.cpp:7-16): x1 = -max(1, trunc(min(1, M00) / 2^16)).
Z secant_x1(const Z& m00, long k);

SecantTrace secant_smallest_eigenvalue(long n, const Z& m00, const DetFn& det,
                                       long k, int digits,
                                       const Z* accepted_root = nullptr);

}  // namespace hgpu
