// sd_eig2.cuh — device-side 2x2 closed-form diagonalization
// (/root/reference/pkg/src/symdiag/eig2.py, cited as eig2.py:line).
#pragma once

#include "sd_math.cuh"

namespace sd {

constexpr double DEGENERACY_EPS_2 = 1e-14;  // eig2.py:14

// diagonalize2 (eig2.py:44-48) = eigenvalues2 (eig2.py:22-26) +
// rotation_angle2 (eig2.py:29-41); _sign(0) = +1 (eig2.py:17-19).
__device__ __forceinline__ uint8_t diagonalize2(double a11, double a12, double a22, double& l1,
                                                double& l2, double& phi) {
  if (!(is_finite(a11) && is_finite(a12) && is_finite(a22))) {
    l1 = l2 = phi = qnan();
    return SD_ERR_NONFINITE_INPUT;  // SymMat2 construction (core.py:62-63)
  }
  Err e;
  const double dd = a11 - a22;
  const double t = a11 + a22;
  const double sg = (dd < 0.0) ? -1.0 : 1.0;
  const double r = sg * py_hypot(dd, 2.0 * a12);
  // SymMat2.scale (core.py:68-73) gates the phi = 0 special case only
  // (eig2.py:37-39): eps = 1e-14 max(1, ||A||_F).  Its sqrt is needed only
  // when both |a11 - a22| and |a12| could be below eps, i.e. below
  // 1e-14 * sqrt(F) * (1 + 2^-40) — otherwise the gate is decided without it.
  const double fro2 = pow2(e, a11) + pow2(e, a22) + 2.0 * pow2(e, a12);
  const double m = pmax(fabs(dd), fabs(a12));
  bool zero_angle = false;
  if (m * m <= 1.0000000001e-28 * pmax(1.0, fro2) || m <= DEGENERACY_EPS_2) {
    const double eps = DEGENERACY_EPS_2 * pmax(1.0, py_sqrt(e, fro2));
    zero_angle = fabs(dd) <= eps && fabs(a12) <= eps;
  }
  double ph = 0.0;
  if (!zero_angle) {
    // wrap_half_pi of a value already in [-pi/2, pi/2]: remainder(x, pi) == x
    // exactly there, so only the -pi/2 -> pi/2 and -0 -> +0 rules remain
    ph = 0.5 * atan2(2.0 * a12 * sg, dd * sg);
    if (ph <= -0.5 * kPi) ph = 0.5 * kPi;
    if (ph == 0.0) ph = 0.0;
  }
  if (e.code) {
    l1 = l2 = phi = qnan();
    return (uint8_t)e.code;
  }
  l1 = 0.5 * (t + r);
  l2 = 0.5 * (t - r);
  phi = ph;
  return SD_CODE_GENERIC;
}

}  // namespace sd
