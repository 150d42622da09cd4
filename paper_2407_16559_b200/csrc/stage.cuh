// stage.cuh — the Runge-Kutta stage combinations x + tau * sum_j a_ij k_j of the reference
// steppers (steppers.cpp:98-159, tableau steppers.hpp:59-74), as ONE expression per kind shared
// by the stage-combination kernel (k_comb, steps.cu) and the RHS kernels that compute a stage
// on the fly from x and the k's instead of reading a materialised stage vector (fused stages):
// the same source expression in both places, so both produce the same bits.
#pragma once
#include <cuda_runtime.h>

namespace agk {

namespace rkf {
constexpr double a21 = 1.0 / 4.0;
constexpr double a31 = 3.0 / 32.0, a32 = 9.0 / 32.0;
constexpr double a41 = 1932.0 / 2197.0, a42 = -7200.0 / 2197.0, a43 = 7296.0 / 2197.0;
constexpr double a51 = 439.0 / 216.0, a52 = -8.0, a53 = 3680.0 / 513.0, a54 = -845.0 / 4104.0;
constexpr double a61 = -8.0 / 27.0, a62 = 2.0, a63 = -3544.0 / 2565.0, a64 = 1859.0 / 4104.0, a65 = -11.0 / 40.0;
constexpr double b5_0 = 16.0 / 135.0, b5_2 = 6656.0 / 12825.0, b5_3 = 28561.0 / 56430.0, b5_4 = -9.0 / 50.0,
                 b5_5 = 2.0 / 55.0;
constexpr double b4_0 = 25.0 / 216.0, b4_2 = 1408.0 / 2565.0, b4_3 = 2197.0 / 4104.0, b4_4 = -1.0 / 5.0;
}  // namespace rkf

enum CombKind {
  C_RK2_ST,   // x + t*y0                                    (steppers.cpp:103)
  C_RK2_OUT,  // x + 0.5*t*(y0 + y1)                         (steppers.cpp:105)
  C_RK4_STH,  // x + 0.5*t*y0                                (steppers.cpp:113,115)
  C_RK4_ST1,  // x + t*y0                                    (steppers.cpp:117)
  C_RK4_OUT,  // x + t*(y0 + 2 y1 + 2 y2 + y3)/6             (steppers.cpp:119-121)
  C_F2, C_F3, C_F4, C_F5, C_F6,                            // (steppers.cpp:130-147)
  C_F_OUT     // n4 (stored) and n5 (reduced / optional)     (steppers.cpp:149-158)
};

// stage-vector inputs of each combination
__host__ __device__ constexpr int comb_inputs(int kind) {
  return kind == C_RK2_ST || kind == C_RK4_STH || kind == C_RK4_ST1 || kind == C_F2 ? 1
         : kind == C_RK2_OUT || kind == C_F3                                      ? 2
         : kind == C_F4                                                           ? 3
         : kind == C_RK4_OUT || kind == C_F5                                      ? 4
                                                                                  : 5;  // C_F6, C_F_OUT
}

// The combination value for every kind but C_F_OUT (which also forms n5; see k_comb), in the
// reference's operation order with every rounding explicit (no FMA contraction: the reference is
// built without it), so a stage is bitwise the reference's for the same inputs and identical in
// every kernel that forms it.
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
template <int KIND>
__device__ __forceinline__ double comb_value(double t, double xi, const double* yy) {
  using namespace rkf;
  switch (KIND) {
    case C_RK2_ST: return dadd(xi, dmul(t, yy[0]));                                         // :103
    case C_RK2_OUT: return dadd(xi, dmul(dmul(0.5, t), dadd(yy[0], yy[1])));                 // :105
    case C_RK4_STH: return dadd(xi, dmul(dmul(0.5, t), yy[0]));                              // :113,115
    case C_RK4_ST1: return dadd(xi, dmul(t, yy[0]));                                         // :117
    case C_RK4_OUT:                                                                          // :119-121
      return dadd(xi, __ddiv_rn(dmul(t, dadd(dadd(dadd(yy[0], dmul(2.0, yy[1])), dmul(2.0, yy[2])), yy[3])), 6.0));
    case C_F2: return dadd(xi, dmul(dmul(t, a21), yy[0]));                                   // :130
    case C_F3: return dadd(xi, dmul(t, dadd(dmul(a31, yy[0]), dmul(a32, yy[1]))));            // :133
    case C_F4:                                                                               // :137
      return dadd(xi, dmul(t, dadd(dadd(dmul(a41, yy[0]), dmul(a42, yy[1])), dmul(a43, yy[2]))));
    case C_F5:                                                                               // :141
      return dadd(xi, dmul(t, dadd(dadd(dadd(dmul(a51, yy[0]), dmul(a52, yy[1])), dmul(a53, yy[2])),
                                   dmul(a54, yy[3]))));
    default:                                                                                 // C_F6 :145-146
      return dadd(xi, dmul(t, dadd(dadd(dadd(dadd(dmul(a61, yy[0]), dmul(a62, yy[1])), dmul(a63, yy[2])),
                                        dmul(a64, yy[3])),
                                   dmul(a65, yy[4]))));
  }
}

// RKF45's closing pair (steppers.cpp:149-152): n5 and n4 from k1, k3, k4, k5, k6 (yy[0..4])
__device__ __forceinline__ void comb_f_out(double t, double xi, const double* yy, double& n4, double& n5) {
  using namespace rkf;
  n5 = dadd(xi, dmul(t, dadd(dadd(dadd(dadd(dmul(b5_0, yy[0]), dmul(b5_2, yy[1])), dmul(b5_3, yy[2])),
                                  dmul(b5_4, yy[3])),
                             dmul(b5_5, yy[4]))));
  n4 = dadd(xi, dmul(t, dadd(dadd(dadd(dmul(b4_0, yy[0]), dmul(b4_2, yy[1])), dmul(b4_3, yy[2])), dmul(b4_4, yy[3]))));
}

// A stage as an RHS input (RhsArgs::st): n_i = comb_value<kind>(tau_mul * *tau, x_i, y_j[i]), x the
// RHS's own input VecRef. on == 0 (a zero-initialised StageIn): no stage, the input is read as is.
struct StageIn {
  int on;
  int kind;
  const double* y[5];
  const double* tau;  // the controller's current step size (device)
  double tau_mul;
};

template <int KIND>
__device__ __forceinline__ double stage_at_k(const StageIn& s, double t, double xi, int64_t i) {
  double yy[5];
#pragma unroll
  for (int j = 0; j < comb_inputs(KIND); ++j) yy[j] = s.y[j][i];
  return comb_value<KIND>(t, xi, yy);
}

// n_i of a fused stage (s.on), x_i given
__device__ __forceinline__ double stage_at(const StageIn& s, double t, double xi, int64_t i) {
  switch (s.kind) {
    case C_RK2_ST: return stage_at_k<C_RK2_ST>(s, t, xi, i);
    case C_RK4_STH: return stage_at_k<C_RK4_STH>(s, t, xi, i);
    case C_RK4_ST1: return stage_at_k<C_RK4_ST1>(s, t, xi, i);
    case C_F2: return stage_at_k<C_F2>(s, t, xi, i);
    case C_F3: return stage_at_k<C_F3>(s, t, xi, i);
    case C_F4: return stage_at_k<C_F4>(s, t, xi, i);
    case C_F5: return stage_at_k<C_F5>(s, t, xi, i);
    default: return stage_at_k<C_F6>(s, t, xi, i);
  }
}

}  // namespace agk
