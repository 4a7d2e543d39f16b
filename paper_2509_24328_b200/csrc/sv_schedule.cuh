// sv_schedule.cuh -- step a4 for one sequence (P L207-239, §5; DESIGN R2-R4), shared by the
// K3 kernel and sv_score_schedule's fused K1 epilogue.  One thread walks j = 0..k left to right
// in fp64 with explicitly rounded operations (__dmul_rn / __dadd_rn / __ddiv_rn: no FMA
// contraction), so gamma, E and g are bit-identical to the oracle's sequential evaluation.
//   P_j = P_{j-1} p_j, E_j = E_{j-1} + P_j (P L231-234, S L378),
//   g_j = (E_j + plus_one) / L[j + plus_one]      (P L211, L236; R2),
//   gamma = smallest argmax_j g_j (strict '>' while scanning; S L396).
// p_hat is read through L2 (__ldcg): in the fused path other CTAs wrote it.
#pragma once

#include <float.h>

#include "sv_internal.h"

namespace sv {

constexpr int kSchedMaxK = 16;  // SV_MAX_K

// p_hat is an acceptance probability (P L176): outside [0, 1] (NaN, inf, negative, > 1) it is
// used as 0 and flagged SV_ROW_PHAT_BAD (DESIGN R22)
__device__ __forceinline__ double phat_val(float v, int &st) {
  if (!(v >= 0.f && v <= 1.f)) {
    st |= 16;
    return 0.0;
  }
  return (double)v;
}

__device__ __forceinline__ void schedule_one(const ScheduleArgs &a, int64_t b) {
  const int k = a.k, po = a.plus_one ? 1 : 0;
  // all loads up front (k <= SV_MAX_K): the fp64 chain below then never waits on memory
  float ph[kSchedMaxK];
  double Lj[kSchedMaxK + 1];
#pragma unroll
  for (int j = 0; j < kSchedMaxK; ++j) ph[j] = j < k ? __ldcg(a.p_hat + b * k + j) : 0.f;
#pragma unroll
  for (int j = 0; j <= kSchedMaxK; ++j) Lj[j] = j <= k ? a.L[j + po] : 1.0;
  int st = 0;
#pragma unroll
  for (int j = 0; j <= kSchedMaxK; ++j) {
    if (j <= k && (!(Lj[j] > 0.0) || !(Lj[j] <= DBL_MAX))) st |= 128;  // SV_ROW_BAD_LATENCY
  }
  if (st) {
    a.gamma[b] = 0;
    if (a.exp_accept) a.exp_accept[b] = 0.f;
    if (a.goodput) a.goodput[b] = __int_as_float(0x7fc00000);
    if (a.status) a.status[b] = st;
    return;
  }
  double P = 1.0, E = 0.0;
  double best_g = __ddiv_rn(po ? 1.0 : 0.0, Lj[0]);
  double best_E = 0.0;
  int best = 0;
#pragma unroll
  for (int j = 1; j <= kSchedMaxK; ++j) {
    if (j > k) break;
    P = __dmul_rn(P, phat_val(ph[j - 1], st));
    E = __dadd_rn(E, P);
    const double g = __ddiv_rn(po ? __dadd_rn(E, 1.0) : E, Lj[j]);
    if (g > best_g) {
      best_g = g;
      best_E = E;
      best = j;
    }
  }
  a.gamma[b] = best;
  if (a.exp_accept) a.exp_accept[b] = (float)best_E;
  if (a.goodput) a.goodput[b] = (float)best_g;
  if (a.status) a.status[b] = st;
}

}  // namespace sv
