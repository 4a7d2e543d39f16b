// sv_schedule.cu -- K3: step a4, verification length per sequence (P L207-252, §5).
//
// PER_ROW: one thread per sequence walks j = 0..k left to right in fp64 with explicitly
// rounded operations (__dmul_rn / __dadd_rn / __ddiv_rn: no FMA contraction), so gamma,
// E and g are bit-identical to the oracle's sequential evaluation (DESIGN R4).
//   P_j = P_{j-1} p_j, E_j = E_{j-1} + P_j (P L231-234, S L378),
//   g_j = (E_j + plus_one) / L[j + plus_one]      (P L211, L236; R2),
//   gamma = smallest argmax_j g_j (strict '>' while scanning; S L396).
// BATCH_GREEDY (NEXT-1, P L247-252; S L402-417; R16, R17): one CTA.  The greedy order
// of the paper equals sorting all B*k candidate tokens by (gain desc, seq asc, pos asc)
// because each sequence's gains P_j are non-increasing in j; the stop rule is evaluated
// on the sorted prefix sums (fp64, same association as the sequential greedy).
#include <float.h>

#include "sv_device.cuh"
#include "sv_internal.h"
#include "sv_schedule.cuh"

namespace sv {

SV_TRACE_DECL

namespace {

__global__ void __launch_bounds__(128) sv_schedule_row_kernel(const __grid_constant__ ScheduleArgs a) {
  pdl_wait();
  pdl_trigger();
  SV_TRACE_START(1);
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < a.B) schedule_one(a, b);
  SV_TRACE_END(1);
}

}  // namespace

cudaError_t launch_schedule_greedy(const ScheduleArgs &a, cudaStream_t st);  // sv_greedy.cu

cudaError_t launch_schedule(const ScheduleArgs &a, cudaStream_t st) {
  if (a.mode == 1) return launch_schedule_greedy(a, st);
  const int nt = 128;
  return launch_k(sv_schedule_row_kernel, dim3((a.B + nt - 1) / nt), dim3(nt), 0, st, a);
}

}  // namespace sv

SV_TRACE_READER(sched)
