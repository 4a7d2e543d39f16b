// sv_step.cu -- the fused small-batch step (sv_step): sv_score -> sv_schedule (per row) ->
// sd_verify of one sequence in ONE thread-block cluster of k R CTAs (R CTAs per draft position i,
// each taking every R-th of the row's cs chunks), phases separated by cluster barriers instead of
// kernel boundaries:
//   A  score row (b, i): K1's pass 1 over the CTA's chunks (the same 256-thread mapping, block
//      merge and published chunk partials as a P1 task), the row merge, pass 2 per chunk (the S
//      partials of the P2 tasks), the row epilogue (sv_score_dev.cuh);
//   B  CTA 0: the per-row schedule of sequence b (sv_schedule.cuh);
//   C  target rows 0..gamma_b: K4's (row, split) items over the cluster's warps;
//   D  CTA 0: the row merges and accept tests (K4b, sd_verify_dev.cuh);
//   E  every CTA: slice masses of row N_b (K5 warp items);
//   F  CTA 0: the token search (K5b).
// Every phase runs the three-kernel path's device code on the same data in the same order, so
// every output bit equals sv_score + sv_schedule + sd_verify_ragged on the same inputs; the only
// change is where the phases meet (cluster barriers: release / acquire at cluster scope, all data
// crossing CTAs goes through global memory exactly as between the kernels).  A sequence never
// waits on another, so clusters need no co-residency.  For small batches the step is a chain of
// dependent phases, each short: one launch instead of six removes five kernel boundaries.
#include <cooperative_groups.h>
#include <float.h>

#include "sd_verify_dev.cuh"
#include "sv_schedule.cuh"
#include "sv_score_dev.cuh"

namespace sv {

namespace {

namespace cg = cooperative_groups;

#ifndef SV_STEP_TRACE
#define SV_STEP_TRACE 0  // timing experiment only: %globaltimer after each phase, CTA (0, 0)
#endif
#if SV_STEP_TRACE
__device__ unsigned long long g_step_trace[8];
#define STEP_MARK(i)                                                                    \
  if (blockIdx.x == 0 && threadIdx.x == 0) {                                          \
    unsigned long long t;                                                             \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));                             \
    g_step_trace[i] = t;                                                              \
  }
#else
#define STEP_MARK(i)
#endif

template <typename T>
__global__ void __launch_bounds__(kScoreThreads) sv_step_kernel(const __grid_constant__ ScoreArgs sa,
                                                                 const __grid_constant__ ScheduleArgs ha,
                                                                 const __grid_constant__ VerifyArgs va, int R) {
  constexpr int NT = kScoreThreads, NW = NT / 32, G = kScoreGroup;
  __shared__ Smem<NW> sm;
  __shared__ float s_M[SV_MAX_K_DEV + 1];
  __shared__ double s_L[SV_MAX_K_DEV + 1];
  cg::cluster_group cl = cg::this_cluster();
  const int k = sa.k, cs = sa.cs;
  const int ncta = k * R;                     // the cluster: R CTAs per draft position
  const int rank = (int)cl.block_rank();
  const int pos = rank / R, h = rank % R;     // draft position i, share h of its chunks
  const int64_t b = blockIdx.x / ncta;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t row = b * k + pos;
  const float cd = sa.cd, cc = sa.cc;
  pdl_wait();
  pdl_trigger();
  STEP_MARK(0);

  // ---- A: score row (b, pos) -- K1's P1 tasks (chunks h, h + R, ...), row merge, P2 tasks,
  // epilogue (CTA h = 0 of the row)
  for (int r = h; r < cs; r += R) {
    const Chunk<T> ch = chunk_of<T>(sa, b, pos, r);
    const P1Out o = pass1_thread<T, NT, G>(GSrc<T>{ch.d, ch.c, l2_policy_evict_last()}, ch, cd, cc);
    p1_publish_head<NW>(o, sm, cd, cc);  // warp partials -> sm.dscr (block barrier)
    if (wid == NW - 1) {  // p1_publish_tail's merge, published without a counter
      auto warp_part = [&](int j) { return (const double *)(sm.dscr + 5 * j); };
      merge_partials_to<decltype(warp_part), false>(sa, NW, warp_part, sm.glob, sm.lam);
      __syncwarp();
      if (lane == 0) {
        double *part = sa.part + ((size_t)row * cs + r) * 5;
#pragma unroll
        for (int j = 0; j < 5; ++j) part[j] = sm.glob[j];
      }
    }
    __syncthreads();
  }
  if (R > 1) cl.sync();  // the row's other chunk partials
  if (wid == NW - 1)     // the row's merge (every P2 task's, sv_score_dev.cuh)
    merge_partials_to(sa, cs, [&](int j) { return sa.part + ((size_t)row * cs + j) * 5; }, sm.wglob[NW - 1],
                      sm.wlam[NW - 1]);
  __syncthreads();
  const float lamd = sm.wlam[NW - 1][0], lamc = sm.wlam[NW - 1][1];
  float *srow = sa.spart + (size_t)row * cs;
  for (int r = h; r < cs; r += R) {
    const Chunk<T> ch = chunk_of<T>(sa, b, pos, r);
    float s_loc = 0.f;
    if (lamd == lamd && lamc == lamc)
      s_loc = pass2_thread<T, NT, G, kScorePoly>(GSrc<T>{ch.d, ch.c, l2_policy_evict_first()}, ch, cd, cc, lamd, lamc);
    p2_finish_head<NW>(s_loc, sm);  // warp sums -> sm.fscr (block barrier)
    if (threadIdx.x == 0) {         // p2_finish_tail's S partial
      float s = sm.fscr[0];
      for (int w = 1; w < NW; ++w) s += sm.fscr[w];
      srow[r] = s;
    }
    __syncthreads();
  }
  if (R > 1) cl.sync();  // the row's other S partials
  if (h == 0 && wid == NW - 1) epilogue<T>(sa, b, pos, sm.wglob[NW - 1], srow, cs, 1, 0, nullptr, 0);
  cl.sync();
  STEP_MARK(1);

  // ---- B: the schedule of sequence b (its k p_hat values are in global memory)
  if (rank == 0 && threadIdx.x == 0) schedule_one(ha, b);
  cl.sync();
  STEP_MARK(2);

  // ---- C: target rows 0..gamma_b, K4's (row, split) items spread over the cluster's warps
  const int g = __ldcg(va.gamma + b);
  const bool gok = g >= 0 && g <= k;
  if (gok) {
    const int64_t items = (int64_t)(g + 1) * va.splits;
    for (int64_t it = (int64_t)rank * NW + wid; it < items; it += (int64_t)ncta * NW) {
      const int i = (int)(it / va.splits);
      const int64_t s = it - (int64_t)i * va.splits;
      const float2 p = rows_warp_item<T>(va, b, i, s);
      if (lane == 0) va.partials[(b * (k + 1) + i) * va.splits + s] = p;
    }
  }
  cl.sync();
  STEP_MARK(3);

  // ---- D: the row merges and accept tests (K4b) -> the sequence's Decision
  if (rank == 0) {
    if (gok)
      for (int i = wid; i <= g; i += NW) {
        float M;
        double L;
        merge_row_warp(va, b, i, M, L);
        if (lane == 0) {
          s_M[i] = M;
          s_L[i] = L;
        }
      }
    __syncthreads();
    if (wid == 0) {
      const bool in = gok && lane <= g;
      decide_warp<T>(va, b, g, in ? s_M[lane] : kMFloor, in ? s_L[lane] : 0.0);
    }
  }
  cl.sync();
  STEP_MARK(4);

  // ---- E: slice masses of row N_b (K5 warp items), spread over the cluster
  const Decision dc = va.dec[b];
  if (!dc.st)
    for (int64_t s = (int64_t)rank * NW + wid; s < va.nsl; s += (int64_t)ncta * NW) resid_item<T>(va, dc, b, s);
  cl.sync();
  STEP_MARK(5);

  // ---- F: the token search (K5b)
  if (rank == 0 && wid == 0) find_seq<T>(va, b);
  STEP_MARK(6);
}

// R = CTAs per draft position: as many of the row's cs chunks in parallel as a cluster of at
// most kStepMaxCluster CTAs allows (R divides cs, so every CTA of a row takes cs / R chunks)
template <typename T>
cudaError_t launch_step_t(const ScoreArgs &sa, const ScheduleArgs &ha, const VerifyArgs &va, cudaStream_t st) {
  const void *fn = (const void *)sv_step_kernel<T>;
  int R = 1;
  while (R * 2 * sa.k <= kStepMaxCluster && sa.cs % (R * 2) == 0) R *= 2;
  if (sa.k * R > 8) {
    const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((int64_t)sa.B * sa.k * R));
  cfg.blockDim = dim3(kScoreThreads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)(sa.k * R);
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, sv_step_kernel<T>, sa, ha, va, R);
}

}  // namespace

#if SV_STEP_TRACE
extern "C" __attribute__((visibility("default"))) int sv_debug_step_trace(void *host) {
  return (int)cudaMemcpyFromSymbol(host, g_step_trace, sizeof(g_step_trace));
}
#endif
cudaError_t launch_step(const ScoreArgs &sa, const ScheduleArgs &ha, const VerifyArgs &va, cudaStream_t st) {
  return sa.bf16 ? launch_step_t<__nv_bfloat16>(sa, ha, va, st) : launch_step_t<float>(sa, ha, va, st);
}

}  // namespace sv
