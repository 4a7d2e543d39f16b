// sv_score.cu -- K1 + K1e: steps a1-a3 of the SV hot path (P L159 S/A, P L164 divergence,
// north_star KL, P L176 profile lookup).
//
// Design (DESIGN.md §5 K1): a DECOUPLED two-pass reduction.  Row (b, i) is split into cs
// vocabulary chunks; each chunk is two tasks (one CTA each), taken in atomic-ticket order:
//   P1(row, r): stream the chunk pair from HBM (16-byte loads, L2 evict_last) and sum
//             l = sum 2^{(x - r) c} for draft and companion and the KL partial
//             w = sum e_d (a_d - a_c) against per-thread references r (the maxima of the thread's
//             first group: no running maximum -- a sum that is not finite sends the thread to the
//             exact path), packed FFMA2 / FADD2, 2 MUFU.EX2 per pair; block merge in fixed warp
//             order; publish (M_d, L_d, M_c, L_c, W) and bump the row's counter (release).
//   P2(row, r): wait for the row's cs P1 partials (acquire; issued ~lag rows earlier, so normally
//             already there), merge them in chunk order (the same bits in every P2 task of the
//             row), re-read the chunk pair -- an L2 hit (evict_first: last use) -- and sum
//             S_r = sum 2^{min(x_d c_d - Lambda_d, x_c c_c - Lambda_c)}, part of the 2^y on the
//             FMA pipe (ex2_poly2) and part on the MUFU; publish S_r.
// Task order interleaves P1 of row j + lag with P2 of row j, so the L2 holds ~lag rows between a
// chunk's two reads.  The row's last P2 task to finish runs the epilogue (S in chunk order, A, KL,
// profile lookup, draft normalisers for sd_verify).  HBM traffic is one read of D and C.  cs and
// the chunking depend on (V, dtype) only, so every reduction order -- and every output bit -- is
// independent of B and of the GPU count.
#include "sv_score_dev.cuh"

namespace sv {

SV_TRACE_DECL

namespace {

// K1: one CTA per chunk task, tasks taken from an atomic TICKET (not blockIdx): every task a P2
// task waits on has a lower ticket, i.e. it was taken earlier by a CTA that is already running,
// so forward progress needs no assumption about the order in which CTAs are dispatched; the CTA
// holding the last ticket re-arms the counter (self-cleaning workspace).  (A persistent grid
// with the next task's loads issued under the current task's tail measured 131-140 us vs 113 us
// here: a finished CTA's slot is refilled at once, while a persistent CTA's warps wait for its
// slowest warp at every task boundary.)
//   P1: pass 1 over the chunk pair (HBM; L2 evict_last: P2 re-reads it) -> block merge -> publish
//       (M_d, L_d, M_c, L_c, W), release the row counter;
//   P2: the first group of pass-2 loads (L2 hits; evict_first: last use) is issued BEFORE the
//       wait for / merge of the row's P1 partials, so the merge latency hides under the loads;
//       pass 2 -> S_r; the row's last P2 task to finish runs the epilogue.
template <typename T, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) sv_score_kernel(const __grid_constant__ ScoreArgs a) {
  constexpr int NW = NT / 32, G = kScoreGroup;
  __shared__ Smem<NW> sm;
  __shared__ uint32_t s_tk;
  pdl_wait();
  pdl_trigger();
  SV_TRACE_START(0);
  if (threadIdx.x == 0) {
    const uint32_t t = atomicAdd(a.ticket, 1u);
    if (t == gridDim.x - 1) *reinterpret_cast<volatile uint32_t *>(a.ticket) = 0u;  // the last claim
    s_tk = t;
  }
  __syncthreads();
  const float cd = a.cd, cc = a.cc;
  const TaskView<T> c = task_view<T>(a, s_tk);
  if (!c.k.p2) {
    const P1Out o = pass1_thread<T, NT, G>(c.src, c.ch, cd, cc);
    p1_publish<NW>(a, c.k, o, sm);
    SV_TRACE_END(0);
    SV_TRACE_END(13);  // P1 tasks: last exit
    return;
  }
  SV_TRACE_START(14);  // P2 tasks: first start
  Pre<G> pre;
  prefetch_first<T, NT, G>(c.src, c.ch, pre);
  const float2 lam = p2_merge_warp<NW>(a, c.k, sm);
  const float lamd = lam.x, lamc = lam.y;
  float s_loc = 0.f;
  if (lamd == lamd && lamc == lamc) s_loc = pass2_thread<T, NT, G, kScorePoly>(c.src, c.ch, cd, cc, lamd, lamc, &pre);
  p2_finish_head<NW>(s_loc, sm);
  p2_finish_tail<T, NW>(a, c.k, sm);
  SV_TRACE_END(0);
}

// K1c: one cluster of cs CTAs per row (CTA rank r = chunk r), both passes in one CTA: pass 1
// (HBM, L2 evict_last) -> block merge into shared memory -> cluster barrier -> every warp merges
// the cs chunk partials from the peers' shared memory (DSMEM) in chunk order -> pass 2 (the same
// chunk again, an L2 hit: it was read microseconds earlier) -> S partial -> cluster barrier ->
// rank 0 runs the row epilogue.  No ticket, no counters, no polling: a row's exchange is two
// cluster barriers, and clusters are independent of each other.  Every arithmetic step is the
// ticket kernel's (same chunking, per-thread units, warp / block / row merge orders, epilogue),
// so the outputs are bit-identical to it.
template <typename T, int NT, int MINB, bool kRes>
__global__ void __launch_bounds__(NT, MINB) sv_score_cluster_kernel(const __grid_constant__ ScoreArgs a) {
  constexpr int NW = NT / 32, G = kScoreGroup;
  __shared__ Smem<NW> sm;
  __shared__ uint64_t s_bar;
  extern __shared__ __align__(128) uint8_t s_chunk[];  // kRes: the chunk pair (D at 0, C at chunk bytes)
  pdl_wait();
  // No griddepcontrol.launch_dependents here: a PDL dependant launched early next to this
  // cluster grid ran ~5.5 us slower after its wait (traced: K3 1.8 -> 7.6 us at config 1); the
  // implicit trigger at grid completion costs ~0.7 us of launch latency instead.
  SV_TRACE_START(6);
  cg::cluster_group cl = cg::this_cluster();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const float cd = a.cd, cc = a.cc;
  Task k;
  k.q = blockIdx.x;
  k.row = k.q / (uint32_t)a.cs;
  k.rank = (int)(k.q - k.row * (uint32_t)a.cs);
  k.bb = k.row / (uint32_t)a.k;
  k.ii = k.row - k.bb * a.k;
  k.p2 = false;
  __shared__ EpiPre s_epi;
  // the epilogue's inputs (token, its logits, profile edges) now, off the row's critical path
  if (k.rank == 0 && wid == NW - 1) epilogue_prefetch<T>(a, k.bb, k.ii, s_epi);
  const Chunk<T> ch = chunk_of<T>(a, k.bb, k.ii, k.rank);
  float s_loc = 0.f;
  auto both_passes = [&](const auto &src1, const auto &src2, auto *pre) {
    const P1Out o = pass1_thread<T, NT, G>(src1, ch, cd, cc);
    p1_publish_head<NW>(o, sm, cd, cc);  // warp partials, block barrier
    if (wid == NW - 1) {                 // the chunk's (M_d, L_d, M_c, L_c, W): the NW warp partials merged
      auto warp_part = [&](int j) { return (const double *)(sm.dscr + 5 * j); };
      merge_partials_to<decltype(warp_part), false>(a, NW, warp_part, sm.glob, sm.lam);
    }
    if (pre) prefetch_first<T, NT, G>(src2, ch, *pre);
    SV_TRACE_POINT(8);
    cl.sync();  // every CTA's chunk partial is in its shared memory
    SV_TRACE_POINT(9);
    auto peer_part = [&](int j) { return (const double *)cl.map_shared_rank(&sm.glob[0], (unsigned)j); };
    merge_partials_to<decltype(peer_part), false>(a, a.cs, peer_part, sm.wglob[wid], sm.wlam[wid]);
    __syncwarp();
    const float lamd = sm.wlam[wid][0], lamc = sm.wlam[wid][1];
    if (lamd == lamd && lamc == lamc) s_loc = pass2_thread<T, NT, G, kScorePoly>(src2, ch, cd, cc, lamd, lamc, pre);
  };
  if constexpr (kRes) {  // one bulk copy per tensor from HBM; both passes read shared memory
    const uint32_t nb = (uint32_t)ch.units * 16u;
    if (threadIdx.x == 0) {
      mbar_init(&s_bar, 1);
      fence_mbar_init();
      if (nb) {
        const uint64_t pol = l2_policy_evict_first();
        mbar_arrive_expect_tx(&s_bar, 2 * nb);
        bulk_g2s(s_chunk, ch.d, nb, &s_bar, pol);
        bulk_g2s(s_chunk + a.chunk * sizeof(T), ch.c, nb, &s_bar, pol);
      }
    }
    __syncthreads();
    if (nb) mbar_wait_bounded(&s_bar, 0);
    SV_TRACE_POINT(7);
    const SSrc src{reinterpret_cast<const uint4 *>(s_chunk),
                   reinterpret_cast<const uint4 *>(s_chunk + a.chunk * sizeof(T))};
    both_passes(src, src, (Pre<G> *)nullptr);
  } else {
    Pre<G> pre;
    both_passes(GSrc<T>{ch.d, ch.c, l2_policy_evict_last()}, GSrc<T>{ch.d, ch.c, l2_policy_evict_first()}, &pre);
  }
  SV_TRACE_POINT(10);
  p2_finish_head<NW>(s_loc, sm);  // warp sums, block barrier
  __shared__ float s_spart[8];    // rank 0: the row's S partials in chunk order (pushed over DSMEM)
  if (wid == NW - 1 && lane == 0) {
    float r = sm.fscr[0];
    for (int w = 1; w < NW; ++w) r += sm.fscr[w];
    *cl.map_shared_rank(&s_spart[k.rank], 0u) = r;
  }
  cl.sync();  // S partials in rank 0 (and no CTA leaves while a peer may still read its glob)
  SV_TRACE_POINT(11);
  if (k.rank == 0 && wid == NW - 1) {
    __syncwarp();
    epilogue<T>(a, k.bb, k.ii, sm.wglob[NW - 1], s_spart, a.cs, 1, 0, nullptr, 0, &s_epi, true);
    if ((threadIdx.x & 31) == 0 && blockIdx.x == 0) SV_TRACE_POINT_ANY(12);
  }
  SV_TRACE_END(6);
}

template <typename T, bool kRes>
cudaError_t launch_score_cluster(const ScoreArgs &a, cudaStream_t st) {
  auto kern = sv_score_cluster_kernel<T, kScoreThreads, kScoreMinBlocks, kRes>;
  const size_t smem = kRes ? 2 * (size_t)a.chunk * sizeof(T) : 0;
  if (kRes) {
    const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((int64_t)a.B * a.k * a.cs));
  cfg.blockDim = dim3(kScoreThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  at[1].id = cudaLaunchAttributeClusterDimension;
  at[1].val.clusterDim.x = (unsigned)a.cs;
  at[1].val.clusterDim.y = 1;
  at[1].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, kern, a);
}

// Which K1 runs for a launch shape (all three give identical bits): the ticket kernel (0) for
// large inputs; K1c (1) when D + C is at most kScoreClusterMaxBytes -- a row's exchange is two
// cluster barriers instead of global counters, which pays while the grid is a few waves; its
// resident form (2) when the chunk pairs fit in shared memory and the grid is one wave.  cs <= 8
// (portable cluster size).  Measured per BASELINE config in DESIGN.md §5.
template <typename T>
int score_variant(const ScoreArgs &a) {
  if (SV_K1_VARIANT >= 0) return SV_K1_VARIANT;
  if (a.cs > 8) return 0;
  const int64_t rows = (int64_t)a.B * a.k, pair = 2 * a.chunk * (int64_t)sizeof(T);
  if (pair <= kScoreResMaxPairBytes) {
    auto kern = sv_score_cluster_kernel<T, kScoreThreads, kScoreMinBlocks, true>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pair) == cudaSuccess &&
        rows * a.cs <= resident_grid((const void *)kern, kScoreThreads, (int)pair))
      return 2;
    cudaGetLastError();
  }
  return rows * a.cs * pair <= kScoreClusterMaxBytes ? 1 : 0;
}

template <typename T>
cudaError_t launch_score_t(const ScoreArgs &a, cudaStream_t st) {
  if ((int64_t)a.B * a.k == 0) return cudaSuccess;
  switch (score_variant<T>(a)) {
    case 2: return launch_score_cluster<T, true>(a, st);
    case 1: return launch_score_cluster<T, false>(a, st);
    default: break;
  }
  const int64_t tasks = 2 * (int64_t)a.B * a.k * a.cs;
  if (tasks == 0) return cudaSuccess;
  return launch_k(sv_score_kernel<T, kScoreThreads, kScoreMinBlocks>, dim3((unsigned)tasks), dim3(kScoreThreads), 0,
                  st, a);
}

template <typename T>
cudaError_t launch_score_cfg(const ScoreArgs &a, cudaStream_t st) {
  return launch_score_t<T>(a, st);
}

// ---------------------------------------------------------------- vocab-sharded staging
// (BASELINE config 4).  Each rank holds columns [v_begin, v_begin + V_local) of
// every row (a.V = V_local, a.cs / a.chunk from V_local); the caller all-gathers the stage
// outputs between the calls.  Merges run over the G x cs chunk partials in (rank, chunk) =
// vocabulary order with the same arithmetic as K1, so every rank computes identical bits.
__device__ __forceinline__ Task shard_task(const ScoreArgs &a) {
  Task k;
  k.q = blockIdx.x;
  k.row = k.q / (uint32_t)a.cs;
  k.rank = (int)(k.q - k.row * (uint32_t)a.cs);
  k.bb = k.row / (uint32_t)a.k;
  k.ii = k.row - k.bb * a.k;
  k.p2 = false;
  return k;
}

// P1 of the rank's chunks: (M_d, L_d, M_c, L_c, W) per (row, chunk) -> part (a.part, no counter);
// chunk 0 also records the token logits x_d(t), x_c(t) when this rank owns t (NaN otherwise).
template <typename T, int NT>
__global__ void __launch_bounds__(NT) sv_shard_p1_kernel(const __grid_constant__ ScoreArgs a, int64_t v_begin,
                                                         float *xtok) {
  constexpr int NW = NT / 32;
  __shared__ Smem<NW> sm;
  pdl_wait();
  pdl_trigger();
  const Task k = shard_task(a);
  const Chunk<T> ch = chunk_of<T>(a, k.bb, k.ii, k.rank);
  const GSrc<T> src{ch.d, ch.c, l2_policy_evict_last()};
  const P1Out t = pass1_thread<T, NT, kScoreGroup>(src, ch, a.cd, a.cc);
  p1_publish<NW>(a, k, t, sm);
  if (k.rank == 0 && threadIdx.x == 0) {
    const int64_t loc = (int64_t)a.tok[k.row] - v_begin;
    float xd = __int_as_float(0x7fc00000), xc = xd;
    if (loc >= 0 && loc < a.V) {
      xd = Elem<T>::load(reinterpret_cast<const T *>(a.d) + (int64_t)k.bb * a.d_sb + (int64_t)k.ii * a.d_si + loc);
      xc = Elem<T>::load(reinterpret_cast<const T *>(a.c) + (int64_t)k.bb * a.c_sb + (int64_t)k.ii * a.c_si + loc);
    }
    xtok[(size_t)k.row * 2] = xd;
    xtok[(size_t)k.row * 2 + 1] = xc;
  }
}

// P2 of the rank's chunks: merge all G x cs partials (xall = [G][rows][cs][5]), then the S
// partial of this chunk -> sout[row][chunk].
template <typename T, int NT>
__global__ void __launch_bounds__(NT) sv_shard_p2_kernel(const __grid_constant__ ScoreArgs a, const double *xall,
                                                         int64_t gs_part, int G, float *sout) {
  constexpr int NW = NT / 32;
  __shared__ Smem<NW> sm;
  pdl_wait();
  pdl_trigger();
  const Task k = shard_task(a);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (wid == NW - 1)
    merge_partials<NW>(a, G * a.cs,
                       [&](int j) { return xall + (size_t)(j / a.cs) * gs_part + ((size_t)k.row * a.cs + j % a.cs) * 5; },
                       sm);
  __syncthreads();
  const float lamd = sm.lam[0], lamc = sm.lam[1];
  const Chunk<T> ch = chunk_of<T>(a, k.bb, k.ii, k.rank);
  float s_loc = 0.f;
  if (lamd == lamd && lamc == lamc)
    s_loc = pass2_thread<T, NT, kScoreGroup, kScorePoly>(GSrc<T>{ch.d, ch.c, l2_policy_evict_first()}, ch, a.cd, a.cc,
                                                         lamd, lamc);
  s_loc = warp_sum(s_loc);
  if (lane == 0) sm.fscr[wid] = s_loc;
  __syncthreads();
  if (threadIdx.x == 0) {
    float r = sm.fscr[0];
    for (int w = 1; w < NW; ++w) r += sm.fscr[w];
    sout[(size_t)k.row * a.cs + k.rank] = r;
  }
}

// Epilogue per row (one warp): the same merge, S over the G x cs partials (sall = [G][rows][cs]),
// token logits from their owner (xtok_all = [G][rows][2]); a.V is the GLOBAL vocabulary here.
template <typename T>
__global__ void __launch_bounds__(32) sv_shard_finish_kernel(const __grid_constant__ ScoreArgs a, const double *xall,
                                                             int64_t gs_part, const float *xtok_all, int64_t gs_tok,
                                                             const float *sall, int64_t gs_s, int G) {
  __shared__ Smem<1> sm;
  pdl_wait();
  pdl_trigger();
  const size_t row = blockIdx.x;
  merge_partials<1>(a, G * a.cs, [&](int j) { return xall + (size_t)(j / a.cs) * gs_part + (row * a.cs + j % a.cs) * 5; },
                    sm);
  __syncwarp();
  epilogue<T>(a, (int64_t)(row / a.k), (int64_t)(row % a.k), sm.glob, sall + row * a.cs, a.cs, G, gs_s,
              xtok_all + row * 2, gs_tok);
}

template <typename T>
cudaError_t shard_score_stage_t(const ShardScoreArgs &h, const ScoreArgs &a, cudaStream_t st) {
  const unsigned rows = (unsigned)((int64_t)a.B * a.k);
  if (rows == 0) return cudaSuccess;
  switch (h.stage) {
    case 0:
      return launch_k(sv_shard_p1_kernel<T, kScoreThreads>, dim3(rows * (unsigned)a.cs), dim3(kScoreThreads), 0, st, a,
                      h.v_begin, h.xtok_out);
    case 1:
      return launch_k(sv_shard_p2_kernel<T, kScoreThreads>, dim3(rows * (unsigned)a.cs), dim3(kScoreThreads), 0, st, a,
                      h.xall, h.gs_part, h.G, h.s_out);
    default:
      return launch_k(sv_shard_finish_kernel<T>, dim3(rows), dim3(32), 0, st, a, h.xall, h.gs_part, h.xtok_all, h.gs_tok,
                      h.sall, h.gs_s, h.G);
  }
}

}  // namespace

cudaError_t launch_score(const ScoreArgs &a, cudaStream_t st) {
  return a.bf16 ? launch_score_cfg<__nv_bfloat16>(a, st) : launch_score_cfg<float>(a, st);
}

cudaError_t launch_shard_score(const ShardScoreArgs &h, const ScoreArgs &a, cudaStream_t st) {
  return a.bf16 ? shard_score_stage_t<__nv_bfloat16>(h, a, st) : shard_score_stage_t<float>(h, a, st);
}

}  // namespace sv

SV_TRACE_READER(score)
