// sv_score.cu -- K1: steps a1-a3 of the SV hot path for one (b, i) row pair per CTA
// cluster (P L159 S/A, P L164 divergence, north_star KL, P L176 profile lookup).
//
// Design (DESIGN.md §5 K1):
//  * One thread-block CLUSTER per (b, i); CTA r of the cluster owns vocabulary chunk
//    [r*chunk, (r+1)*chunk) of BOTH the draft and the companion row and keeps it in
//    shared memory for the whole kernel, so each logit is read from HBM exactly once.
//  * The chunk arrives through the bulk-copy (TMA) engine in 4 mbarrier stages; threads
//    start on stage 0 while later stages are in flight.
//  * Phase 1 (per thread, online): raw maxima m_d, m_c, l = sum 2^{(x-m) log2e/tau}, and
//    the KL partial w = sum e_d ((a_d) - (a_c)) in log2 units, rescaled exactly when a
//    maximum moves.  Per-unit fp32 sums feed fp64 per-thread accumulators.
//  * Block merge (fixed warp/lane order) -> cluster merge through DSMEM in rank order
//    (identical bits in every CTA) -> Lambda = m c + log2 l.
//  * Phase 2 over the chunk still in smem: S_r = sum 2^{min(x_d c_d - Lambda_d,
//    x_c c_c - Lambda_c)} (one MUFU per pair), pushed to rank 0's smem.
//  * Rank 0 epilogue (fp64): S, A = min(1, p_c(t)/p_d(t)), KL = ln2 w/l_d - ln(l_d/l_c),
//    bin lookup of (S, A) in the profile, draft normalisers for sd_verify.
#include <float.h>

#include "sv_device.cuh"
#include "sv_internal.h"

namespace sv {

namespace {

struct ScoreSmemTail {
  uint64_t bar[2];             // one "chunk landed" barrier per buffer
  double part[2][5];           // this CTA's (M_d, L_d, M_c, L_c, W) per buffer, for the cluster merge
  float sarr[2][kMaxCluster];  // S partials, per buffer (valid in the epilogue CTA)
  double glob[5];              // merged values (broadcast to the CTA)
  float fscr[2 * (kScoreThreads / 32)];
  double dscr[3 * (kScoreThreads / 32)];
};

template <typename T, int EPU>
__device__ __forceinline__ void unpack(const T *base, int u, float (&x)[EPU]) {
  const uint4 v = *reinterpret_cast<const uint4 *>(base + (size_t)u * EPU);
  Elem<T>::unit(v, x);
}

// Pass A: the thread's raw maxima over its units (packed bf16x2 max for bf16 data).
template <typename T>
__device__ __forceinline__ void thread_max(const T *sd, const T *sc, int units, float &md, float &mc) {
  constexpr int NT = kScoreThreads;
  if constexpr (sizeof(T) == 2) {
    __nv_bfloat162 pd = __halves2bfloat162(__ushort_as_bfloat16(0xFF80), __ushort_as_bfloat16(0xFF80));
    __nv_bfloat162 pc = pd;
    for (int u = threadIdx.x; u < units; u += NT) {
      const uint4 vd = *reinterpret_cast<const uint4 *>(sd + (size_t)u * 8);
      const uint4 vc = *reinterpret_cast<const uint4 *>(sc + (size_t)u * 8);
      pd = __hmax2(__hmax2(pd, *reinterpret_cast<const __nv_bfloat162 *>(&vd.x)),
                   __hmax2(*reinterpret_cast<const __nv_bfloat162 *>(&vd.y),
                           __hmax2(*reinterpret_cast<const __nv_bfloat162 *>(&vd.z),
                                   *reinterpret_cast<const __nv_bfloat162 *>(&vd.w))));
      pc = __hmax2(__hmax2(pc, *reinterpret_cast<const __nv_bfloat162 *>(&vc.x)),
                   __hmax2(*reinterpret_cast<const __nv_bfloat162 *>(&vc.y),
                           __hmax2(*reinterpret_cast<const __nv_bfloat162 *>(&vc.z),
                                   *reinterpret_cast<const __nv_bfloat162 *>(&vc.w))));
    }
    md = fmaxf(md, fmaxf(__low2float(pd), __high2float(pd)));
    mc = fmaxf(mc, fmaxf(__low2float(pc), __high2float(pc)));
  } else {
    for (int u = threadIdx.x; u < units; u += NT) {
      float xd[4], xc[4];
      unpack<T, 4>(sd, u, xd);
      unpack<T, 4>(sc, u, xc);
      md = fmaxf(md, fmaxf(fmaxf(xd[0], xd[1]), fmaxf(xd[2], xd[3])));
      mc = fmaxf(mc, fmaxf(fmaxf(xc[0], xc[1]), fmaxf(xc[2], xc[3])));
    }
  }
}

// Pass B: sums of 2^{a} and the KL partial sum e_d (a_d - a_c) against the thread's fixed
// maxima.  kGuard = false is the fast path; a NaN partial (only possible from 0 * (-inf)
// when the row holds -inf logits) is recomputed with kGuard = true.
template <typename T, bool kGuard>
__device__ __forceinline__ void thread_sums(const T *sd, const T *sc, int units, int n, float cd, float cc,
                                            float nmd, float nmc, float &ld, float &lc, float &w) {
  constexpr int NT = kScoreThreads, EPU = Elem<T>::kPerUnit;
  float ld0 = 0.f, ld1 = 0.f, lc0 = 0.f, lc1 = 0.f, w0 = 0.f, w1 = 0.f;
  for (int u = threadIdx.x; u < units; u += NT) {
    float xd[EPU], xc[EPU];
    unpack<T, EPU>(sd, u, xd);
    unpack<T, EPU>(sc, u, xc);
#pragma unroll
    for (int j = 0; j < EPU; j += 2) {
      const float ad0 = fmaf(xd[j], cd, nmd), ac0 = fmaf(xc[j], cc, nmc);
      const float ad1 = fmaf(xd[j + 1], cd, nmd), ac1 = fmaf(xc[j + 1], cc, nmc);
      const float ed0 = ex2(ad0), ec0 = ex2(ac0), ed1 = ex2(ad1), ec1 = ex2(ac1);
      ld0 += ed0;
      lc0 += ec0;
      ld1 += ed1;
      lc1 += ec1;
      if (kGuard) {
        w0 += ed0 > 0.f ? ed0 * (ad0 - ac0) : 0.f;
        w1 += ed1 > 0.f ? ed1 * (ad1 - ac1) : 0.f;
      } else {
        w0 = fmaf(ed0, ad0 - ac0, w0);
        w1 = fmaf(ed1, ad1 - ac1, w1);
      }
    }
  }
  const int e = units * EPU + threadIdx.x;  // ragged tail: < EPU elements, one per thread
  if (e < n) {
    const float ad = fmaf(Elem<T>::load(sd + e), cd, nmd), ac = fmaf(Elem<T>::load(sc + e), cc, nmc);
    const float ed = ex2(ad);
    ld0 += ed;
    lc0 += ex2(ac);
    if (kGuard)
      w0 += ed > 0.f ? ed * (ad - ac) : 0.f;
    else
      w0 = fmaf(ed, ad - ac, w0);
  }
  ld = ld0 + ld1;
  lc = lc0 + lc1;
  w = w0 + w1;
}

// Persistent kernel: a cluster owns rows cid, cid + ncl, ... and keeps two chunk buffers,
// so the bulk copy of row j + 1 is in flight while row j is being reduced.
template <typename T>
__global__ void __launch_bounds__(kScoreThreads, 1) sv_score_kernel(const ScoreArgs a) {
  constexpr int NT = kScoreThreads, NW = NT / 32;
  constexpr int EPU = Elem<T>::kPerUnit;
  cg::cluster_group cluster = cg::this_cluster();
  const int cs = a.cs;
  const int rank = (int)cluster.block_rank();
  const int64_t cid = blockIdx.x / cs, ncl = gridDim.x / cs;
  const int64_t rows = (int64_t)a.B * a.k;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t v0 = (int64_t)rank * a.chunk;
  const int n = (int)max((int64_t)0, min(a.chunk, (int64_t)a.V - v0));
  const int units = n / EPU;
  const float cd = a.cd, cc = a.cc;

  extern __shared__ __align__(128) uint8_t smem[];
  T *buf = reinterpret_cast<T *>(smem);  // [2 buffers][d, c][chunk]
  ScoreSmemTail *tl = reinterpret_cast<ScoreSmemTail *>(smem + 4 * (size_t)a.chunk * sizeof(T));

  auto drow = [&](int64_t row) {
    return reinterpret_cast<const T *>(a.d) + (row / a.k) * a.d_sb + (row % a.k) * a.d_si;
  };
  auto crow = [&](int64_t row) {
    return reinterpret_cast<const T *>(a.c) + (row / a.k) * a.c_sb + (row % a.k) * a.c_si;
  };
  auto bulk_ok = [&](int64_t row) {
    return units > 0 && ((reinterpret_cast<uintptr_t>(drow(row) + v0) | reinterpret_cast<uintptr_t>(crow(row) + v0)) &
                         15) == 0;
  };
  // tid 0: start the chunk pair of `row` into buffer `bs` (every use of a barrier completes
  // one phase: a row without bulk-eligible alignment just arrives)
  auto issue = [&](int64_t row, int bs) {
    uint64_t *bar = &tl->bar[bs];
    if (!bulk_ok(row)) {
      mbar_arrive(bar);
      return;
    }
    T *sd = buf + (size_t)(2 * bs) * a.chunk, *sc = sd + a.chunk;
    const T *gd = drow(row) + v0, *gc = crow(row) + v0;
    fence_proxy_async();  // order earlier generic-proxy smem accesses before the async writes
    mbar_arrive_expect_tx(bar, 2u * (uint32_t)units * 16u);
    constexpr int kPieces = 4;
    const int per = (units + kPieces - 1) / kPieces;
    for (int s = 0; s < kPieces; ++s) {
      const int u0 = s * per, u1 = min(units, u0 + per);
      if (u1 <= u0) break;
      const uint32_t bytes = (uint32_t)(u1 - u0) * 16u;
      bulk_g2s(sd + (size_t)u0 * EPU, gd + (size_t)u0 * EPU, bytes, bar);
      bulk_g2s(sc + (size_t)u0 * EPU, gc + (size_t)u0 * EPU, bytes, bar);
    }
  };

  if (tid == 0) {
    mbar_init(&tl->bar[0], 1);
    mbar_init(&tl->bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0 && cid < rows) issue(cid, 0);

  int it = 0;
  for (int64_t row = cid; row < rows; row += ncl, ++it) {
    const int bs = it & 1;
    T *sd = buf + (size_t)(2 * bs) * a.chunk, *sc = sd + a.chunk;
    if (tid == 0 && row + ncl < rows) issue(row + ncl, bs ^ 1);  // prefetch the next row
    const T *rowd = drow(row), *rowc = crow(row);
    const int bu = bulk_ok(row) ? units : 0;
    for (int e = bu * EPU + tid; e < n; e += NT) {  // unaligned rows / ragged tail
      sd[e] = rowd[v0 + e];
      sc[e] = rowc[v0 + e];
    }
    const int epi = it % cs;  // the epilogue rotates over the cluster's CTAs
    const int32_t t = a.tok[row];
    const bool tok_ok = t >= 0 && t < a.V;
    float xdt = 0.f, xct = 0.f;
    if (rank == epi && tid == 0 && tok_ok) {  // token logits: independent loads, latency hidden
      xdt = Elem<T>::load(rowd + t);
      xct = Elem<T>::load(rowc + t);
    }
    __syncthreads();
    mbar_wait(&tl->bar[bs], (it >> 1) & 1);

    // ---- pass A: thread maxima; pass B: sums against them
    float md = kMFloor, mc = kMFloor;
    thread_max<T>(sd, sc, units, md, mc);
    {
      const int e = units * EPU + tid;
      if (e < n) {
        md = fmaxf(md, Elem<T>::load(sd + e));
        mc = fmaxf(mc, Elem<T>::load(sc + e));
      }
    }
    const float nmd = -md * cd, nmc = -mc * cc;
    float lf_d, lf_c, wf;
    thread_sums<T, false>(sd, sc, units, n, cd, cc, nmd, nmc, lf_d, lf_c, wf);
    if (wf != wf && lf_d == lf_d && lf_c == lf_c)  // 0 * (-inf) from masked logits: guarded redo
      thread_sums<T, true>(sd, sc, units, n, cd, cc, nmd, nmc, lf_d, lf_c, wf);

    // ---- block merge (fixed warp / lane order)
    float Md = warp_max(md), Mc = warp_max(mc);
    if (lane == 0) {
      tl->fscr[wid] = Md;
      tl->fscr[NW + wid] = Mc;
    }
    __syncthreads();
    Md = tl->fscr[0];
    Mc = tl->fscr[NW];
#pragma unroll
    for (int q = 1; q < NW; ++q) {
      Md = fmaxf(Md, tl->fscr[q]);
      Mc = fmaxf(Mc, tl->fscr[NW + q]);
    }
    {
      const float sdf = ex2((md - Md) * cd), scf = ex2((mc - Mc) * cc);
      const float delta = (Mc - mc) * cc - (Md - md) * cd;
      double ww = wf;
      if (lf_d > 0.f) ww += (double)lf_d * (double)delta;
      double v[3] = {(double)lf_d * sdf, (double)lf_c * scf, ww * sdf};
#pragma unroll
      for (int j = 0; j < 3; ++j) v[j] = warp_sum_d(v[j]);
      if (lane == 0)
#pragma unroll
        for (int j = 0; j < 3; ++j) tl->dscr[j * NW + wid] = v[j];
      __syncthreads();
      if (tid == 0) {
        double r[3];
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          r[j] = tl->dscr[j * NW];
          for (int q = 1; q < NW; ++q) r[j] += tl->dscr[j * NW + q];
        }
        double *pp = tl->part[bs];
        pp[0] = Md;
        pp[1] = r[0];
        pp[2] = Mc;
        pp[3] = r[1];
        pp[4] = r[2];
      }
    }
    cluster.sync();  // (A) partials of this row visible cluster-wide

    // ---- cluster merge in rank order (identical in every CTA): lane r of warp 0 fetches
    // rank r's partial through DSMEM (one round trip), shuffles combine them in rank order
    if (wid == 0) {
      double pr[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
      pr[0] = pr[2] = kMFloor;
      if (lane < cs) {
        const double *rp = cluster.map_shared_rank(&tl->part[bs][0], lane);
#pragma unroll
        for (int j = 0; j < 5; ++j) pr[j] = rp[j];
      }
      const float rmd = (float)pr[0], rmc = (float)pr[2];
      const float GMd = warp_max(rmd), GMc = warp_max(rmc);
      const float sdf = ex2((rmd - GMd) * cd), scf = ex2((rmc - GMc) * cc);
      const float delta = (GMc - rmc) * cc - (GMd - rmd) * cd;
      double ww = pr[4];
      if (pr[1] > 0.0) ww += pr[1] * (double)delta;
      const double cl_d = pr[1] * sdf, cl_c = pr[3] * scf, cw = ww * sdf;
      double L_d = 0.0, L_c = 0.0, W = 0.0;
      for (int r = 0; r < cs; ++r) {  // rank order
        L_d += __shfl_sync(0xffffffffu, cl_d, r);
        L_c += __shfl_sync(0xffffffffu, cl_c, r);
        W += __shfl_sync(0xffffffffu, cw, r);
      }
      if (lane == 0) {
        tl->glob[0] = GMd;
        tl->glob[1] = L_d;
        tl->glob[2] = GMc;
        tl->glob[3] = L_c;
        tl->glob[4] = W;
      }
    }
    __syncthreads();
    const float GMd = (float)tl->glob[0], GMc = (float)tl->glob[2];
    const double L_d = tl->glob[1], L_c = tl->glob[3];
    const bool row_ok = L_d > 0.0 && L_c > 0.0 && L_d < 1e300 && L_c < 1e300 && GMd < FLT_MAX && GMc < FLT_MAX;

    // ---- phase 2: S partial over the chunk still resident in smem
    float s_loc = 0.f;
    if (row_ok) {
      const float lamd = (float)((double)GMd * cd + log2(L_d));
      const float lamc = (float)((double)GMc * cc + log2(L_c));
      float acc0 = 0.f, acc1 = 0.f;
      for (int u = tid; u < units; u += NT) {
        float xd[EPU], xc[EPU];
        unpack<T, EPU>(sd, u, xd);
        unpack<T, EPU>(sc, u, xc);
#pragma unroll
        for (int j = 0; j < EPU; j += 2) {
          acc0 += ex2(fminf(fmaf(xd[j], cd, -lamd), fmaf(xc[j], cc, -lamc)));
          acc1 += ex2(fminf(fmaf(xd[j + 1], cd, -lamd), fmaf(xc[j + 1], cc, -lamc)));
        }
      }
      const int e = units * EPU + tid;
      if (e < n)
        acc0 += ex2(fminf(fmaf(Elem<T>::load(sd + e), cd, -lamd), fmaf(Elem<T>::load(sc + e), cc, -lamc)));
      s_loc = acc0 + acc1;
    }
    {
      float v = warp_sum(s_loc);
      if (lane == 0) tl->fscr[wid] = v;
      __syncthreads();
      if (tid == 0) {
        float r = tl->fscr[0];
        for (int q = 1; q < NW; ++q) r += tl->fscr[q];
        cluster.map_shared_rank(&tl->sarr[bs][0], epi)[rank] = r;
      }
    }
    cluster.sync();  // (B) S partials landed in the epilogue CTA; buffer bs is free again

    if (rank != epi || wid != 0) continue;
    // ---- epilogue (one warp of one CTA, fp64, independent pieces on separate lanes).  The
    // draft-side outputs depend on the draft row alone: a bad companion row does not poison them.
    auto row_bits = [](double L, float M) {
      if (!(L == L) || !(L < 1e300) || !(M < FLT_MAX)) return 1; /*SV_ROW_NAN*/
      return (L > 0.0) ? 0 : 2;                                  /*SV_ROW_ALL_NEG_INF*/
    };
    const int d_st = row_bits(L_d, GMd), c_st = row_bits(L_c, GMc);
    int st = d_st | c_st | (tok_ok ? 0 : 4 /*SV_ROW_BAD_TOKEN*/);
    xdt = __shfl_sync(0xffffffffu, xdt, 0);
    xct = __shfl_sync(0xffffffffu, xct, 0);
    double piece = 0.0;  // lane 0: log2 p_d(t); lane 1: log2 p_c(t); lane 2: ln(L_d / L_c); lane 3: S
    if (lane == 0 && !d_st && tok_ok) piece = (double)xdt * cd - (double)(GMd * cd) - log2(L_d);
    if (lane == 1 && !st) piece = (double)xct * cc - (double)(GMc * cc) - log2(L_c);
    if (lane == 2 && !st) piece = log(L_d / L_c);
    if (lane == 3)
      for (int r = 0; r < cs; ++r) piece += (double)tl->sarr[bs][r];
    const double argd = __shfl_sync(0xffffffffu, piece, 0);
    double piece2 = 0.0;  // lane 0: p_d(t); lane 1: A (before min)
    if (lane == 0 && !d_st && tok_ok) piece2 = exp2(argd);
    if (lane == 1 && !st) piece2 = exp2(piece - argd);
    const double pdt = __shfl_sync(0xffffffffu, piece2, 0);
    const double Ar = __shfl_sync(0xffffffffu, piece2, 1);
    const double lnr = __shfl_sync(0xffffffffu, piece, 2);
    const double S = __shfl_sync(0xffffffffu, piece, 3);
    if (!d_st && tok_ok && pdt == 0.0) st |= 8; /*SV_ROW_DRAFT_ZERO*/
    double A = 0.0, KL = 0.0;
    if (!st) {
      A = fmin(1.0, Ar);
      KL = 0.6931471805599453 * (tl->glob[4] / L_d) - lnr;
      if (KL > 1e20) KL = __longlong_as_double(0x7ff0000000000000LL);  // p_c = 0 where p_d > 0
    }
    float phat = 0.f;
    if (!st && a.p_hat) {  // bin = number of interior edges strictly below the value (R9)
      const float Sf = (float)S, Af = (float)A;
      int si = 0, ai = 0;
      for (int j = lane + 1; j < a.n_s; j += 32) si += (a.s_edges[j] < Sf) ? 1 : 0;
      for (int j = lane + 1; j < a.n_a; j += 32) ai += (a.a_edges[j] < Af) ? 1 : 0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        si += __shfl_xor_sync(0xffffffffu, si, o);
        ai += __shfl_xor_sync(0xffffffffu, ai, o);
      }
      phat = a.cells[si * a.n_a + ai];
    }
    if (lane == 0) {
      const float nanf_ = __int_as_float(0x7fc00000);
      if (a.S) a.S[row] = st ? nanf_ : (float)S;
      if (a.A) a.A[row] = st ? nanf_ : (float)A;
      if (a.KL) a.KL[row] = st ? nanf_ : (float)KL;
      if (a.p_hat) a.p_hat[row] = phat;
      a.dm[row] = GMd;
      a.dl[row] = (d_st & 1) ? nanf_ : ((d_st & 2) ? 0.f : (float)L_d);
      a.dpt[row] = (d_st || !tok_ok) ? nanf_ : (float)pdt;
      if (a.status) a.status[row] = st;
    }
  }
}

}  // namespace

cudaError_t launch_score(const ScoreArgs &a, cudaStream_t st) {
  const int elem = a.bf16 ? 2 : 4;
  const size_t smem = 4 * (size_t)a.chunk * elem + sizeof(ScoreSmemTail);
  const void *fn = a.bf16 ? (const void *)sv_score_kernel<__nv_bfloat16> : (const void *)sv_score_kernel<float>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (a.cs > 8) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(kScoreThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = a.cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // persistent grid: as many clusters as can be co-resident (never more than rows)
  const int64_t rows = (int64_t)a.B * a.k;
  int ncl = max_active_clusters(fn, cfg, (int)smem, a.cs);
  if ((int64_t)ncl > rows) ncl = (int)rows;
  cfg.gridDim = dim3((unsigned)(ncl * a.cs));
  if (a.bf16) return cudaLaunchKernelEx(&cfg, sv_score_kernel<__nv_bfloat16>, a);
  return cudaLaunchKernelEx(&cfg, sv_score_kernel<float>, a);
}

}  // namespace sv
