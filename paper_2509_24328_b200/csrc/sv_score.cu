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

constexpr int kStages = 4;

struct ScoreSmemTail {
  uint64_t bars[kStages];
  double part[5];   // this CTA's (M_d, L_d, M_c, L_c, W) for the cluster merge
  double glob[5];   // merged values (broadcast to the CTA)
  float sarr[kMaxCluster];  // S partials (valid in rank 0)
  double dscr[3 * (kScoreThreads / 32)];
  float fscr[kScoreThreads / 32];
};

template <typename T, int EPU>
__device__ __forceinline__ void unpack(const T *base, int u, float (&x)[EPU]) {
  const uint4 v = *reinterpret_cast<const uint4 *>(base + (size_t)u * EPU);
  Elem<T>::unit(v, x);
}

// Phase-1 accumulation of EPU (d, c) pairs into the thread's online state.
template <int EPU>
__device__ __forceinline__ void accum_unit(const float (&xd)[EPU], const float (&xc)[EPU], int cnt, float cd,
                                           float cc, float &md, float &mc, float &nmd, float &nmc, double &ld,
                                           double &lc, double &w) {
  float vmd = xd[0], vmc = xc[0];
#pragma unroll
  for (int j = 1; j < EPU; ++j)
    if (j < cnt) {
      vmd = fmaxf(vmd, xd[j]);
      vmc = fmaxf(vmc, xc[j]);
    }
  const float nd = fmaxf(md, vmd), nc = fmaxf(mc, vmc);
  if (nd > md || nc > mc) {  // a running maximum moved: rescale exactly
    const float sdf = ex2((md - nd) * cd), scf = ex2((mc - nc) * cc);
    const float delta = (nc - mc) * cc - (nd - md) * cd;
    if (ld > 0.0) w += ld * (double)delta;
    w *= sdf;
    ld *= sdf;
    lc *= scf;
    md = nd;
    mc = nc;
    nmd = -md * cd;
    nmc = -mc * cc;
  }
  float ed[EPU], ec[EPU], wt[EPU];
#pragma unroll
  for (int j = 0; j < EPU; ++j) {
    const float ad = fmaf(xd[j], cd, nmd), ac = fmaf(xc[j], cc, nmc);
    ed[j] = (j < cnt) ? ex2(ad) : 0.f;
    ec[j] = (j < cnt) ? ex2(ac) : 0.f;
    // p_d = 0 terms contribute 0 even when a_d - a_c is -inf / NaN; a_c = -inf with
    // p_d > 0 keeps +inf (KL = +inf, correct).
    wt[j] = ed[j] * fmaxf(ad - ac, -FLT_MAX);
  }
#pragma unroll
  for (int s = 1; s < EPU; s <<= 1)
#pragma unroll
    for (int j = 0; j + s < EPU; j += 2 * s) {
      ed[j] += ed[j + s];
      ec[j] += ec[j + s];
      wt[j] += wt[j + s];
    }
  ld += ed[0];
  lc += ec[0];
  w += wt[0];
}

template <typename T>
__global__ void __launch_bounds__(kScoreThreads) sv_score_kernel(const ScoreArgs a) {
  constexpr int NT = kScoreThreads;
  constexpr int EPU = Elem<T>::kPerUnit;
  cg::cluster_group cluster = cg::this_cluster();
  const int cs = a.cs;
  const int rank = (int)cluster.block_rank();
  const int64_t row = blockIdx.x / cs;
  const int64_t b = row / a.k, i = row % a.k;
  const int64_t v0 = (int64_t)rank * a.chunk;
  const int n = (int)max((int64_t)0, min(a.chunk, (int64_t)a.V - v0));
  const int tid = threadIdx.x;

  extern __shared__ __align__(128) uint8_t smem[];
  const size_t cbytes = (size_t)a.chunk * sizeof(T);
  T *sd = reinterpret_cast<T *>(smem);
  T *sc = reinterpret_cast<T *>(smem + cbytes);
  ScoreSmemTail *tl = reinterpret_cast<ScoreSmemTail *>(smem + 2 * cbytes);

  const T *rowd = reinterpret_cast<const T *>(a.d) + b * a.d_sb + i * a.d_si;
  const T *rowc = reinterpret_cast<const T *>(a.c) + b * a.c_sb + i * a.c_si;
  const T *gd = rowd + v0, *gc = rowc + v0;
  const int units = n / EPU;
  const bool bulk = units > 0 && ((reinterpret_cast<uintptr_t>(gd) | reinterpret_cast<uintptr_t>(gc)) & 15) == 0;
  const int bulk_units = bulk ? units : 0;
  const int per_stage = (bulk_units + kStages - 1) / kStages;

  // rank 0 prefetches the token logits (independent loads, latency overlaps the stream)
  const int32_t t = a.tok[row];
  const bool tok_ok = t >= 0 && t < a.V;
  float xdt = 0.f, xct = 0.f;
  if (rank == 0 && tid == 0 && tok_ok) {
    xdt = Elem<T>::load(rowd + t);
    xct = Elem<T>::load(rowc + t);
  }

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&tl->bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0 && bulk) {
    for (int s = 0; s < kStages; ++s) {
      const int u0 = s * per_stage, u1 = min(bulk_units, u0 + per_stage);
      if (u1 <= u0) break;
      const uint32_t bytes = (uint32_t)(u1 - u0) * 16u;
      mbar_arrive_expect_tx(&tl->bars[s], 2u * bytes);
      bulk_g2s(sd + (size_t)u0 * EPU, gd + (size_t)u0 * EPU, bytes, &tl->bars[s]);
      bulk_g2s(sc + (size_t)u0 * EPU, gc + (size_t)u0 * EPU, bytes, &tl->bars[s]);
    }
  }
  for (int e = bulk_units * EPU + tid; e < n; e += NT) {  // unaligned rows / ragged tail
    sd[e] = gd[e];
    sc[e] = gc[e];
  }
  __syncthreads();

  const float cd = a.cd, cc = a.cc;
  float md = kMFloor, mc = kMFloor, nmd = -kMFloor * cd, nmc = -kMFloor * cc;
  double ld = 0.0, lc = 0.0, w = 0.0;
  int waited = -1;
  for (int u = tid; u < units; u += NT) {
    if (u < bulk_units) {
      const int s = u / per_stage;
      if (s != waited) {
        mbar_wait(&tl->bars[s], 0);
        waited = s;
      }
    }
    float xd[EPU], xc[EPU];
    unpack<T, EPU>(sd, u, xd);
    unpack<T, EPU>(sc, u, xc);
    accum_unit<EPU>(xd, xc, EPU, cd, cc, md, mc, nmd, nmc, ld, lc, w);
  }
  if (tid < n - units * EPU) {  // ragged tail: < EPU elements, one per thread
    float xd[EPU], xc[EPU];
    const int e = units * EPU + tid;
#pragma unroll
    for (int j = 0; j < EPU; ++j) {
      xd[j] = Elem<T>::load(sd + e);
      xc[j] = Elem<T>::load(sc + e);
    }
    accum_unit<EPU>(xd, xc, 1, cd, cc, md, mc, nmd, nmc, ld, lc, w);
  }

  // ---- block merge (fixed order)
  const float Md = block_max<NT>(md, tl->fscr);
  const float Mc = block_max<NT>(mc, tl->fscr);
  {
    const float sdf = ex2((md - Md) * cd), scf = ex2((mc - Mc) * cc);
    const float delta = (Mc - mc) * cc - (Md - md) * cd;
    double ww = w;
    if (ld > 0.0) ww += ld * (double)delta;
    double v[3] = {ld * sdf, lc * scf, ww * sdf};
    constexpr int NW = NT / 32;
    const int wid = tid >> 5, lane = tid & 31;
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
      tl->part[0] = Md;
      tl->part[1] = r[0];
      tl->part[2] = Mc;
      tl->part[3] = r[1];
      tl->part[4] = r[2];
    }
  }
  cluster.sync();  // (A) all partials visible cluster-wide

  // ---- cluster merge in rank order (identical in every CTA)
  if (tid == 0) {
    double pm[kMaxCluster][5];
    for (int r = 0; r < cs; ++r) {
      const double *rp = cluster.map_shared_rank(tl->part, r);
#pragma unroll
      for (int j = 0; j < 5; ++j) pm[r][j] = rp[j];
    }
    float GMd = (float)pm[0][0], GMc = (float)pm[0][2];
    for (int r = 1; r < cs; ++r) {
      GMd = fmaxf(GMd, (float)pm[r][0]);
      GMc = fmaxf(GMc, (float)pm[r][2]);
    }
    double L_d = 0.0, L_c = 0.0, W = 0.0;
    for (int r = 0; r < cs; ++r) {
      const float rmd = (float)pm[r][0], rmc = (float)pm[r][2];
      const float sdf = ex2((rmd - GMd) * cd), scf = ex2((rmc - GMc) * cc);
      const float delta = (GMc - rmc) * cc - (GMd - rmd) * cd;
      double ww = pm[r][4];
      if (pm[r][1] > 0.0) ww += pm[r][1] * (double)delta;
      L_d += pm[r][1] * sdf;
      L_c += pm[r][3] * scf;
      W += ww * sdf;
    }
    tl->glob[0] = GMd;
    tl->glob[1] = L_d;
    tl->glob[2] = GMc;
    tl->glob[3] = L_c;
    tl->glob[4] = W;
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
    if (tid < n - units * EPU) {
      const int e = units * EPU + tid;
      acc0 += ex2(fminf(fmaf(Elem<T>::load(sd + e), cd, -lamd), fmaf(Elem<T>::load(sc + e), cc, -lamc)));
    }
    s_loc = acc0 + acc1;
  }
  {
    float v[1] = {s_loc};
    block_sum<NT, 1>(v, tl->fscr);
    if (tid == 0) cluster.map_shared_rank(tl->sarr, 0)[rank] = v[0];
  }
  cluster.sync();  // (B) S partials landed in rank 0; no DSMEM access after this point

  if (rank != 0 || tid != 0) return;
  // ---- epilogue (rank 0, one thread, fp64)
  int st = 0;
  if (!row_ok) {
    const bool nan = !(L_d == L_d) || !(L_c == L_c) || !(GMd < FLT_MAX) || !(GMc < FLT_MAX) ||
                     !(L_d < 1e300) || !(L_c < 1e300);
    st |= nan ? 1 /*SV_ROW_NAN*/ : 2 /*SV_ROW_ALL_NEG_INF*/;
  }
  if (!tok_ok) st |= 4; /*SV_ROW_BAD_TOKEN*/
  double S = 0.0;
  for (int r = 0; r < cs; ++r) S += (double)tl->sarr[r];
  double A = 0.0, KL = 0.0, pdt = __longlong_as_double(0x7ff8000000000000LL);
  if (!st) {
    // e(t) with the same exponent shift as the row sums: x c - fl(m c)
    const double ld2 = log2(L_d), lc2 = log2(L_c);
    const double argd = (double)xdt * cd - (double)(GMd * cd) - ld2;
    const double argc = (double)xct * cc - (double)(GMc * cc) - lc2;
    pdt = exp2(argd);
    if (pdt == 0.0) {
      st |= 8; /*SV_ROW_DRAFT_ZERO*/
    } else {
      A = fmin(1.0, exp2(argc - argd));
      KL = 0.6931471805599453 * (tl->glob[4] / L_d) - log(L_d / L_c);
    }
  }
  const float nanf_ = __int_as_float(0x7fc00000);
  float phat = 0.f;
  if (!st) {
    const float Sf = (float)S, Af = (float)A;
    int si = 0, ai = 0;
    for (int j = 1; j < a.n_s; ++j) si += (a.s_edges[j] < Sf) ? 1 : 0;
    for (int j = 1; j < a.n_a; ++j) ai += (a.a_edges[j] < Af) ? 1 : 0;
    phat = a.cells[si * a.n_a + ai];
  }
  if (a.S) a.S[row] = st ? nanf_ : (float)S;
  if (a.A) a.A[row] = st ? nanf_ : (float)A;
  if (a.KL) a.KL[row] = st ? nanf_ : (float)KL;
  if (a.p_hat) a.p_hat[row] = phat;
  a.dm[row] = GMd;
  a.dl[row] = (st & 3) ? ((st & 1) ? nanf_ : 0.f) : (float)L_d;
  a.dpt[row] = (st & 8) ? 0.f : (st ? nanf_ : (float)pdt);
  if (a.status) a.status[row] = st;
}

}  // namespace

cudaError_t launch_score(const ScoreArgs &a, cudaStream_t st) {
  const int elem = a.bf16 ? 2 : 4;
  const size_t smem = 2 * (size_t)a.chunk * elem + sizeof(ScoreSmemTail);
  const void *fn = a.bf16 ? (const void *)sv_score_kernel<__nv_bfloat16> : (const void *)sv_score_kernel<float>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (a.cs > 8) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((int64_t)a.B * a.k * a.cs));
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
  if (a.bf16) return cudaLaunchKernelEx(&cfg, sv_score_kernel<__nv_bfloat16>, a);
  return cudaLaunchKernelEx(&cfg, sv_score_kernel<float>, a);
}

}  // namespace sv
