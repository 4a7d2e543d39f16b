// sv_score.cu -- K1: steps a1-a3 of the SV hot path (P L159 S/A, P L164 divergence,
// north_star KL, P L176 profile lookup).
//
// Design (DESIGN.md §5 K1).  One thread-block CLUSTER of cs CTAs per (b, i): CTA r owns the
// vocabulary chunk [r*chunk, (r+1)*chunk) of BOTH the draft and the companion row and keeps it in
// shared memory for the whole kernel, so every logit crosses HBM exactly once.
//   load    : the chunk pair arrives through the bulk-copy (TMA) engine (one mbarrier)
//   pass A  : thread maxima on packed bf16x2 (HMNMX2)
//   pass B  : l = sum 2^{(x - m) log2e / tau} and the KL partial w = sum e_d (a_d - a_c)
//             (log2 units) with packed fp32x2 FFMA2 / FADD2 -- two logits per instruction
//   merge   : block merge in fixed warp order, then a cluster barrier and a DSMEM gather of the
//             cs partials in rank order (identical bits in every CTA) -> Lambda = m c + log2 l
//   phase 2 : S_r = sum 2^{min(x_d c_d - Lambda_d, x_c c_c - Lambda_c)} over the chunk still
//             resident in smem (one MUFU per pair), pushed into rank 0's smem
//   epilogue: rank 0 (one warp, fp64): S, A = min(1, p_c(t)/p_d(t)), KL, profile lookup,
//             draft normalisers for sd_verify.
// The cluster size is the smallest power of two that fits the (draft, companion) row pair in
// the on-chip budget, a function of (V, dtype) only, so every reduction order -- and therefore
// every output bit -- is independent of B and of how a batch is split across GPUs.
#include <float.h>

#include "sv_device.cuh"
#include "sv_internal.h"

namespace sv {

namespace {

template <int NT>
struct ScoreTail {
  uint64_t bar;
  double part[kMaxCluster][5];  // (M_d, L_d, M_c, L_c, W) of every rank, pushed by the ranks
  double glob[5];           // merged values
  float lam[2];             // Lambda_d, Lambda_c
  float sarr[kMaxCluster];  // S partials (valid in rank 0)
  float fscr[2 * (NT / 32)];
  double dscr[3 * (NT / 32)];
};

__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// ---------------------------------------------------------------- pass B arithmetic
struct P1 {
  f2 ld, lc;  // l_d, l_c partials, two lanes each
  f2 w;       // KL partial, two lanes
};

__device__ __forceinline__ void p1_pair(f2 xd, f2 xc, f2 cdd, f2 ccc, f2 nmdd, f2 nmcc, P1 &acc) {
  const f2 ad = fma2(xd, cdd, nmdd), ac = fma2(xc, ccc, nmcc);
  const f2 ed = ex2x2(ad), ec = ex2x2(ac);
  acc.ld = add2(acc.ld, ed);
  acc.lc = add2(acc.lc, ec);
  acc.w = fma2(ed, sub2(ad, ac), acc.w);
}

template <typename T>
__device__ __forceinline__ void p1_unit(const uint4 &ud, const uint4 &uc, f2 cdd, f2 ccc, f2 nmdd, f2 nmcc,
                                        P1 &acc) {
  if constexpr (sizeof(T) == 2) {  // 8 bf16: lane pairs (x_2j, x_2j+1) share an FFMA2
    const uint32_t wd[4] = {ud.x, ud.y, ud.z, ud.w}, wc[4] = {uc.x, uc.y, uc.z, uc.w};
#pragma unroll
    for (int p = 0; p < 4; ++p)
      p1_pair(f2{bf_lo(wd[p]), bf_hi(wd[p])}, f2{bf_lo(wc[p]), bf_hi(wc[p])}, cdd, ccc, nmdd, nmcc, acc);
  } else {
    p1_pair(f2{__uint_as_float(ud.x), __uint_as_float(ud.y)}, f2{__uint_as_float(uc.x), __uint_as_float(uc.y)}, cdd,
            ccc, nmdd, nmcc, acc);
    p1_pair(f2{__uint_as_float(ud.z), __uint_as_float(ud.w)}, f2{__uint_as_float(uc.z), __uint_as_float(uc.w)}, cdd,
            ccc, nmdd, nmcc, acc);
  }
}

// element-wise (ragged tail / unaligned rows / guarded redo): p_d = 0 terms add 0 to w
__device__ __forceinline__ void p1_one(float xd, float xc, float cd, float cc, float nmd, float nmc, P1 &acc) {
  const float ad = fmaf(xd, cd, nmd), ac = fmaf(xc, cc, nmc);
  const float ed = ex2(ad);
  acc.ld.x += ed;
  acc.lc.x += ex2(ac);
  acc.w.x += ed > 0.f ? ed * (ad - ac) : 0.f;
}

__device__ __forceinline__ void umax(__nv_bfloat162 &m, const uint4 &v) {
  const __nv_bfloat162 *p = reinterpret_cast<const __nv_bfloat162 *>(&v);
  m = __hmax2(__hmax2(m, p[0]), __hmax2(p[1], __hmax2(p[2], p[3])));
}

// phase-2 arithmetic on one 16-byte unit of each tensor
template <typename T>
__device__ __forceinline__ void p2_unit(const uint4 &ud, const uint4 &uc, f2 cdd, f2 ccc, f2 lamdd, f2 lamcc,
                                        f2 &acc) {
  auto pair = [&](f2 xd, f2 xc) {
    const f2 ad = fma2(xd, cdd, lamdd), ac = fma2(xc, ccc, lamcc);
    acc = add2(acc, f2{ex2(fminf(ad.x, ac.x)), ex2(fminf(ad.y, ac.y))});
  };
  if constexpr (sizeof(T) == 2) {
    const uint32_t wd[4] = {ud.x, ud.y, ud.z, ud.w}, wc[4] = {uc.x, uc.y, uc.z, uc.w};
#pragma unroll
    for (int p = 0; p < 4; ++p) pair(f2{bf_lo(wd[p]), bf_hi(wd[p])}, f2{bf_lo(wc[p]), bf_hi(wc[p])});
  } else {
    pair(f2{__uint_as_float(ud.x), __uint_as_float(ud.y)}, f2{__uint_as_float(uc.x), __uint_as_float(uc.y)});
    pair(f2{__uint_as_float(ud.z), __uint_as_float(ud.w)}, f2{__uint_as_float(uc.z), __uint_as_float(uc.w)});
  }
}

// Values the epilogue needs from global memory, loaded by rank 0's warp 0 at kernel start so
// their latency hides under the streaming phases.
struct EpiPre {
  int32_t t;
  float xdt, xct;       // draft / companion logit of the draft token (lanes 0 / 1)
  float se[2], ae[2];   // interior profile edges j = lane + 1 and lane + 33 (+inf past the end)
};

template <typename T>
__device__ __forceinline__ EpiPre epi_prefetch(const ScoreArgs &a, int64_t row) {
  const int lane = threadIdx.x & 31;
  const int64_t b = row / a.k, i = row % a.k;
  EpiPre p;
  p.t = a.tok[row];
  p.xdt = p.xct = 0.f;
  const bool tok_ok = p.t >= 0 && p.t < a.V;
  if (lane == 0 && tok_ok) p.xdt = Elem<T>::load(reinterpret_cast<const T *>(a.d) + b * a.d_sb + i * a.d_si + p.t);
  if (lane == 1 && tok_ok) p.xct = Elem<T>::load(reinterpret_cast<const T *>(a.c) + b * a.c_sb + i * a.c_si + p.t);
  const float inf = __int_as_float(0x7f800000);
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int j = lane + 1 + 32 * h;
    p.se[h] = (a.p_hat && j < a.n_s) ? a.s_edges[j] : inf;
    p.ae[h] = (a.p_hat && j < a.n_a) ? a.a_edges[j] : inf;
  }
  return p;
}

// Epilogue of one row (warp 0 of rank 0; independent pieces on separate lanes, fp64 range
// reduction + fp32 transcendentals).  The draft-side outputs depend on the draft row alone: a bad
// companion row does not poison them.
template <int NT>
__device__ __noinline__ void epilogue(const ScoreArgs &a, int64_t row, const ScoreTail<NT> *tl, int cs,
                                      const EpiPre &pre) {
  const int lane = threadIdx.x & 31;
  const float cd = a.cd, cc = a.cc;
  const float GMd = (float)tl->glob[0], GMc = (float)tl->glob[2];
  const double L_d = tl->glob[1], L_c = tl->glob[3], W = tl->glob[4];
  auto row_bits = [](double L, float M) {
    if (!(L == L) || !(L < 1e300) || !(M < FLT_MAX)) return 1; /*SV_ROW_NAN*/
    return (L > 0.0) ? 0 : 2;                                  /*SV_ROW_ALL_NEG_INF*/
  };
  const int d_st = row_bits(L_d, GMd), c_st = row_bits(L_c, GMc);
  const bool tok_ok = pre.t >= 0 && pre.t < a.V;
  int st = d_st | c_st | (tok_ok ? 0 : 4 /*SV_ROW_BAD_TOKEN*/);
  // lane 0: log2 p_d(t); lane 1: log2 p_c(t); lane 2: log2 L_d - log2 L_c; lane 3: S (rank order)
  double piece = 0.0;
  if (lane == 0 && !d_st && tok_ok) piece = (double)pre.xdt * cd - (double)(GMd * cd) - log2_acc(L_d);
  if (lane == 1 && !st) piece = (double)pre.xct * cc - (double)(GMc * cc) - log2_acc(L_c);
  if (lane == 2 && !st) piece = log2_acc(L_d) - log2_acc(L_c);
  if (lane == 3)
    for (int r = 0; r < cs; ++r) piece += (double)tl->sarr[r];
  const double argd = __shfl_sync(0xffffffffu, piece, 0);
  double piece2 = 0.0;  // lane 0: p_d(t); lane 1: p_c(t) / p_d(t)
  if (lane == 0 && !d_st && tok_ok) piece2 = exp2_acc(argd);
  if (lane == 1 && !st) piece2 = exp2_acc(piece - argd);
  const double pdt = __shfl_sync(0xffffffffu, piece2, 0);
  const double Ar = __shfl_sync(0xffffffffu, piece2, 1);
  const double l2r = __shfl_sync(0xffffffffu, piece, 2);
  const double S = __shfl_sync(0xffffffffu, piece, 3);
  if (!d_st && tok_ok && pdt == 0.0) st |= 8; /*SV_ROW_DRAFT_ZERO*/
  double A = 0.0, KL = 0.0;
  if (!st) {
    A = fmin(1.0, Ar);
    KL = 0.6931471805599453 * (W / L_d - l2r);
    if (KL > 1e20) KL = __longlong_as_double(0x7ff0000000000000LL);  // p_c = 0 where p_d > 0
  }
  float phat = 0.f;
  if (!st && a.p_hat) {  // bin = number of interior edges strictly below the value (R9)
    const float Sf = (float)S, Af = (float)A;
    int si = (pre.se[0] < Sf) + (pre.se[1] < Sf), ai = (pre.ae[0] < Af) + (pre.ae[1] < Af);
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

#ifdef SV_TRACE
__device__ unsigned long long *g_trace = nullptr;  // debug builds only: [cta][8] timestamps
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define TR(k) \
  if (trp && threadIdx.x == blockDim.x - 32) trp[(size_t)blockIdx.x * 12 + (k)] = gtime();
#else
#define TR(k)
#endif

template <typename T, int NT>
__global__ void __launch_bounds__(NT, 1024 / NT) sv_score_kernel(const ScoreArgs a) {
#ifdef SV_TRACE
  unsigned long long *const trp = g_trace;  // loaded once
#endif
  TR(0);
  cluster_arrive();  // (0) this CTA has started: peers may write its shared memory after wait (0)
  EpiPre pre{};
  constexpr int NW = NT / 32, EPU = Elem<T>::kPerUnit;
  cg::cluster_group cluster = cg::this_cluster();
  const int cs = a.cs;
  const int rank = (int)cluster.block_rank();
  const int64_t row = blockIdx.x / cs;
  const int64_t b = row / a.k, i = row % a.k;
  const int64_t v0 = (int64_t)rank * a.chunk;
  const int n = (int)max((int64_t)0, min(a.chunk, (int64_t)a.V - v0));
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  // Serial per-CTA work (bulk-copy issue, merges, epilogue) runs on the LAST warp: the warp
  // arbiter favours high warp ids, so the critical path is not starved by co-resident compute.
  const bool ctl = wid == NW - 1;
  const float cd = a.cd, cc = a.cc;

  extern __shared__ __align__(128) uint8_t smem[];
  const size_t cbytes = (size_t)a.chunk * sizeof(T);
  T *sd = reinterpret_cast<T *>(smem);
  T *sc = reinterpret_cast<T *>(smem + cbytes);
  ScoreTail<NT> *tl = reinterpret_cast<ScoreTail<NT> *>(smem + 2 * cbytes);

  const T *gd = reinterpret_cast<const T *>(a.d) + b * a.d_sb + i * a.d_si + v0;
  const T *gc = reinterpret_cast<const T *>(a.c) + b * a.c_sb + i * a.c_si + v0;
  const bool al = ((reinterpret_cast<uintptr_t>(gd) | reinterpret_cast<uintptr_t>(gc)) & 15) == 0;
  if (rank == 0 && ctl) pre = epi_prefetch<T>(a, row);
  const int units = al ? n / EPU : 0;  // 16-byte units moved by the bulk-copy engine
  const int e0 = units * EPU;          // elements [e0, n) are handled element-wise

  if (ctl && lane == 0) {
    mbar_init(&tl->bar, 1);
    fence_mbar_init();
    if (units > 0) {
      const uint32_t bytes = (uint32_t)units * 16u;
      mbar_arrive_expect_tx(&tl->bar, 2u * bytes);
      const uint32_t half = (bytes / 2) / 16 * 16;  // two pieces per tensor
      bulk_g2s(sd, gd, half, &tl->bar);
      bulk_g2s(sc, gc, half, &tl->bar);
      if (bytes > half) {
        bulk_g2s(reinterpret_cast<uint8_t *>(sd) + half, reinterpret_cast<const uint8_t *>(gd) + half, bytes - half,
                 &tl->bar);
        bulk_g2s(reinterpret_cast<uint8_t *>(sc) + half, reinterpret_cast<const uint8_t *>(gc) + half, bytes - half,
                 &tl->bar);
      }
    }
  }
  for (int e = e0 + tid; e < n; e += NT) {  // ragged tail / unaligned rows
    sd[e] = gd[e];
    sc[e] = gc[e];
  }
  __syncthreads();
  if (units > 0) mbar_wait(&tl->bar, 0);
  TR(1);

  // ---- pass A: thread maxima
  float md = kMFloor, mc = kMFloor;
  if constexpr (sizeof(T) == 2) {
    __nv_bfloat162 pd = __halves2bfloat162(__ushort_as_bfloat16(0xFF80), __ushort_as_bfloat16(0xFF80));
    __nv_bfloat162 pc = pd;
#pragma unroll 4
    for (int u = tid; u < units; u += NT) {
      umax(pd, reinterpret_cast<const uint4 *>(sd)[u]);
      umax(pc, reinterpret_cast<const uint4 *>(sc)[u]);
    }
    md = fmaxf(md, fmaxf(__low2float(pd), __high2float(pd)));
    mc = fmaxf(mc, fmaxf(__low2float(pc), __high2float(pc)));
  } else {
#pragma unroll 4
    for (int u = tid; u < units; u += NT) {
      const float4 xd = reinterpret_cast<const float4 *>(sd)[u], xc = reinterpret_cast<const float4 *>(sc)[u];
      md = fmaxf(md, fmaxf(fmaxf(xd.x, xd.y), fmaxf(xd.z, xd.w)));
      mc = fmaxf(mc, fmaxf(fmaxf(xc.x, xc.y), fmaxf(xc.z, xc.w)));
    }
  }
  for (int e = e0 + tid; e < n; e += NT) {
    md = fmaxf(md, Elem<T>::load(sd + e));
    mc = fmaxf(mc, Elem<T>::load(sc + e));
  }
  // ---- pass B: sums against the thread maxima
  const float nmd = -md * cd, nmc = -mc * cc;
  P1 acc{{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};
  {
    const f2 cdd{cd, cd}, ccc{cc, cc}, nmdd{nmd, nmd}, nmcc{nmc, nmc};
#pragma unroll 2
    for (int u = tid; u < units; u += NT)
      p1_unit<T>(reinterpret_cast<const uint4 *>(sd)[u], reinterpret_cast<const uint4 *>(sc)[u], cdd, ccc, nmdd, nmcc,
                 acc);
  }
  for (int e = e0 + tid; e < n; e += NT) p1_one(Elem<T>::load(sd + e), Elem<T>::load(sc + e), cd, cc, nmd, nmc, acc);
  float lf_d = acc.ld.x + acc.ld.y, lf_c = acc.lc.x + acc.lc.y, wf = acc.w.x + acc.w.y;
  if (wf != wf && lf_d == lf_d && lf_c == lf_c) {  // 0 * (-inf) from masked logits: guarded redo
    P1 g{{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};      // (same elements per thread as the fast path)
    for (int u = tid; u < units; u += NT)
      for (int j = 0; j < EPU; ++j)
        p1_one(Elem<T>::load(sd + u * EPU + j), Elem<T>::load(sc + u * EPU + j), cd, cc, nmd, nmc, g);
    for (int e = e0 + tid; e < n; e += NT) p1_one(Elem<T>::load(sd + e), Elem<T>::load(sc + e), cd, cc, nmd, nmc, g);
    lf_d = g.ld.x;
    lf_c = g.lc.x;
    wf = g.w.x;
  }

  TR(2);
  cluster_wait();  // (0) every peer CTA has started (completes at once by now): DSMEM pushes are safe
  // ---- block merge (fixed warp / lane order)
  {
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
    if (ctl) {  // control warp: lanes 0..2 sum the 3 quantities over warps (in warp order)
      double r = 0.0;
      if (lane < 3)
        for (int q = 0; q < NW; ++q) r += tl->dscr[lane * NW + q];
      const double r1 = __shfl_sync(0xffffffffu, r, 1), r2 = __shfl_sync(0xffffffffu, r, 2);
      const double r0 = __shfl_sync(0xffffffffu, r, 0);
      if (lane < cs) {  // push this CTA's partial into slot [rank] of every CTA of the cluster
        double *dst = cluster.map_shared_rank(&tl->part[rank][0], lane);
        dst[0] = Md;
        dst[1] = r0;
        dst[2] = Mc;
        dst[3] = r1;
        dst[4] = r2;
      }
    }
  }
  TR(3);
  cluster_arrive();  // (A) partials of this CTA published
  cluster_wait();
  TR(4);

  // ---- cluster merge in rank order (identical in every CTA): lane r of warp 0 fetches rank r's
  // partial through DSMEM in one round trip; shuffles combine them in rank order
  if (ctl) {
    double pr[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    pr[0] = pr[2] = kMFloor;
    if (lane < cs) {
#pragma unroll
      for (int j = 0; j < 5; ++j) pr[j] = tl->part[lane][j];  // local: pushed before barrier (A)
    }
    const float rmd = (float)pr[0], rmc = (float)pr[2];
    const float GMd = warp_max(rmd), GMc = warp_max(rmc);
    TR(8);
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
    TR(9);
    if (lane == 0) {
      tl->glob[0] = GMd;
      tl->glob[1] = L_d;
      tl->glob[2] = GMc;
      tl->glob[3] = L_c;
      tl->glob[4] = W;
      const bool ok = L_d > 0.0 && L_c > 0.0 && L_d < 1e300 && L_c < 1e300 && GMd < FLT_MAX && GMc < FLT_MAX;
      tl->lam[0] = ok ? (float)((double)GMd * cd + log2_acc(L_d)) : __int_as_float(0x7fc00000);
      tl->lam[1] = ok ? (float)((double)GMc * cc + log2_acc(L_c)) : __int_as_float(0x7fc00000);
    }
    TR(10);
  }
  __syncthreads();

  TR(5);
  // ---- phase 2: S partial over the chunk still resident in smem (bad rows skip it)
  const float lamd = tl->lam[0], lamc = tl->lam[1];
  float s_loc = 0.f;
  if (lamd == lamd && lamc == lamc) {
    const f2 cdd{cd, cd}, ccc{cc, cc}, ld2{-lamd, -lamd}, lc2{-lamc, -lamc};
    f2 acc2{0.f, 0.f};
#pragma unroll 2
    for (int u = tid; u < units; u += NT)
      p2_unit<T>(reinterpret_cast<const uint4 *>(sd)[u], reinterpret_cast<const uint4 *>(sc)[u], cdd, ccc, ld2, lc2,
                 acc2);
    for (int e = e0 + tid; e < n; e += NT)
      acc2.x += ex2(fminf(fmaf(Elem<T>::load(sd + e), cd, -lamd), fmaf(Elem<T>::load(sc + e), cc, -lamc)));
    s_loc = acc2.x + acc2.y;
  }
  {
    const float v = warp_sum(s_loc);
    if (lane == 0) tl->fscr[wid] = v;
    __syncthreads();
    if (ctl && lane == 0) {
      float r = tl->fscr[0];
      for (int q = 1; q < NW; ++q) r += tl->fscr[q];
      cluster.map_shared_rank(tl->sarr, 0)[rank] = r;
    }
  }
  TR(6);
  cluster_arrive();  // (B) S partials landed in rank 0; no DSMEM access after this point
  cluster_wait();
  TR(7);
  if (rank == 0 && ctl) epilogue<NT>(a, row, tl, cs, pre);
}

}  // namespace

#ifdef SV_TRACE
extern "C" __attribute__((visibility("default"))) int sv_debug_set_trace(void *buf) {
  return (int)cudaMemcpyToSymbol(g_trace, &buf, sizeof(buf));
}
#endif

namespace {

template <typename T, int NT>
cudaError_t launch_score_t(const ScoreArgs &a, cudaStream_t st) {
  const int elem = (int)sizeof(T);
  const size_t smem = 2 * (size_t)a.chunk * elem + sizeof(ScoreTail<NT>);
  const void *fn = (const void *)sv_score_kernel<T, NT>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (a.cs > 8) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((int64_t)a.B * a.k * a.cs));
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = a.cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, sv_score_kernel<T, NT>, a);
}

}  // namespace

cudaError_t launch_score(const ScoreArgs &a, cudaStream_t st) {
  // 16 warps per CTA when a CTA holds a large chunk (2 CTAs / SM), 8 warps for small chunks
  static const int nt = tune_knob("SV_SCORE_THREADS", 0);
  const bool big = nt ? nt == 512 : (int64_t)a.chunk * (a.bf16 ? 2 : 4) * 2 > 48 * 1024;
  if (a.bf16) return big ? launch_score_t<__nv_bfloat16, 512>(a, st) : launch_score_t<__nv_bfloat16, 256>(a, st);
  return big ? launch_score_t<float, 512>(a, st) : launch_score_t<float, 256>(a, st);
}

}  // namespace sv
