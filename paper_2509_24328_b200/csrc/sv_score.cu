// sv_score.cu -- K1: steps a1-a3 of the SV hot path (P L159 S/A, P L164 divergence,
// north_star KL, P L176 profile lookup).
//
// Design (DESIGN.md §5 K1): a PERSISTENT, warp-specialised, cluster-pipelined kernel.
//  * A cluster of cs CTAs owns rows (b, i) = cid, cid + ncl, ...; CTA r of the cluster owns the
//    vocabulary chunk [r*chunk, (r+1)*chunk) of the draft AND the companion row.
//  * 15 compute warps per CTA; the 16th (highest id, favoured by the warp arbiter) is a control
//    warp that runs every latency-bound step: DSMEM pushes, mbarrier waits, merges, epilogue.
//  * Iteration j overlaps three rows of the cluster:
//      pass 1 (row j, compute warps): stream the chunk pair from HBM (16-byte loads, L2
//        evict_last), thread maxima, l = sum 2^{(x - m) log2e / tau}, KL partial
//        w = sum e_d (a_d - a_c) with packed FFMA2 / FADD2; block merge -> 5 partials, which the
//        control warp pushes into every CTA of the cluster (DSMEM + remote mbarrier arrive);
//      pass 2 (row j - 1, compute warps): the control warp has merged row j - 1's partials in
//        rank order (identical bits in every CTA) into Lambda = m c + log2 l while pass 1 ran;
//        re-read the chunk pair -- an L2 hit, it was streamed one iteration ago -- and sum
//        S_r = sum 2^{min(x_d c_d - Lambda_d, x_c c_c - Lambda_c)}; push S_r to the row's
//        epilogue CTA;
//      epilogue (row j - 2, control warp of CTA (j - 2) % cs): S, A, KL, profile lookup, draft
//        normalisers for sd_verify.
//    Slots are double-buffered with full / empty mbarriers, so no cluster-wide barrier is
//    needed in steady state and every exchange latency hides under the other warps' streaming.
//  * HBM traffic is one read of D and C; the second read is served by L2 (~15 TB/s measured).
// The cluster size and chunking depend on (V, dtype) only, so every reduction order -- and
// therefore every output bit -- is independent of B, of the grid size and of the GPU count.
#include <float.h>

#include "sv_device.cuh"
#include "sv_internal.h"

namespace sv {

namespace {

constexpr int NT = kScoreThreads, NW = NT / 32;
constexpr int NCW = NW - 2;   // compute warps
constexpr int NC = NCW * 32;  // compute threads
constexpr int PW = NW - 2;    // producer warp (bulk copies into the ring)
constexpr int XW = NW - 1;    // exchange warp (highest id: merges, pushes, epilogue)
constexpr int kSlots = kScoreSlots;
constexpr int kStageBytes = kScoreStageBytes;
constexpr int NX = NC + 32;   // participants of the compute <-> exchange barriers

// named barriers (id 0 is __syncthreads).  The compute warps may run ahead of the control warp
// by up to two pass-1s and one pass-2 (the LamReady chain bounds them), so the per-row barriers
// rotate over 3 (P1Done) and 2 (LamReady, P2Done) ids and never mix two rows.
enum : int { kBarCompute = 1, kBarP1Done0 = 2, kBarLam0 = 5, kBarP2Done0 = 7 };
__device__ __forceinline__ int bar_p1done(int64_t row) { return kBarP1Done0 + (int)(row % 3); }
__device__ __forceinline__ int bar_lam(int64_t row) { return kBarLam0 + (int)(row & 1); }
__device__ __forceinline__ int bar_p2done(int64_t row) { return kBarP2Done0 + (int)(row & 1); }
__device__ __forceinline__ void bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void bar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

struct Smem {
  uint64_t ring_full[kSlots], ring_empty[kSlots];
  uint64_t full_p[2], empty_p[2], full_s[2], empty_s[2];
  double part[2][kMaxCluster][5];  // (M_d, L_d, M_c, L_c, W) pushed by every rank, per slot
  float sarr[2][kMaxCluster];      // S partials pushed to the epilogue CTA, per slot
  double glob[3][5];               // merged (M_d, L_d, M_c, L_c, W), per row % 3
  float lam[2][2];                 // Lambda_d, Lambda_c, per row parity
  double mine[3][6];               // this CTA's pass-1 partial, per row % 3 ([4] unused)
  float s_mine[2];                 // this CTA's pass-2 partial, per row parity
  float fscr[2 * NCW];
  float fscr2[NCW];
  double dscr[3 * NCW];
};

__device__ __forceinline__ uint32_t remote(const void *p, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void remote_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void st_remote_f64(uint32_t addr, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
}
__device__ __forceinline__ void st_remote_f32(uint32_t addr, float v) {
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
__device__ __forceinline__ void wait_cluster(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "W_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra W_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void wait_cta(uint64_t *bar, uint32_t parity) { mbar_wait(bar, parity); }
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint4 ldg_hint(const void *p, uint64_t pol) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p), "l"(pol));
  return r;
}

// ---------------------------------------------------------------- element arithmetic
struct P1 {
  f2 ld, lc;  // l_d, l_c partials, two lanes each
  f2 w;       // KL partial, two lanes
};

template <bool kGuard>
__device__ __forceinline__ void p1_pair(f2 xd, f2 xc, f2 cdd, f2 ccc, f2 nmdd, f2 nmcc, P1 &acc) {
  const f2 ad = fma2(xd, cdd, nmdd), ac = fma2(xc, ccc, nmcc);
  const f2 ed = ex2x2(ad), ec = ex2x2(ac);
  acc.ld = add2(acc.ld, ed);
  acc.lc = add2(acc.lc, ec);
  if (kGuard) {  // p_d = 0 terms contribute 0 even against a_c = -inf
    acc.w.x += ed.x > 0.f ? ed.x * (ad.x - ac.x) : 0.f;
    acc.w.y += ed.y > 0.f ? ed.y * (ad.y - ac.y) : 0.f;
  } else {
    acc.w = fma2(ed, sub2(ad, ac), acc.w);
  }
}

template <typename T>
__device__ __forceinline__ void unit_pairs(const uint4 &u, f2 (&x)[Elem<T>::kPerUnit / 2]) {
  if constexpr (sizeof(T) == 2) {
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int p = 0; p < 4; ++p) x[p] = f2{bf_lo(w[p]), bf_hi(w[p])};
  } else {
    x[0] = f2{__uint_as_float(u.x), __uint_as_float(u.y)};
    x[1] = f2{__uint_as_float(u.z), __uint_as_float(u.w)};
  }
}

__device__ __forceinline__ float unit_max_bf16(const uint4 &v) {
  const __nv_bfloat162 *p = reinterpret_cast<const __nv_bfloat162 *>(&v);
  const __nv_bfloat162 m = __hmax2(__hmax2(p[0], p[1]), __hmax2(p[2], p[3]));
  return fmaxf(__low2float(m), __high2float(m));
}
template <typename T>
__device__ __forceinline__ float unit_max(const uint4 &v) {
  if constexpr (sizeof(T) == 2) {
    return unit_max_bf16(v);
  } else {
    return fmaxf(fmaxf(__uint_as_float(v.x), __uint_as_float(v.y)), fmaxf(__uint_as_float(v.z), __uint_as_float(v.w)));
  }
}

// ---------------------------------------------------------------- stages
// A row's chunk is consumed in stages of kStageBytes per tensor.  The producer warp moves each
// stage (draft part + companion part) into a ring slot with the bulk-copy engine; the compute
// warps read it from shared memory.  Both sides walk the same (row, pass, stage) sequence.
template <typename T>
struct Stage {
  const T *d, *c;  // global source of this stage
  int n;           // elements in the stage
  int units;       // 16-byte units moved by the bulk-copy engine (0: unaligned rows)
};
template <typename T>
__device__ __forceinline__ int stages_per_row(const ScoreArgs &a, int rank) {
  const int64_t n = max((int64_t)0, min(a.chunk, (int64_t)a.V - (int64_t)rank * a.chunk));
  constexpr int SE = kStageBytes / sizeof(T);
  return (int)((n + SE - 1) / SE);
}
template <typename T>
__device__ __forceinline__ Stage<T> stage_of(const ScoreArgs &a, int64_t row, int rank, int st) {
  constexpr int SE = kStageBytes / sizeof(T), EPU = Elem<T>::kPerUnit;
  const int64_t b = row / a.k, i = row % a.k;
  const int64_t n_rank = max((int64_t)0, min(a.chunk, (int64_t)a.V - (int64_t)rank * a.chunk));
  const int64_t v0 = (int64_t)rank * a.chunk + (int64_t)st * SE;
  Stage<T> s;
  s.d = reinterpret_cast<const T *>(a.d) + b * a.d_sb + i * a.d_si + v0;
  s.c = reinterpret_cast<const T *>(a.c) + b * a.c_sb + i * a.c_si + v0;
  s.n = (int)min((int64_t)SE, n_rank - (int64_t)st * SE);
  const bool al = ((reinterpret_cast<uintptr_t>(s.d) | reinterpret_cast<uintptr_t>(s.c)) & 15) == 0;
  s.units = al ? s.n / EPU : 0;
  return s;
}

// Walk of the (row, pass, stage) sequence shared by the producer and the compute warps:
// iteration j = pass 1 of row j (if j < nrows), then pass 2 of row j - 2 (if valid).
template <typename F>
__device__ __forceinline__ void walk_stages(int64_t nrows, int nst, F &&f) {
  int64_t g = 0;  // global stage counter -> ring slot g % kSlots, use g / kSlots
  for (int64_t j = 0; j <= nrows + 1; ++j) {
    if (j < nrows)
      for (int st = 0; st < nst; ++st, ++g) f(g, j, 1, st);
    if (j >= 2 && j - 2 < nrows)
      for (int st = 0; st < nst; ++st, ++g) f(g, j - 2, 2, st);
  }
}

// pass-1 state of one compute thread across the stages of a row
struct P1State {
  float md, mc, ld, lc, w;
};

__device__ __forceinline__ void p1_rescale(P1State &t, float gmd, float gmc, float cd, float cc) {
  if (gmd > t.md || gmc > t.mc) {  // exact online rescale of the running sums
    const float sdf = ex2((t.md - gmd) * cd), scf = ex2((t.mc - gmc) * cc);
    const float delta = (gmc - t.mc) * cc - (gmd - t.md) * cd;
    if (t.ld > 0.f) t.w = fmaf(t.ld, delta, t.w);
    t.w *= sdf;
    t.ld *= sdf;
    t.lc *= scf;
    t.md = gmd;
    t.mc = gmc;
  }
}

// Pass 1 on one stage (smem copy sd / sc, or global when unaligned).
template <typename T, bool kGuard>
__device__ __forceinline__ void p1_stage(const Stage<T> &sg, const T *sd, const T *sc, float cd, float cc,
                                         P1State &t) {
  constexpr int EPU = Elem<T>::kPerUnit, UPT = kStageBytes / 16 / NC;
  const int tid = threadIdx.x;
  uint4 rd[UPT], rc[UPT];
  float gmd = t.md, gmc = t.mc;
#pragma unroll
  for (int q = 0; q < UPT; ++q) {
    const int u = tid + q * NC;
    if (u < sg.units) {
      rd[q] = reinterpret_cast<const uint4 *>(sd)[u];
      rc[q] = reinterpret_cast<const uint4 *>(sc)[u];
      gmd = fmaxf(gmd, unit_max<T>(rd[q]));
      gmc = fmaxf(gmc, unit_max<T>(rc[q]));
    }
  }
  const int e0 = sg.units * EPU;  // element-wise remainder, read from global
  for (int e = e0 + tid; e < sg.n; e += NC) {
    gmd = fmaxf(gmd, Elem<T>::load(sg.d + e));
    gmc = fmaxf(gmc, Elem<T>::load(sg.c + e));
  }
  p1_rescale(t, gmd, gmc, cd, cc);
  const float nmd = -t.md * cd, nmc = -t.mc * cc;
  const f2 cdd{cd, cd}, ccc{cc, cc}, nmdd{nmd, nmd}, nmcc{nmc, nmc};
  P1 acc{{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};
#pragma unroll
  for (int q = 0; q < UPT; ++q)
    if (tid + q * NC < sg.units) {
      f2 xd[EPU / 2], xc[EPU / 2];
      unit_pairs<T>(rd[q], xd);
      unit_pairs<T>(rc[q], xc);
#pragma unroll
      for (int p = 0; p < EPU / 2; ++p) p1_pair<kGuard>(xd[p], xc[p], cdd, ccc, nmdd, nmcc, acc);
    }
  t.ld += acc.ld.x + acc.ld.y;
  t.lc += acc.lc.x + acc.lc.y;
  t.w += acc.w.x + acc.w.y;
  for (int e = e0 + tid; e < sg.n; e += NC) {
    const float ad = fmaf(Elem<T>::load(sg.d + e), cd, nmd), ac = fmaf(Elem<T>::load(sg.c + e), cc, nmc);
    const float ed = ex2(ad);
    t.ld += ed;
    t.lc += ex2(ac);
    t.w += ed > 0.f ? ed * (ad - ac) : 0.f;
  }
}

// Pass 2 on one stage: the thread's S partial.
template <typename T>
__device__ __forceinline__ float p2_stage(const Stage<T> &sg, const T *sd, const T *sc, float cd, float cc,
                                          float lamd, float lamc) {
  constexpr int EPU = Elem<T>::kPerUnit, UPT = kStageBytes / 16 / NC;
  const int tid = threadIdx.x;
  const f2 cdd{cd, cd}, ccc{cc, cc}, ld2{-lamd, -lamd}, lc2{-lamc, -lamc};
  f2 acc{0.f, 0.f};
#pragma unroll
  for (int q = 0; q < UPT; ++q) {
    const int u = tid + q * NC;
    if (u < sg.units) {
      f2 xd[EPU / 2], xc[EPU / 2];
      unit_pairs<T>(reinterpret_cast<const uint4 *>(sd)[u], xd);
      unit_pairs<T>(reinterpret_cast<const uint4 *>(sc)[u], xc);
#pragma unroll
      for (int p = 0; p < EPU / 2; ++p) {
        const f2 ad = fma2(xd[p], cdd, ld2), ac = fma2(xc[p], ccc, lc2);
        acc = add2(acc, f2{ex2(fminf(ad.x, ac.x)), ex2(fminf(ad.y, ac.y))});
      }
    }
  }
  for (int e = sg.units * EPU + tid; e < sg.n; e += NC)
    acc.x += ex2(fminf(fmaf(Elem<T>::load(sg.d + e), cd, -lamd), fmaf(Elem<T>::load(sg.c + e), cc, -lamc)));
  return acc.x + acc.y;
}

// Epilogue of one row (control warp of its epilogue CTA; independent pieces on separate lanes,
// fp64 range reduction + fp32 transcendentals).  The draft-side outputs depend on the draft row
// alone: a bad companion row does not poison them.
template <typename T>
__device__ __noinline__ void epilogue(const ScoreArgs &a, int64_t row, const double *glob, const float *sarr,
                                      int cs) {
  const int lane = threadIdx.x & 31;
  const float cd = a.cd, cc = a.cc;
  const float GMd = (float)glob[0], GMc = (float)glob[2];
  const double L_d = glob[1], L_c = glob[3], W = glob[4];
  auto row_bits = [](double L, float M) {
    if (!(L == L) || !(L < 1e300) || !(M < FLT_MAX)) return 1; /*SV_ROW_NAN*/
    return (L > 0.0) ? 0 : 2;                                  /*SV_ROW_ALL_NEG_INF*/
  };
  const int d_st = row_bits(L_d, GMd), c_st = row_bits(L_c, GMc);
  const int64_t b = row / a.k, i = row % a.k;
  const int32_t t = a.tok[row];
  const bool tok_ok = t >= 0 && t < a.V;
  int st = d_st | c_st | (tok_ok ? 0 : 4 /*SV_ROW_BAD_TOKEN*/);
  // profile edges j = lane + 1, lane + 33 (+inf past the end) -- loads issued early
  const float inf = __int_as_float(0x7f800000);
  float se[2], ae[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int j = lane + 1 + 32 * h;
    se[h] = (a.p_hat && j < a.n_s) ? a.s_edges[j] : inf;
    ae[h] = (a.p_hat && j < a.n_a) ? a.a_edges[j] : inf;
  }
  // lane 0: log2 p_d(t); lane 1: log2 p_c(t); lane 2: log2 L_d - log2 L_c; lane 3: S (rank order)
  double piece = 0.0;
  if (lane == 0 && !d_st && tok_ok) {
    const float x = Elem<T>::load(reinterpret_cast<const T *>(a.d) + b * a.d_sb + i * a.d_si + t);
    piece = (double)x * cd - (double)(GMd * cd) - log2_acc(L_d);
  }
  if (lane == 1 && !st) {
    const float x = Elem<T>::load(reinterpret_cast<const T *>(a.c) + b * a.c_sb + i * a.c_si + t);
    piece = (double)x * cc - (double)(GMc * cc) - log2_acc(L_c);
  }
  if (lane == 2 && !st) piece = log2_acc(L_d) - log2_acc(L_c);
  if (lane == 3)
    for (int r = 0; r < cs; ++r) piece += (double)sarr[r];
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
    int si = (se[0] < Sf) + (se[1] < Sf), ai = (ae[0] < Af) + (ae[1] < Af);
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

__device__ __forceinline__ void bulk_g2s_hint(void *dst, const void *src, uint32_t bytes, uint64_t *bar,
                                              uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

template <typename T>
__global__ void __launch_bounds__(kScoreThreads, 2) sv_score_kernel(const ScoreArgs a) {
  constexpr int SE = kStageBytes / sizeof(T);
  __shared__ Smem sm;
  extern __shared__ __align__(128) uint8_t ring_raw[];
  T *const ring = reinterpret_cast<T *>(ring_raw);  // kSlots x [draft stage | companion stage]
  cg::cluster_group cluster = cg::this_cluster();
  const int cs = a.cs;
  const int rank = (int)cluster.block_rank();
  const int64_t cid = blockIdx.x / cs, ncl = gridDim.x / cs;
  const int64_t rows = (int64_t)a.B * a.k;
  const int64_t nrows = rows > cid ? (rows - cid + ncl - 1) / ncl : 0;  // rows of this cluster
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const float cd = a.cd, cc = a.cc;
  const int nst = stages_per_row<T>(a, rank);
  auto row_of = [&](int64_t j) { return cid + j * ncl; };

  if (tid == 0) {
    for (int k = 0; k < kSlots; ++k) {
      mbar_init(&sm.ring_full[k], 1);
      mbar_init(&sm.ring_empty[k], NCW);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&sm.full_p[s], cs);
      mbar_init(&sm.empty_p[s], cs);
      mbar_init(&sm.full_s[s], cs);
      mbar_init(&sm.empty_s[s], 1);
    }
    fence_mbar_init();
  }
  cluster_sync_all();  // every barrier of the cluster is initialised before any remote arrive

  if (wid < NCW) {
    // ================================================================ compute warps
    P1State t{kMFloor, kMFloor, 0.f, 0.f, 0.f};
    float lamd = 0.f, lamc = 0.f, s_acc = 0.f;
    walk_stages(nrows, nst, [&](int64_t g, int64_t row, int pass, int st) {
      const int slot = (int)(g % kSlots);
      const Stage<T> sg = stage_of<T>(a, row_of(row), rank, st);  // row = local index
      const T *sd = ring + (size_t)slot * 2 * SE, *sc = sd + SE;
      if (pass == 1) {
        if (st == 0) t = P1State{kMFloor, kMFloor, 0.f, 0.f, 0.f};
        mbar_wait(&sm.ring_full[slot], (uint32_t)((g / kSlots) & 1));
        const P1State t0 = t;
        p1_stage<T, false>(sg, sd, sc, cd, cc, t);
        if (t.w != t.w && t.ld == t.ld && t.lc == t.lc) {  // 0 * (-inf) from masked logits: redo guarded
          t = t0;
          p1_stage<T, true>(sg, sd, sc, cd, cc, t);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.ring_empty[slot]);
        if (st == nst - 1) {  // ---- block merge of the row's pass 1 (fixed warp / lane order)
          float Md = warp_max(t.md), Mc = warp_max(t.mc);
          if (lane == 0) {
            sm.fscr[wid] = Md;
            sm.fscr[NCW + wid] = Mc;
          }
          bar_sync(kBarCompute, NC);
          Md = sm.fscr[0];
          Mc = sm.fscr[NCW];
#pragma unroll
          for (int q = 1; q < NCW; ++q) {
            Md = fmaxf(Md, sm.fscr[q]);
            Mc = fmaxf(Mc, sm.fscr[NCW + q]);
          }
          const float sdf = ex2((t.md - Md) * cd), scf = ex2((t.mc - Mc) * cc);
          const float delta = (Mc - t.mc) * cc - (Md - t.md) * cd;
          double ww = t.w;
          if (t.ld > 0.f) ww += (double)t.ld * (double)delta;
          double v[3] = {(double)t.ld * sdf, (double)t.lc * scf, ww * sdf};
#pragma unroll
          for (int k = 0; k < 3; ++k) v[k] = warp_sum_d(v[k]);
          if (lane == 0)
#pragma unroll
            for (int k = 0; k < 3; ++k) sm.dscr[k * NCW + wid] = v[k];
          bar_sync(kBarCompute, NC);
          double *mine = sm.mine[row % 3];
          if (tid < 3) {
            double r = 0.0;
            for (int q = 0; q < NCW; ++q) r += sm.dscr[tid * NCW + q];
            mine[1 + 2 * tid] = r;  // tid 0 -> L_d [1], 1 -> L_c [3], 2 -> W [5]
          }
          if (tid == 0) {
            mine[0] = Md;
            mine[2] = Mc;
          }
          bar_arrive(bar_p1done(row), NX);  // the exchange warp may push the partial
        }
      } else {
        if (st == 0) {
          bar_sync(bar_lam(row), NX);  // the exchange warp merged this row
          lamd = sm.lam[row & 1][0];
          lamc = sm.lam[row & 1][1];
          s_acc = 0.f;
        }
        mbar_wait(&sm.ring_full[slot], (uint32_t)((g / kSlots) & 1));
        if (lamd == lamd && lamc == lamc) s_acc += p2_stage<T>(sg, sd, sc, cd, cc, lamd, lamc);  // bad rows skip
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.ring_empty[slot]);
        if (st == nst - 1) {
          const float sl = warp_sum(s_acc);
          if (lane == 0) sm.fscr2[wid] = sl;
          bar_sync(kBarCompute, NC);
          if (tid == 0) {
            float r = sm.fscr2[0];
            for (int q = 1; q < NCW; ++q) r += sm.fscr2[q];
            sm.s_mine[row & 1] = r;
          }
          bar_arrive(bar_p2done(row), NX);
        }
      }
    });
  } else if (wid == PW) {
    // ================================================================ producer warp
    if (lane == 0) {
      const uint64_t pol_keep = l2_policy_evict_last(), pol_last = l2_policy_evict_first();
      walk_stages(nrows, nst, [&](int64_t g, int64_t row, int pass, int st) {
        const int slot = (int)(g % kSlots);
        if (g >= kSlots) wait_cta(&sm.ring_empty[slot], (uint32_t)(((g / kSlots) - 1) & 1));
        const Stage<T> sg = stage_of<T>(a, row_of(row), rank, st);  // row = local index
        T *sd = ring + (size_t)slot * 2 * SE, *sc = sd + SE;
        if (sg.units > 0) {
          const uint32_t bytes = (uint32_t)sg.units * 16u;
          const uint64_t pol = pass == 1 ? pol_keep : pol_last;  // pass 2 is the last use
          fence_proxy_async();
          mbar_arrive_expect_tx(&sm.ring_full[slot], 2u * bytes);
          bulk_g2s_hint(sd, sg.d, bytes, &sm.ring_full[slot], pol);
          bulk_g2s_hint(sc, sg.c, bytes, &sm.ring_full[slot], pol);
        } else {
          mbar_arrive(&sm.ring_full[slot]);  // unaligned / empty stage: read from global
        }
      });
    }
    __syncwarp();
  } else {
    // ================================================================ exchange warp
    for (int64_t j = 0; j <= nrows + 2; ++j) {
      // (1) merge row j - 1's partials (pushed during the peers' iteration j - 1) while the
      //     compute warps stream; their pass 2 of that row starts one iteration later
      if (j >= 1 && j - 1 < nrows) {
        const int64_t r1 = j - 1;
        const int s = (int)(r1 & 1);
        wait_cluster(&sm.full_p[s], (uint32_t)((r1 >> 1) & 1));
        double pr[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
        pr[0] = pr[2] = kMFloor;
        if (lane < cs)
#pragma unroll
          for (int k = 0; k < 5; ++k) pr[k] = sm.part[s][lane][k];
        __syncwarp();
        if (lane < cs) remote_arrive(remote(&sm.empty_p[s], lane));  // slot s of every peer is free
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
          double *gl = sm.glob[r1 % 3];
          gl[0] = GMd;
          gl[1] = L_d;
          gl[2] = GMc;
          gl[3] = L_c;
          gl[4] = W;
          const bool ok = L_d > 0.0 && L_c > 0.0 && L_d < 1e300 && L_c < 1e300 && GMd < FLT_MAX && GMc < FLT_MAX;
          sm.lam[s][0] = ok ? (float)((double)GMd * cd + log2_acc(L_d)) : __int_as_float(0x7fc00000);
          sm.lam[s][1] = ok ? (float)((double)GMc * cc + log2_acc(L_c)) : __int_as_float(0x7fc00000);
        }
        __syncwarp();
        bar_arrive(bar_lam(r1), NX);
      }
      // (2) push this CTA's pass-1 partial of row j into slot j % 2 of every peer
      if (j < nrows) {
        const int s = (int)(j & 1);
        bar_sync(bar_p1done(j), NX);
        if (j >= 2) wait_cluster(&sm.empty_p[s], (uint32_t)(((j >> 1) - 1) & 1));
        if (lane < cs) {
          const double *mine = sm.mine[j % 3];
          const double v[5] = {mine[0], mine[1], mine[2], mine[3], mine[5]};
#pragma unroll
          for (int k = 0; k < 5; ++k) st_remote_f64(remote(&sm.part[s][rank][k], lane), v[k]);
          remote_arrive(remote(&sm.full_p[s], lane));
        }
      }
      // (3) push this CTA's S partial of row j - 2 to the row's epilogue CTA
      if (j >= 2 && j - 2 < nrows) {
        const int64_t r2 = j - 2;
        const int s = (int)(r2 & 1);
        const int epi = (int)(r2 % cs);
        bar_sync(bar_p2done(r2), NX);
        if (r2 >= 2) wait_cluster(&sm.empty_s[s], (uint32_t)(((r2 >> 1) - 1) & 1));
        if (lane == 0) {
          st_remote_f32(remote(&sm.sarr[s][rank], epi), sm.s_mine[s]);
          remote_arrive(remote(&sm.full_s[s], epi));
        }
        __syncwarp();
      }
      // (4) epilogue of row j - 3 (its S partials were pushed during iteration j - 1)
      if (j >= 3 && j - 3 < nrows && (int)((j - 3) % cs) == rank) {
        const int64_t r3 = j - 3;
        const int s = (int)(r3 & 1);
        // this CTA's full_s[s] completes once per row r with r % 2 == s and r % cs == rank: the
        // completion index of row r is r / lcm(2, cs)
        const int64_t lcm2 = cs == 1 ? 2 : cs;
        wait_cluster(&sm.full_s[s], (uint32_t)((r3 / lcm2) & 1));
        epilogue<T>(a, row_of(r3), sm.glob[r3 % 3], sm.sarr[s], cs);
        __syncwarp();
        if (lane < cs) remote_arrive(remote(&sm.empty_s[s], lane));  // slot s free for row r3 + 2
      }
    }
  }
  cluster_sync_all();  // no CTA exits while a peer may still write its shared memory
}

}  // namespace

cudaError_t launch_score(const ScoreArgs &a, cudaStream_t st) {
  const void *fn = a.bf16 ? (const void *)sv_score_kernel<__nv_bfloat16> : (const void *)sv_score_kernel<float>;
  const size_t smem = (size_t)kSlots * 2 * kStageBytes;
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
  // persistent: as many clusters as can be co-resident, never more than rows (clusters are
  // independent, so residency is a performance choice, not a correctness requirement)
  const int64_t rows = (int64_t)a.B * a.k;
  int64_t ncl = max_active_clusters(fn, cfg, (int)smem, a.cs);
  static const int mult = tune_knob("SV_SCORE_CLUSTER_MULT", 1);
  ncl *= mult;
  if (ncl > rows) ncl = rows;
  if (ncl < 1) ncl = 1;
  cfg.gridDim = dim3((unsigned)(ncl * a.cs));
  if (a.bf16) return cudaLaunchKernelEx(&cfg, sv_score_kernel<__nv_bfloat16>, a);
  return cudaLaunchKernelEx(&cfg, sv_score_kernel<float>, a);
}

}  // namespace sv
