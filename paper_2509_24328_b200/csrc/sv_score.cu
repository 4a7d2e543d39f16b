// sv_score.cu -- K1: steps a1-a3 of the SV hot path (P L159 S/A, P L164 divergence,
// north_star KL, P L176 profile lookup).
//
// Design (DESIGN.md §5 K1).  A row pair (draft row + companion row of one (b, i)) is cut
// into nch vocabulary chunks of NT x U x 16 bytes per tensor (16384 bf16 / 8192 fp32
// logits); a work item is one (row, chunk).  A persistent grid of co-resident CTAs walks the
// items; in iteration j a CTA runs
//   phase 1 on item j*G + cta: stream the chunk pair from HBM with 16 independent 16-byte
//     loads per thread, thread maxima (packed bf16x2 max), l = sum 2^{(x - m) log2e / tau}
//     and the KL partial w = sum e_d (a_d - a_c) (log2 units), block merge in fixed order,
//     publish the 5 partials + a release increment of the row's arrival counter;
//   phase 2 on item (j - 2)*G + cta: acquire the row's nch partials, merge them in chunk
//     order (identical bits in every CTA), re-read the chunk pair -- from L2: it was streamed
//     two iterations ago, far inside the 126 MB L2's reuse window -- and accumulate
//     S_q = sum 2^{min(x_d c_d - Lambda_d, x_c c_c - Lambda_c)} (one MUFU per pair); the CTA
//     that completes a row's phase 2 runs the epilogue: S, A, KL in fp64, profile lookup,
//     draft normalisers for sd_verify, and resets the row's counters.
// Every logit is read from HBM once; there are no thread-block clusters, so all 148 SMs are
// used whatever the GPC layout.  Waits only ever point at phase-1 work of earlier or equal
// iterations, which never waits, so the co-resident grid cannot deadlock.  All reduction
// orders depend on (V, dtype) only: results are bitwise identical for any B, grid size or
// GPU count.
#include <float.h>

#include "sv_device.cuh"
#include "sv_internal.h"

namespace sv {

namespace {

constexpr int NT = kScoreThreads, NW = NT / 32, U = kScoreUnits;

struct ScoreWs {
  int32_t *cnt1, *cnt2;  // [rows] phase-1 / phase-2 arrivals (self-resetting)
  ItemPart *part;        // [rows * nch]
  float *spart;          // [rows * nch]
};

__device__ __forceinline__ ScoreWs carve(const ScoreArgs &a) {
  ScoreWs w;
  const int64_t rows = (int64_t)a.B * a.k;
  uint8_t *p = reinterpret_cast<uint8_t *>(a.ws);
  w.cnt1 = reinterpret_cast<int32_t *>(p);
  w.cnt2 = w.cnt1 + rows;
  w.part = reinterpret_cast<ItemPart *>(p + score_ws_part_offset(rows));
  w.spart = reinterpret_cast<float *>(p + score_ws_spart_offset(rows, a.nch));
  return w;
}

__device__ __forceinline__ int ld_acquire(const int32_t *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <typename T>
struct Chunk {
  const T *d, *c;  // chunk start in the draft / companion row
  int n;           // elements
  bool vec;        // both 16-byte aligned: unit loads
};

template <typename T>
__device__ __forceinline__ Chunk<T> chunk_of(const ScoreArgs &a, int64_t item) {
  const int64_t row = item / a.nch, q = item % a.nch;
  const int64_t b = row / a.k, i = row % a.k, v0 = q * a.chunk;
  Chunk<T> ch;
  ch.d = reinterpret_cast<const T *>(a.d) + b * a.d_sb + i * a.d_si + v0;
  ch.c = reinterpret_cast<const T *>(a.c) + b * a.c_sb + i * a.c_si + v0;
  ch.n = (int)min(a.chunk, (int64_t)a.V - v0);
  ch.vec = ((reinterpret_cast<uintptr_t>(ch.d) | reinterpret_cast<uintptr_t>(ch.c)) & 15) == 0;
  return ch;
}

// Load the thread's units of the chunk pair (all loads issued before any use).
template <typename T>
__device__ __forceinline__ int load_units(const Chunk<T> &ch, uint4 (&rd)[U], uint4 (&rc)[U]) {
  constexpr int EPU = Elem<T>::kPerUnit;
  const int units = ch.n / EPU;
#pragma unroll
  for (int q = 0; q < U; ++q) {
    const int u = threadIdx.x + q * NT;
    if (u < units) {
      rd[q] = ldg_stream(ch.d + (size_t)u * EPU);
      rc[q] = ldg_stream(ch.c + (size_t)u * EPU);
    }
  }
  return units;
}

// Packed max of a 16-byte unit of bf16 into a running bf16x2 max.
__device__ __forceinline__ void umax(__nv_bfloat162 &m, const uint4 &v) {
  const __nv_bfloat162 *p = reinterpret_cast<const __nv_bfloat162 *>(&v);
  m = __hmax2(__hmax2(m, p[0]), __hmax2(p[1], __hmax2(p[2], p[3])));
}

// Phase-1 sums on registers against the thread maxima.  kGuard = false is the fast path;
// a NaN KL partial (only possible from 0 * (-inf) when the row holds -inf logits) is
// recomputed with kGuard = true.
template <typename T, bool kGuard>
__device__ __forceinline__ void sums_units(const uint4 (&rd)[U], const uint4 (&rc)[U], int units, float cd, float cc,
                                           float nmd, float nmc, float &ld, float &lc, float &w) {
  constexpr int EPU = Elem<T>::kPerUnit;
  float ld0 = 0.f, ld1 = 0.f, lc0 = 0.f, lc1 = 0.f, w0 = 0.f, w1 = 0.f;
#pragma unroll
  for (int q = 0; q < U; ++q) {
    if (threadIdx.x + q * NT < units) {
      float xd[EPU], xc[EPU];
      Elem<T>::unit(rd[q], xd);
      Elem<T>::unit(rc[q], xc);
#pragma unroll
      for (int j = 0; j < EPU; j += 2) {
        const float ad0 = fmaf(xd[j], cd, nmd), ac0 = fmaf(xc[j], cc, nmc);
        const float ad1 = fmaf(xd[j + 1], cd, nmd), ac1 = fmaf(xc[j + 1], cc, nmc);
        const float ed0 = ex2(ad0), ec0 = ex2(ac0), ed1 = ex2(ad1), ec1 = ex2(ac1);
        ld0 += ed0;
        lc0 += ec0;
        ld1 += ed1;
        lc1 += ec1;
        if (kGuard) {  // p_d = 0 terms contribute 0 even against a_c = -inf
          w0 += ed0 > 0.f ? ed0 * (ad0 - ac0) : 0.f;
          w1 += ed1 > 0.f ? ed1 * (ad1 - ac1) : 0.f;
        } else {
          w0 = fmaf(ed0, ad0 - ac0, w0);
          w1 = fmaf(ed1, ad1 - ac1, w1);
        }
      }
    }
  }
  ld += ld0 + ld1;
  lc += lc0 + lc1;
  w += w0 + w1;
}

template <bool kGuard>
__device__ __forceinline__ void sums_one(float xd, float xc, float cd, float cc, float nmd, float nmc, float &ld,
                                         float &lc, float &w) {
  const float ad = fmaf(xd, cd, nmd), ac = fmaf(xc, cc, nmc);
  const float ed = ex2(ad);
  ld += ed;
  lc += ex2(ac);
  if (kGuard)
    w += ed > 0.f ? ed * (ad - ac) : 0.f;
  else
    w = fmaf(ed, ad - ac, w);
}

struct BlockScratch {
  float fscr[2 * NW];
  double dscr[3 * NW];
  double glob[5];
  float lam[2];
  int last;
};

template <typename T>
__device__ void phase1(const ScoreArgs &a, const ScoreWs &ws, int64_t item, BlockScratch &sh) {
  constexpr int EPU = Elem<T>::kPerUnit;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const float cd = a.cd, cc = a.cc;
  const Chunk<T> ch = chunk_of<T>(a, item);
  float md = kMFloor, mc = kMFloor, lf_d = 0.f, lf_c = 0.f, wf = 0.f;
  if (ch.vec) {
    uint4 rd[U], rc[U];
    const int units = load_units<T>(ch, rd, rc);
    const int e = units * EPU + tid;  // ragged tail: < EPU elements, one per thread
    const float xdt = e < ch.n ? Elem<T>::load(ch.d + e) : kMFloor;
    const float xct = e < ch.n ? Elem<T>::load(ch.c + e) : kMFloor;
    if constexpr (sizeof(T) == 2) {
      __nv_bfloat162 pd = __halves2bfloat162(__ushort_as_bfloat16(0xFF80), __ushort_as_bfloat16(0xFF80));
      __nv_bfloat162 pc = pd;
#pragma unroll
      for (int q = 0; q < U; ++q)
        if (tid + q * NT < units) {
          umax(pd, rd[q]);
          umax(pc, rc[q]);
        }
      md = fmaxf(md, fmaxf(__low2float(pd), __high2float(pd)));
      mc = fmaxf(mc, fmaxf(__low2float(pc), __high2float(pc)));
    } else {
#pragma unroll
      for (int q = 0; q < U; ++q)
        if (tid + q * NT < units) {
          float xd[4], xc[4];
          Elem<T>::unit(rd[q], xd);
          Elem<T>::unit(rc[q], xc);
          md = fmaxf(md, fmaxf(fmaxf(xd[0], xd[1]), fmaxf(xd[2], xd[3])));
          mc = fmaxf(mc, fmaxf(fmaxf(xc[0], xc[1]), fmaxf(xc[2], xc[3])));
        }
    }
    md = fmaxf(md, xdt);
    mc = fmaxf(mc, xct);
    const float nmd = -md * cd, nmc = -mc * cc;
    sums_units<T, false>(rd, rc, units, cd, cc, nmd, nmc, lf_d, lf_c, wf);
    if (e < ch.n) sums_one<false>(xdt, xct, cd, cc, nmd, nmc, lf_d, lf_c, wf);
    if (wf != wf && lf_d == lf_d && lf_c == lf_c) {  // 0 * (-inf) from masked logits: guarded redo
      lf_d = lf_c = wf = 0.f;                          // (reloads the chunk: L2 hits, rare path)
      load_units<T>(ch, rd, rc);
      sums_units<T, true>(rd, rc, units, cd, cc, nmd, nmc, lf_d, lf_c, wf);
      if (e < ch.n) sums_one<true>(xdt, xct, cd, cc, nmd, nmc, lf_d, lf_c, wf);
    }
  } else {  // unaligned rows (edge cases): element-wise, two passes over global memory
    for (int e = tid; e < ch.n; e += NT) {
      md = fmaxf(md, Elem<T>::load(ch.d + e));
      mc = fmaxf(mc, Elem<T>::load(ch.c + e));
    }
    const float nmd = -md * cd, nmc = -mc * cc;
    for (int e = tid; e < ch.n; e += NT)
      sums_one<true>(Elem<T>::load(ch.d + e), Elem<T>::load(ch.c + e), cd, cc, nmd, nmc, lf_d, lf_c, wf);
  }
  // ---- block merge (fixed warp / lane order)
  float Md = warp_max(md), Mc = warp_max(mc);
  if (lane == 0) {
    sh.fscr[wid] = Md;
    sh.fscr[NW + wid] = Mc;
  }
  __syncthreads();
  Md = sh.fscr[0];
  Mc = sh.fscr[NW];
#pragma unroll
  for (int q = 1; q < NW; ++q) {
    Md = fmaxf(Md, sh.fscr[q]);
    Mc = fmaxf(Mc, sh.fscr[NW + q]);
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
    for (int j = 0; j < 3; ++j) sh.dscr[j * NW + wid] = v[j];
  __syncthreads();
  if (tid == 0) {
    ItemPart p;
    p.md = Md;
    p.mc = Mc;
    p.ld = sh.dscr[0];
    p.lc = sh.dscr[NW];
    p.w = sh.dscr[2 * NW];
    for (int q = 1; q < NW; ++q) {
      p.ld += sh.dscr[q];
      p.lc += sh.dscr[NW + q];
      p.w += sh.dscr[2 * NW + q];
    }
    ws.part[item] = p;
    __threadfence();
    atomicAdd(ws.cnt1 + item / a.nch, 1);
  }
}

// Merge a row's nch phase-1 partials in chunk order (warp 0; every CTA gets the same bits).
__device__ __noinline__ void merge_row(const ScoreArgs &a, const ScoreWs &ws, int64_t row, BlockScratch &sh) {
  const int lane = threadIdx.x & 31;
  const float cd = a.cd, cc = a.cc;
  const ItemPart *pp = ws.part + row * a.nch;
  float GMd = kMFloor, GMc = kMFloor;
  for (int q = lane; q < a.nch; q += 32) {
    GMd = fmaxf(GMd, (float)__ldcg(&pp[q].md));
    GMc = fmaxf(GMc, (float)__ldcg(&pp[q].mc));
  }
  GMd = warp_max(GMd);
  GMc = warp_max(GMc);
  double L_d = 0.0, L_c = 0.0, W = 0.0;
  for (int q0 = 0; q0 < a.nch; q0 += 32) {
    double cl_d = 0.0, cl_c = 0.0, cw = 0.0;
    const int q = q0 + lane;
    if (q < a.nch) {
      const float rmd = (float)__ldcg(&pp[q].md), rmc = (float)__ldcg(&pp[q].mc);
      const double rld = __ldcg(&pp[q].ld), rlc = __ldcg(&pp[q].lc), rw = __ldcg(&pp[q].w);
      const float sdf = ex2((rmd - GMd) * cd), scf = ex2((rmc - GMc) * cc);
      const float delta = (GMc - rmc) * cc - (GMd - rmd) * cd;
      double ww = rw;
      if (rld > 0.0) ww += rld * (double)delta;
      cl_d = rld * sdf;
      cl_c = rlc * scf;
      cw = ww * sdf;
    }
    const int m = min(32, a.nch - q0);
    for (int r = 0; r < m; ++r) {  // chunk order
      L_d += __shfl_sync(0xffffffffu, cl_d, r);
      L_c += __shfl_sync(0xffffffffu, cl_c, r);
      W += __shfl_sync(0xffffffffu, cw, r);
    }
  }
  if (lane == 0) {
    sh.glob[0] = GMd;
    sh.glob[1] = L_d;
    sh.glob[2] = GMc;
    sh.glob[3] = L_c;
    sh.glob[4] = W;
    const bool ok = L_d > 0.0 && L_c > 0.0 && L_d < 1e300 && L_c < 1e300 && GMd < FLT_MAX && GMc < FLT_MAX;
    sh.lam[0] = ok ? (float)((double)GMd * cd + log2(L_d)) : __int_as_float(0x7fc00000);
    sh.lam[1] = ok ? (float)((double)GMc * cc + log2(L_c)) : __int_as_float(0x7fc00000);
  }
}

// Epilogue of one row (warp 0 of the CTA that completed the row's phase 2; fp64, independent
// pieces on separate lanes).  The draft-side outputs depend on the draft row alone.
template <typename T>
__device__ __noinline__ void epilogue(const ScoreArgs &a, const ScoreWs &ws, int64_t row, const BlockScratch &sh) {
  const int lane = threadIdx.x & 31;
  const float cd = a.cd, cc = a.cc;
  const float GMd = (float)sh.glob[0], GMc = (float)sh.glob[2];
  const double L_d = sh.glob[1], L_c = sh.glob[3];
  auto row_bits = [](double L, float M) {
    if (!(L == L) || !(L < 1e300) || !(M < FLT_MAX)) return 1; /*SV_ROW_NAN*/
    return (L > 0.0) ? 0 : 2;                                  /*SV_ROW_ALL_NEG_INF*/
  };
  const int d_st = row_bits(L_d, GMd), c_st = row_bits(L_c, GMc);
  const int32_t t = a.tok[row];
  const bool tok_ok = t >= 0 && t < a.V;
  int st = d_st | c_st | (tok_ok ? 0 : 4 /*SV_ROW_BAD_TOKEN*/);
  const int64_t b = row / a.k, i = row % a.k;
  // lane 0: log2 p_d(t); lane 1: log2 p_c(t); lane 2: ln(L_d / L_c); lane 3: S (chunk order)
  double piece = 0.0;
  if (lane == 0 && !d_st && tok_ok) {
    const float x = Elem<T>::load(reinterpret_cast<const T *>(a.d) + b * a.d_sb + i * a.d_si + t);
    piece = (double)x * cd - (double)(GMd * cd) - log2(L_d);
  }
  if (lane == 1 && !st) {
    const float x = Elem<T>::load(reinterpret_cast<const T *>(a.c) + b * a.c_sb + i * a.c_si + t);
    piece = (double)x * cc - (double)(GMc * cc) - log2(L_c);
  }
  if (lane == 2 && !st) piece = log(L_d / L_c);
  if (lane == 3)
    for (int q = 0; q < a.nch; ++q) piece += (double)__ldcg(ws.spart + row * a.nch + q);
  const double argd = __shfl_sync(0xffffffffu, piece, 0);
  double piece2 = 0.0;  // lane 0: p_d(t); lane 1: p_c(t) / p_d(t)
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
    KL = 0.6931471805599453 * (sh.glob[4] / L_d) - lnr;
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
    ws.cnt1[row] = 0;  // leave the counters zeroed for the next call
    ws.cnt2[row] = 0;
  }
}

template <typename T>
__device__ void phase2(const ScoreArgs &a, const ScoreWs &ws, int64_t item, BlockScratch &sh) {
  constexpr int EPU = Elem<T>::kPerUnit;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t row = item / a.nch;
  if (wid == 0) {
    if (lane == 0)
      while (ld_acquire(ws.cnt1 + row) < a.nch) __nanosleep(64);
    __syncwarp();
    merge_row(a, ws, row, sh);
  }
  __syncthreads();
  const float lamd = sh.lam[0], lamc = sh.lam[1];
  const float cd = a.cd, cc = a.cc;
  float s = 0.f;
  if (lamd == lamd && lamc == lamc) {  // bad rows skip the S sweep
    const Chunk<T> ch = chunk_of<T>(a, item);
    float acc0 = 0.f, acc1 = 0.f;
    if (ch.vec) {
      uint4 rd[U], rc[U];
      const int units = load_units<T>(ch, rd, rc);  // L2 hits: streamed two iterations ago
#pragma unroll
      for (int q = 0; q < U; ++q) {
        if (tid + q * NT < units) {
          float xd[EPU], xc[EPU];
          Elem<T>::unit(rd[q], xd);
          Elem<T>::unit(rc[q], xc);
#pragma unroll
          for (int j = 0; j < EPU; j += 2) {
            acc0 += ex2(fminf(fmaf(xd[j], cd, -lamd), fmaf(xc[j], cc, -lamc)));
            acc1 += ex2(fminf(fmaf(xd[j + 1], cd, -lamd), fmaf(xc[j + 1], cc, -lamc)));
          }
        }
      }
      const int e = units * EPU + tid;
      if (e < ch.n)
        acc0 += ex2(fminf(fmaf(Elem<T>::load(ch.d + e), cd, -lamd), fmaf(Elem<T>::load(ch.c + e), cc, -lamc)));
    } else {
      for (int e = tid; e < ch.n; e += NT)
        acc0 += ex2(fminf(fmaf(Elem<T>::load(ch.d + e), cd, -lamd), fmaf(Elem<T>::load(ch.c + e), cc, -lamc)));
    }
    s = acc0 + acc1;
  }
  s = warp_sum(s);
  if (lane == 0) sh.fscr[wid] = s;
  __syncthreads();
  if (tid == 0) {
    float r = sh.fscr[0];
    for (int q = 1; q < NW; ++q) r += sh.fscr[q];
    ws.spart[item] = r;
    __threadfence();
    const int old = atomicAdd(ws.cnt2 + row, 1);
    sh.last = (old == a.nch - 1);
    if (sh.last) __threadfence();  // acquire side: every chunk's S partial is visible
  }
  __syncthreads();
  if (sh.last && wid == 0) epilogue<T>(a, ws, row, sh);
  // the next phase's first __syncthreads orders the epilogue's smem reads before any reuse
}

template <typename T>
__global__ void __launch_bounds__(kScoreThreads, 2) sv_score_kernel(const ScoreArgs a) {
  __shared__ BlockScratch sh;
  const ScoreWs ws = carve(a);
  const int64_t G = gridDim.x, items = (int64_t)a.B * a.k * a.nch;
  for (int64_t j = 0;; ++j) {
    const int64_t i1 = j * G + blockIdx.x, i2 = (j - kScoreLag) * G + blockIdx.x;
    if (i2 >= items) break;
    if (i1 < items) phase1<T>(a, ws, i1, sh);
    if (i2 >= 0) phase2<T>(a, ws, i2, sh);
  }
}

}  // namespace

cudaError_t launch_score(const ScoreArgs &a, cudaStream_t st) {
  const void *fn = a.bf16 ? (const void *)sv_score_kernel<__nv_bfloat16> : (const void *)sv_score_kernel<float>;
  const int64_t items = (int64_t)a.B * a.k * a.nch;
  int64_t grid = resident_grid(fn, kScoreThreads, 0);  // co-resident: phase 2 waits on other CTAs
  if (grid > items) grid = items;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kScoreThreads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // guarantees co-residency (or fails loudly)
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (a.bf16) return cudaLaunchKernelEx(&cfg, sv_score_kernel<__nv_bfloat16>, a);
  return cudaLaunchKernelEx(&cfg, sv_score_kernel<float>, a);
}

}  // namespace sv
