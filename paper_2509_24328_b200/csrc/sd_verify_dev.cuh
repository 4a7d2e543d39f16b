// sd_verify_dev.cuh -- the device code of K4..K5b (steps a5-a6): target-row partials, the row
// merges and accept tests, residual slice masses, the token search, as per-warp / per-sequence
// device functions (included by sd_verify.cu, the verify kernels).
#pragma once
#include <float.h>

#include "sv_device.cuh"
#include "sv_internal.h"

namespace sv {

namespace {

#define kNaNf __int_as_float(0x7fc00000)
#define SV_MAX_K_DEV 16
constexpr int kFindChunks = 8;  // K5b: slice-mass chunks of 32 loaded together

// Target row i of sequence b: dense [B, k+1, V] (strides) or ragged / compacted (NEXT-3, P L266:
// rows of sequence b at t_rowptr[b] + i, i <= gamma_b, row stride t_si)
template <typename T>
__device__ __forceinline__ const T *trow(const VerifyArgs &a, int64_t b, int64_t i) {
  const T *base = reinterpret_cast<const T *>(a.t);
  return a.t_rowptr ? base + (a.t_rowptr[b] + i) * a.t_si : base + b * a.t_sb + i * a.t_si;
}

// ------------------------------------------------------------------ K4
// The lane's part of one (row, split) item from its units r[j] = unit lane + 32 j (< units) and
// one tail element xt (kMFloor if none): the exact maximum m, then l = sum 2^{(x - m) c} (fp32
// per unit, fp64 per lane).  The tail's term is added by the caller.
template <typename T>
__device__ __forceinline__ void rows_units_core(const uint4 (&r)[kRowUnitsPerThread], int units, float xt, float c,
                                                float &m, double &l) {
  constexpr int EPU = Elem<T>::kPerUnit, U = kRowUnitsPerThread;
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int j = 0; j < U; ++j) {
    if (lane + 32 * j < units) {
      float x[EPU];
      Elem<T>::unit(r[j], x);
#pragma unroll
      for (int e = 0; e < EPU; ++e) m = fmaxf(m, x[e]);
    }
  }
  m = fmaxf(m, xt);
  const float nm = -m * c;
#pragma unroll
  for (int j = 0; j < U; ++j) {
    if (lane + 32 * j < units) {
      float x[EPU], ex[EPU];
      Elem<T>::unit(r[j], x);
#pragma unroll
      for (int e = 0; e < EPU; ++e) ex[e] = ex2(fmaf(x[e], c, nm));
#pragma unroll
      for (int s = 1; s < EPU; s <<= 1)
#pragma unroll
        for (int e = 0; e + s < EPU; e += 2 * s) ex[e] += ex[e + s];
      l += ex[0];
    }
  }
}

// One warp item (row, split): the (M, sum-exp) partial of 32 lanes x U 16-byte units of the
// target row (unit u = lane + 32 j: every load instruction reads 512 contiguous bytes).
template <typename T>
__device__ __forceinline__ float2 rows_warp_item(const VerifyArgs &a, int64_t b, int64_t i, int64_t split) {
  constexpr int EPU = Elem<T>::kPerUnit, U = kRowUnitsPerThread;
  const int lane = threadIdx.x & 31;
  const int64_t v0 = split * a.rows_chunk;
  const int n = (int)min(a.rows_chunk, (int64_t)a.V - v0);
  const T *src = trow<T>(a, b, i) + v0;
  const float c = a.ct;
  float m = kMFloor;
  double l = 0.0;
  if ((reinterpret_cast<uintptr_t>(src) & 15) == 0) {
    const int units = n / EPU;
    uint4 r[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int u = lane + 32 * j;
      if (u < units) r[j] = ldg_stream(src + (size_t)u * EPU);
    }
    const int tail = n - units * EPU;  // < EPU <= 32
    float xt = kMFloor;
    if (lane < tail) xt = Elem<T>::load(src + units * EPU + lane);
    rows_units_core<T>(r, units, xt, c, m, l);
    const float nm = -m * c;
    if (lane < tail) l += ex2(fmaf(xt, c, nm));
  } else {  // unaligned row start (edge cases): element-wise online loop
    for (int e = lane; e < n; e += 32) {
      const float x = Elem<T>::load(src + e);
      if (x > m) {
        l *= ex2((m - x) * c);
        m = x;
      }
      l += ex2(fmaf(x, c, -m * c));
    }
  }
  const float M = warp_max(m);
  const double v = warp_sum_d(l * ex2((m - M) * c));
  return make_float2(M, (float)v);
}

// Merge of target row i of sequence b (one warp): its G x splits partials (rank, split) =
// vocabulary order, lane-strided sequential, then butterfly -> (M_i, L_i) in every lane.
__device__ __forceinline__ void merge_row_warp(const VerifyArgs &a, int64_t b, int i, float &M, double &L) {
  const int lane = threadIdx.x & 31, k = a.k;
  const int64_t sp = a.splits, ns = (int64_t)a.G * sp;
  auto pidx = [&](int64_t j) { return (j / sp) * a.gs_part + (b * (k + 1) + i) * sp + j % sp; };
  const float2 *pp = a.partials;
  double l = 0.0;
  if (ns <= 128) {  // all partials in flight at once
    float2 p[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) p[j] = (lane + 32 * j < ns) ? __ldcg(pp + pidx(lane + 32 * j)) : make_float2(kMFloor, 0.f);
    float m = kMFloor;
#pragma unroll
    for (int j = 0; j < 4; ++j) m = fmaxf(m, p[j].x);
    M = warp_max(m);
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (lane + 32 * j < ns) l += (double)p[j].y * ex2((p[j].x - M) * a.ct);
  } else {
    float m = kMFloor;
    for (int64_t s = lane; s < ns; s += 32) m = fmaxf(m, __ldcg(pp + pidx(s)).x);
    M = warp_max(m);
    for (int64_t s = lane; s < ns; s += 32) {
      const float2 p = __ldcg(pp + pidx(s));
      l += (double)p.y * ex2((p.x - M) * a.ct);
    }
  }
  L = warp_sum_d(l);
}

// Per-lane inputs of the accept tests that K4 does not produce (lane i < k: draft token t_i, the
// draft normalisers and p_d(t_i) from sv_score, the target logit x_t(t_i); lane i <= k: the
// Philox block of position i).  K4b loads them BEFORE its griddepcontrol.wait: they were written
// two or more launches earlier, and every libsv kernel triggers its dependants only after its own
// wait, so K4b's launch already implies their completion (the vocab-sharded token logits come
// from a collective and are read after the wait).
struct DecidePre {
  int t;
  float dl, dpt, dmv, xt;
  uint4 w;
};
template <typename T>
__device__ __forceinline__ DecidePre decide_prefetch(const VerifyArgs &a, int64_t b) {
  const int lane = threadIdx.x & 31, k = a.k;
  DecidePre p{-1, 0.f, 0.f, 0.f, 0.f, make_uint4(0u, 0u, 0u, 0u)};
  if (lane <= k) {
    const uint64_t off = a.offset_dev ? *a.offset_dev : a.offset;  // device offset: graph replays
    if (lane < k) {
      const int64_t ri = b * k + lane;
      p.t = a.tok[ri];
      p.dl = a.dl[ri];
      p.dpt = a.dpt[ri];
      p.dmv = a.dm[ri];
      if (!a.xtok_all && p.t >= 0 && p.t < a.Vg) p.xt = Elem<T>::load(trow<T>(a, b, lane) + p.t);
    }
    p.w = sv_philox(a.seed, off, a.seq_base + b, lane);
  }
  return p;
}

// The accept tests of sequence b by one warp, lane i <= g holding row i's merged (Mi, Li):
// p_t(t_i), ratio_i = p_t(t_i) / p_d(t_i), u_i, N_b = first rejection, u_s; writes the Decision
// for K5 (+ n_accept, accept_ratio and, for a bad sequence, its sentinels).
template <typename T>
__device__ __forceinline__ void decide_warp(const VerifyArgs &a, int64_t b, int g, float Mi, double Li,
                                            const DecidePre &pre) {
  const int lane = threadIdx.x & 31, k = a.k;
  const bool gok = g >= 0 && g <= k;
  int t = -1;
  float dl = 0.f, dpt = 0.f, dmv = 0.f, xt = 0.f;
  uint4 w = make_uint4(0u, 0u, 0u, 0u);
  if (gok && lane <= g) {
    if (lane < g) {
      t = pre.t;
      dl = pre.dl;
      dpt = pre.dpt;
      dmv = pre.dmv;
      xt = pre.xt;
      if (a.xtok_all && t >= 0 && t < a.Vg) {  // vocab-sharded: the owner rank's logit (NaN elsewhere)
        xt = __int_as_float(0x7fc00000);
        for (int q = 0; q < a.G; ++q) {
          const float v = a.xtok_all[(int64_t)q * a.gs_tok + b * k + lane];
          if (xt != xt) xt = v;
        }
      }
    }
    w = pre.w;
  }
  int st = gok ? 0 : 64 /*BAD_GAMMA*/;
  const int gg = st ? -1 : g;
  if (lane > gg) {
    Mi = kMFloor;
    Li = 0.0;
  }
  int lst = 0;
  bool acc = true;
  double ratio = 0.0;
  if (lane <= gg) {
    if (!(Li == Li) || !(Mi < FLT_MAX) || !(Li < 1e300)) lst |= 1;
    else if (!(Li > 0.0)) lst |= 2;
    if (lane < gg) {
      if (!(dl == dl)) lst |= 1;
      else if (!(dl > 0.f)) lst |= 2;
      if (t < 0 || t >= a.Vg) lst |= 4;
      else if (!lst) {
        if (!(dpt > 0.f)) {
          lst |= (dpt == 0.f) ? 8 : 1;
        } else {
          const double pt = exp2((double)xt * a.ct - (double)(Mi * a.ct)) / Li;
          ratio = pt / (double)dpt;
          acc = u24(w.x) < ratio;
        }
      }
    }
  }
  // statuses of rows 0..g-1 always count; row g (target) only if it is sampled
  const unsigned rej = __ballot_sync(0xffffffffu, lane < gg && !acc);
  const int N = st ? 0 : (rej ? (__ffs(rej) - 1) : gg);
  int all = lst;
  if (lane == gg && N != gg) all = 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) all |= __shfl_xor_sync(0xffffffffu, all, o);
  st |= all;
  const float MN = __shfl_sync(0xffffffffu, Mi, st ? 0 : N);
  const double LN = __shfl_sync(0xffffffffu, Li, st ? 0 : N);
  const float dmN = __shfl_sync(0xffffffffu, dmv, N), dlN = __shfl_sync(0xffffffffu, dl, N);
  const uint32_t w1N = __shfl_sync(0xffffffffu, w.y, N);
  if (a.ratio && lane < k) a.ratio[b * k + lane] = (!st && lane < gg) ? (float)fmin(1.0, ratio) : kNaNf;
  if (lane == 0) {
    Decision dc;
    dc.N = N;
    dc.st = st;
    dc.Mt = MN;
    dc.Lt = LN;
    const bool resid = !st && N < gg;
    dc.dm = resid ? dmN : 0.f;
    dc.dl = resid ? (double)dlN : 1.0;
    dc.us = st ? 0.0 : u24(w1N);
    dc.mode = resid ? 1 : 0;  // 1 = residual, 0 = target (bonus)
    dc.pad = 0;
    a.dec[b] = dc;
    a.n_accept[b] = st ? 0 : N;
    if (st) {
      if (a.out_tok) a.out_tok[b] = -1;
      if (a.resid) a.resid[b] = kNaNf;
      if (a.status) a.status[b] = st;
    }
  }
}

// ------------------------------------------------------------------ K5
template <typename T>
struct SampleRow {
  const T *t, *d;  // target / draft row N_b
  float ct, nmt, ilt, cd, nmd, ild;
};

template <typename T>
__device__ __forceinline__ SampleRow<T> sample_row(const VerifyArgs &a, const Decision &dc, int64_t b) {
  SampleRow<T> r;
  r.t = trow<T>(a, b, dc.N);
  r.d = reinterpret_cast<const T *>(a.d) + b * a.d_sb + (int64_t)dc.N * a.d_si;
  r.ct = a.ct;
  r.nmt = -(dc.Mt * a.ct);
  r.ilt = (float)(1.0 / dc.Lt);
  r.cd = a.cd;
  r.nmd = -(dc.dm * a.cd);
  r.ild = (float)(1.0 / dc.dl);
  return r;
}

// Sum of one 16-byte unit's values in a fixed fp32 tree (packed pairs, then the two halves).
template <int EPU>
__device__ __forceinline__ float unit_tree(const f2 (&v)[EPU / 2]) {
  if constexpr (EPU == 8) {
    const f2 s = add2(add2(v[0], v[1]), add2(v[2], v[3]));
    return s.x + s.y;
  } else {
    const f2 s = add2(v[0], v[1]);
    return s.x + s.y;
  }
}

// This lane's EPT contiguous elements of warp slice s: r_v (residual when kMode = 1, else p_t),
// one fp32 tree sum per 16-byte unit (u[q]; packed FFMA2 / FMUL2 / FADD2 arithmetic), and in
// vocabulary order the fp64 sum of the unit sums (and the same for p_t, the R10 fallback mass).
// K5 and K5b's recomputation of the owning slice call this with the same arguments, so the
// unit sums are bit-identical in both.
template <typename T, int kMode, bool kKeep>
__device__ __forceinline__ bool slice_lane(const VerifyArgs &a, const SampleRow<T> &sr, int64_t s, float *r,
                                           float *u, double &sum, double &sum_t) {
  constexpr int EPU = Elem<T>::kPerUnit, UPT = kSampleUnitsPerThread, EPT = UPT * EPU;
  const int lane = threadIdx.x & 31;
  const int64_t v0 = s * a.slice + (int64_t)lane * EPT;
  const int n = (int)max((int64_t)0, min((int64_t)EPT, (int64_t)a.V - v0));
  const T *tp = sr.t + v0, *dp = sr.d + v0;
  const bool vec = n == EPT && ((reinterpret_cast<uintptr_t>(tp) & 15) == 0) &&
                   (!kMode || (reinterpret_cast<uintptr_t>(dp) & 15) == 0);
  sum = 0.0;
  sum_t = 0.0;
  if (vec) {
    uint4 ut[UPT], ud[kMode ? UPT : 1];
#pragma unroll
    for (int q = 0; q < UPT; ++q) ut[q] = *reinterpret_cast<const uint4 *>(tp + q * EPU);
    if (kMode) {
#pragma unroll
      for (int q = 0; q < UPT; ++q) ud[q] = *reinterpret_cast<const uint4 *>(dp + q * EPU);
    }
    const f2 ct{sr.ct, sr.ct}, nmt{sr.nmt, sr.nmt}, ilt{sr.ilt, sr.ilt};
    const f2 cd{sr.cd, sr.cd}, nmd{sr.nmd, sr.nmd}, ild{sr.ild, sr.ild};
#pragma unroll
    for (int q = 0; q < UPT; ++q) {
      f2 xt[EPU / 2], xd[EPU / 2], pt[EPU / 2], v[EPU / 2];
      unit_pairs<T>(ut[q], xt);
      if (kMode) unit_pairs<T>(ud[q], xd);
#pragma unroll
      for (int p = 0; p < EPU / 2; ++p) {
        pt[p] = mul2(ex2x2(fma2(xt[p], ct, nmt)), ilt);
        if (kMode) {
          const f2 dd = sub2(pt[p], mul2(ex2x2(fma2(xd[p], cd, nmd)), ild));
          v[p] = f2{fmaxf(0.f, dd.x), fmaxf(0.f, dd.y)};
        } else {
          v[p] = pt[p];
        }
        if (kKeep) {
          r[q * EPU + 2 * p] = v[p].x;
          r[q * EPU + 2 * p + 1] = v[p].y;
        }
      }
      const float uq = unit_tree<EPU>(v);
      if (kKeep) u[q] = uq;
      sum += (double)uq;
      if (kMode) sum_t += (double)unit_tree<EPU>(pt);
    }
  } else {  // ragged tail / unaligned rows: one element per "unit"
    for (int e = 0; e < EPT; ++e) {
      float v = 0.f, pt = 0.f;
      if (e < n) {
        pt = ex2(fmaf(Elem<T>::load(tp + e), sr.ct, sr.nmt)) * sr.ilt;
        v = kMode ? fmaxf(0.f, pt - ex2(fmaf(Elem<T>::load(dp + e), sr.cd, sr.nmd)) * sr.ild) : pt;
      }
      if (kKeep) r[e] = v;
      sum += (double)v;
      if (kMode) sum_t += (double)pt;
    }
  }
  if (!kMode) sum_t = sum;
  return vec;
}

// Exclusive / inclusive warp prefix (fixed Kogge-Stone order).
__device__ __forceinline__ void warp_scan_d(double v, double &incl, double &excl) {
  const int lane = threadIdx.x & 31;
  incl = warp_incl_scan_d(v, lane);
  excl = __shfl_up_sync(0xffffffffu, incl, 1);
  if (lane == 0) excl = 0.0;
}

// The sequence's last warp: Z, theta = u_s Z, the owning slice, then the token inside it.
// Prefixes over slices: chunks of 32 slices, warp scan per chunk, running total across chunks
// (all in fp64, fixed order); the owning slice is the first q with P_q + m_q > theta, and
// inside it the same test is repeated on the lanes' scan -- bit-identical at the slice end,
// so a crossing lane always exists.
template <typename T>
__device__ __forceinline__ void find_seq(const VerifyArgs &a, int64_t b) {
  constexpr int EPT = kSampleUnitsPerThread * Elem<T>::kPerUnit;
  const int lane = threadIdx.x & 31;
  const Decision dc = a.dec[b];
  if (dc.st) {  // sentinels (K4b wrote them too, except in the vocab-sharded staging)
    if (lane == 0) {
      a.out_tok[b] = -1;
      if (a.resid) a.resid[b] = kNaNf;
      if (a.status) a.status[b] = dc.st;
    }
    return;
  }
  const SampleRow<T> sr = sample_row<T>(a, dc, b);
  const int nsl = a.nsl;
  int mode = dc.mode, st = 0;
  // mass entry q of G x nsl (rank, slice) = vocabulary order; G = 1 unless vocab-sharded
  const int nq = a.G * nsl;
  auto midx = [&](int half, int q) { return (int64_t)(q / nsl) * a.gs_mass + (b * 2 + half) * nsl + q % nsl; };
  const double *sm = a.smass;
  // Z: first the residual masses; R10 (Z = 0) falls back to the target masses (same row).
  // Lane l owns the contiguous entries [q0, q1) (vocabulary order): a sequential fp64 sum per
  // lane, one fixed-order warp scan over the lanes; the crossing lane then walks its own entries
  // from its exclusive prefix.  Up to kFindChunks entries per lane stay in registers.
  const int per = (nq + 31) / 32;
  const int q0 = min(nq, lane * per), q1 = min(nq, q0 + per);
  const bool cached = per <= kFindChunks;
  double mreg[kFindChunks];
  auto mass = [&](int half, int q) { return __ldcg(sm + midx(half, q)); };
  auto lane_sum = [&](int half) {
    double s = 0.0;
    if (cached) {
#pragma unroll
      for (int j = 0; j < kFindChunks; ++j) mreg[j] = q0 + j < q1 ? mass(half, q0 + j) : 0.0;
#pragma unroll
      for (int j = 0; j < kFindChunks; ++j)
        if (q0 + j < q1) s += mreg[j];
    } else {
      for (int q = q0; q < q1; ++q) s += mass(half, q);
    }
    return s;
  };
  double Z = 0.0, lsum = 0.0, incl = 0.0, excl = 0.0;
  for (int pass = 0; pass < 2; ++pass) {
    lsum = lane_sum(mode ? 0 : 1);
    warp_scan_d(lsum, incl, excl);
    Z = __shfl_sync(0xffffffffu, incl, 31);
    if (mode == 1 && !(Z > 0.0)) {
      mode = 0;
      st = 32;  // SV_ROW_RESID_ZERO
      continue;
    }
    break;
  }
  const double theta = dc.us * Z;
  const int half = mode ? 0 : 1;
  // the owning entry: the first q with P_q + m_q > theta; if rounding leaves none (or inside the
  // crossing lane), the last entry with mass (then the token is its last positive element)
  int own = -1, pos_q = -1;
  double Pc = 0.0;
  const unsigned cross = __ballot_sync(0xffffffffu, q1 > q0 && incl > theta);
  const unsigned posl = __ballot_sync(0xffffffffu, lsum > 0.0);
  const int wl = cross ? __ffs(cross) - 1 : (posl ? 31 - __clz(posl) : -1);
  if (lane == wl) {
    double P = excl;
    auto step = [&](int q, double m) {
      if (m > 0.0) pos_q = q;
      if (cross && own < 0 && P + m > theta) {
        own = q;
        Pc = P;
      }
      P += m;
    };
    if (cached) {
#pragma unroll
      for (int j = 0; j < kFindChunks; ++j)
        if (q0 + j < q1) step(q0 + j, mreg[j]);
    } else {
      for (int q = q0; q < q1; ++q) step(q, mass(half, q));
    }
  }
  own = __shfl_sync(0xffffffffu, wl >= 0 ? own : -1, wl >= 0 ? wl : 0);
  Pc = __shfl_sync(0xffffffffu, Pc, wl >= 0 ? wl : 0);
  const int last_pos = __shfl_sync(0xffffffffu, wl >= 0 ? pos_q : -1, wl >= 0 ? wl : 0);
  const bool exact = own >= 0;
  if (!exact) own = last_pos;
  int tok = -1;
  // the owning slice lives on rank own / nsl: only that rank locates the token (others: -1)
  const int own_rank = own >= 0 ? own / nsl : -1;
  own = own >= 0 ? own % nsl : -1;
  if (own >= 0 && own_rank == a.rank) {
    constexpr int EPU = Elem<T>::kPerUnit, UPT = kSampleUnitsPerThread;
    float r[EPT], uu[UPT];
    double mine, mine_t;
    const bool vec = mode ? slice_lane<T, 1, true>(a, sr, own, r, uu, mine, mine_t)
                          : slice_lane<T, 0, true>(a, sr, own, r, uu, mine, mine_t);
    double incl, excl;
    warp_scan_d(mine, incl, excl);
    // crossing lane (exact), else the last lane with mass (fallback)
    const unsigned sel = exact ? __ballot_sync(0xffffffffu, Pc + incl > theta) : __ballot_sync(0xffffffffu, mine > 0.0);
    if (sel) {
      const int ls = exact ? __ffs(sel) - 1 : 31 - __clz(sel);
      if (lane == ls) {
        // the lane's sum is the fp64 sum of its unit sums (vec) or of its elements: find the
        // crossing unit in that order, then the element inside it by a sequential fp64 scan
        double cum = Pc + excl;
        int lastp = -1;
        if (vec) {
#pragma unroll
          for (int q = 0; q < UPT; ++q) {
            const double next = cum + (double)uu[q];
            if (exact && tok < 0 && next > theta) {
              double c2 = cum;
              int lq = -1;
#pragma unroll
              for (int e = 0; e < EPU; ++e) {
                if (r[q * EPU + e] > 0.f) lq = q * EPU + e;
                c2 += (double)r[q * EPU + e];
                if (tok < 0 && c2 > theta) tok = q * EPU + e;
              }
              if (tok < 0) tok = lq;  // rounding inside the unit: its last positive element
            }
#pragma unroll
            for (int e = 0; e < EPU; ++e)
              if (r[q * EPU + e] > 0.f) lastp = q * EPU + e;
            cum = next;
          }
        } else {
#pragma unroll
          for (int e = 0; e < EPT; ++e) {
            if (r[e] > 0.f) lastp = e;
            cum += (double)r[e];
            if (exact && tok < 0 && cum > theta) tok = e;
          }
        }
        if (tok < 0) tok = lastp;  // rounding left no crossing: the last positive element
        if (tok >= 0) tok = (int)(a.v_begin + (int64_t)own * a.slice + (int64_t)ls * EPT + tok);
      }
      tok = __shfl_sync(0xffffffffu, tok, ls);
    }
  }
  if (lane == 0) {
    a.out_tok[b] = tok;
    if (a.resid) a.resid[b] = (float)Z;
    if (a.status) a.status[b] = st;
  }
}

// One K5 warp item: slice s of sequence b's row N -> its residual mass and target mass, each the
// lane-31 value of a fixed-order warp scan.
template <typename T>
__device__ __forceinline__ void resid_item(const VerifyArgs &a, const Decision &dc, int64_t b, int64_t s) {
  const int lane = threadIdx.x & 31;
  const SampleRow<T> sr = sample_row<T>(a, dc, b);
  double mine, mine_t;
  if (dc.mode) slice_lane<T, 1, false>(a, sr, s, nullptr, nullptr, mine, mine_t);
  else slice_lane<T, 0, false>(a, sr, s, nullptr, nullptr, mine, mine_t);
  double incl, excl, incl_t, excl_t;
  warp_scan_d(mine, incl, excl);
  warp_scan_d(mine_t, incl_t, excl_t);
  if (lane == 31) {
    double *sm = a.smass + b * 2 * (int64_t)a.nsl;
    sm[s] = incl;
    sm[a.nsl + s] = incl_t;
  }
}

}  // namespace
}  // namespace sv
