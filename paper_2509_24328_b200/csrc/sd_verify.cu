// sd_verify.cu -- K4 + K5: steps a5-a6 (standard SD verification and the correction /
// bonus sample; P L29 citing Leviathan et al.; S L148-165, L82-90; DESIGN R1, R10-R13).
//
// Four kernels, each launched with programmatic dependent launch (PDL): a kernel enters
// griddepcontrol.wait before it reads anything its predecessor wrote, so the stream order is the
// only synchronisation -- there are no completion counters or spin waits in sd_verify.
//   K4  sv_rows_kernel   (persistent, warp-granular) over the COMPACTED list of (sequence b,
//       target row i <= gamma_b, vocabulary split) items -- rows past gamma_b are never read.
//       A warp streams 32 lanes x 8 16-byte units of one row and writes one (max, sum-exp)
//       partial (fp32 per unit, fp64 per lane and butterfly).
//   K4b sv_decide_kernel (one CTA of k+1 warps per sequence): warp i merges row i's partials in
//       a fixed order; warp 0 computes p_t(t_i), ratio_i = p_t(t_i) / p_d(t_i), the Philox u_i,
//       N_b = first rejection and u_s (word 1 of position N_b), and writes the sequence's
//       Decision (+ n_accept, accept_ratio).
//   K5  sv_resid_kernel  (persistent, one warp per (sequence, slice of 32 lanes x 4 contiguous
//       16-byte units)): r_v = max(0, p_t - p_d) on row N_b (or p_t for the bonus), every lane
//       summing its contiguous elements in vocabulary order in fp64; a fixed-order warp scan
//       gives the slice's residual mass and its target mass (the R10 fallback).
//   K5b sv_find_kernel   (one warp per sequence): Z and theta = u_s Z over the slice masses in
//       vocabulary order, the owning slice, its recomputation (identical bits, an L2 hit) and
//       the smallest j with cum_j > theta (R11) by warp scan + in-lane sequential scan.
// Every reduction order is a function of V and the dtype only.
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

// K4b sv_decide_kernel: one CTA of k+1 warps per sequence.  Warp i <= gamma_b merges row i's
// split partials in a fixed order (lane-strided sequential, then butterfly) into (M_i, L_i);
// warp 0 then runs the accept tests: p_t(t_i), ratio_i = p_t(t_i) / p_d(t_i), u_i, N_b =
// first rejection, and writes the Decision for K5 (+ n_accept, accept_ratio).
template <typename T>
__global__ void __launch_bounds__(32 * (SV_MAX_K_DEV + 1)) sv_decide_kernel(const __grid_constant__ VerifyArgs a) {
  __shared__ float s_M[SV_MAX_K_DEV + 1];
  __shared__ double s_L[SV_MAX_K_DEV + 1];
  pdl_wait();
  pdl_trigger();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, k = a.k;
  const int64_t b = blockIdx.x;
  const int g = a.gamma[b];
  const bool gok = g >= 0 && g <= k;
  // warp 0 issues everything the accept tests need that does not depend on the merged rows
  int t = -1;
  float dl = 0.f, dpt = 0.f, dmv = 0.f, xt = 0.f;
  uint4 w = make_uint4(0u, 0u, 0u, 0u);
  if (wid == 0 && gok && lane <= g) {
    const uint64_t off = a.offset_dev ? *a.offset_dev : a.offset;  // device offset: graph replays
    if (lane < g) {
      const int64_t ri = b * k + lane;
      t = a.tok[ri];
      dl = a.dl[ri];
      dpt = a.dpt[ri];
      dmv = a.dm[ri];
      if (t >= 0 && t < a.Vg) {
        if (a.xtok_all) {  // vocab-sharded: the owner rank's logit (NaN elsewhere)
          xt = __int_as_float(0x7fc00000);
          for (int q = 0; q < a.G; ++q) {
            const float v = a.xtok_all[(int64_t)q * a.gs_tok + b * k + lane];
            if (xt != xt) xt = v;
          }
        } else {
          xt = Elem<T>::load(trow<T>(a, b, lane) + t);
        }
      }
    }
    w = sv_philox(a.seed, off, a.seq_base + b, lane);
  }
  if (gok && wid <= g) {  // merge row wid: lane-strided sequential, then butterfly
    // partial j of G x splits (rank, split) = vocabulary order; G = 1 unless vocab-sharded
    const int64_t sp = a.splits, ns = (int64_t)a.G * sp;
    auto pidx = [&](int64_t j) { return (j / sp) * a.gs_part + (b * (k + 1) + wid) * sp + j % sp; };
    const float2 *pp = a.partials;
    float M;
    double l = 0.0;
    if (ns <= 128) {  // all partials in flight at once
      float2 p[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) p[j] = (lane + 32 * j < ns) ? pp[pidx(lane + 32 * j)] : make_float2(kMFloor, 0.f);
      float m = kMFloor;
#pragma unroll
      for (int j = 0; j < 4; ++j) m = fmaxf(m, p[j].x);
      M = warp_max(m);
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (lane + 32 * j < ns) l += (double)p[j].y * ex2((p[j].x - M) * a.ct);
    } else {
      float m = kMFloor;
      for (int64_t s = lane; s < ns; s += 32) m = fmaxf(m, pp[pidx(s)].x);
      M = warp_max(m);
      for (int64_t s = lane; s < ns; s += 32) {
        const float2 p = pp[pidx(s)];
        l += (double)p.y * ex2((p.x - M) * a.ct);
      }
    }
    const double L = warp_sum_d(l);
    if (lane == 0) {
      s_M[wid] = M;
      s_L[wid] = L;
    }
  }
  __syncthreads();
  if (wid != 0) return;

  int st = gok ? 0 : 64 /*BAD_GAMMA*/;
  const int gg = st ? -1 : g;
  float Mi = kMFloor;
  double Li = 0.0;
  int lst = 0;
  bool acc = true;
  double ratio = 0.0;
  if (lane <= gg) {
    Mi = s_M[lane];
    Li = s_L[lane];
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

// Persistent warp-granular K4 over the items (b, i <= gamma_b, split), in sequence order.
template <typename T>
__global__ void __launch_bounds__(kRowsThreads, 4) sv_rows_kernel(const __grid_constant__ VerifyArgs a) {
  constexpr int NT = kRowsThreads, NW = NT / 32;
  __shared__ int s_pref[NT + 1];
  __shared__ int s_wtot[NW];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  pdl_wait();
  pdl_trigger();
  const int splits = (int)a.splits;
  const int64_t nwarps = (int64_t)gridDim.x * NW;
  int64_t base = 0, my = (int64_t)blockIdx.x * NW + wid;
  for (int b0 = 0; b0 < a.B; b0 += NT) {
    const int nb = min(NT, a.B - b0);
    int cnt = 0;
    if (tid < nb) {
      const int g = a.gamma[b0 + tid];
      cnt = (g >= 0 && g <= a.k) ? (g + 1) * splits : 0;
    }
    int v = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += t;
    }
    __syncthreads();  // previous chunk's readers are done
    if (lane == 31) s_wtot[wid] = v;
    __syncthreads();
    int off = 0;
    for (int w = 0; w < wid; ++w) off += s_wtot[w];
    s_pref[tid + 1] = v + off;
    if (tid == 0) s_pref[0] = 0;
    __syncthreads();
    const int total = s_pref[nb];
    for (; my < base + total; my += nwarps) {
      const int local = (int)(my - base);
      int lo = 0, hi = nb - 1;  // largest j with s_pref[j] <= local (empty sequences skipped)
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (s_pref[mid] <= local) lo = mid;
        else hi = mid - 1;
      }
      const int64_t b = b0 + lo;
      const int rem = local - s_pref[lo];
      const int i = rem / splits, split = rem - i * splits;
      const float2 p = rows_warp_item<T>(a, b, i, split);
      if (lane == 0) {
        a.partials[(b * (a.k + 1) + i) * a.splits + split] = p;
        if (a.xtok_out && split == 0 && i < a.k) {  // vocab-sharded: token logit if owned, else NaN
          const int64_t loc = (int64_t)a.tok[b * a.k + i] - a.v_begin;
          a.xtok_out[b * a.k + i] = (loc >= 0 && loc < a.V)
                                        ? Elem<T>::load(trow<T>(a, b, i) + loc)
                                        : __int_as_float(0x7fc00000);
        }
      }
    }
    base += total;
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

// This lane's EPT contiguous elements of warp slice s: r_v (residual when kMode = 1, else p_t)
// and, in vocabulary order, their fp64 sum (and the fp64 sum of p_t, the R10 fallback mass).
template <typename T, int kMode, bool kKeep>
__device__ __forceinline__ void slice_lane(const VerifyArgs &a, const SampleRow<T> &sr, int64_t s, float *r,
                                           double &sum, double &sum_t) {
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
#pragma unroll
    for (int q = 0; q < UPT; ++q) {
      float xt[EPU], xd[EPU];
      Elem<T>::unit(ut[q], xt);
      if (kMode) Elem<T>::unit(ud[q], xd);
#pragma unroll
      for (int e = 0; e < EPU; ++e) {
        const float pt = ex2(fmaf(xt[e], sr.ct, sr.nmt)) * sr.ilt;
        const float v = kMode ? fmaxf(0.f, pt - ex2(fmaf(xd[e], sr.cd, sr.nmd)) * sr.ild) : pt;
        if (kKeep) r[q * EPU + e] = v;
        sum += (double)v;
        if (kMode) sum_t += (double)pt;
      }
    }
  } else {
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
__global__ void __launch_bounds__(256) sv_find_kernel(const __grid_constant__ VerifyArgs a) {
  constexpr int EPT = kSampleUnitsPerThread * Elem<T>::kPerUnit;
  const int lane = threadIdx.x & 31;
  pdl_wait();
  pdl_trigger();
  const int64_t b = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (b >= a.B) return;
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
  // Slices go in chunks of 32 (one warp scan each, running total across chunks); the loads of
  // kFindChunks chunks are issued together.
  double Z = 0.0;
  // one chunk group covers every slice (V <= 32 kFindChunks slices): the crossing scan below
  // reuses these registers instead of loading the masses again
  double mc[kFindChunks];
  int mc_half = -1;
  for (int pass = 0; pass < 2; ++pass) {
    const int half = mode ? 0 : 1;
    double run = 0.0;
    for (int c0 = 0; c0 < nq; c0 += 32 * kFindChunks) {
      double m[kFindChunks];
#pragma unroll
      for (int j = 0; j < kFindChunks; ++j) {
        const int q = c0 + 32 * j + lane;
        m[j] = q < nq ? __ldcg(sm + midx(half, q)) : 0.0;
      }
      if (nq <= 32 * kFindChunks) {
#pragma unroll
        for (int j = 0; j < kFindChunks; ++j) mc[j] = m[j];
        mc_half = half;
      }
#pragma unroll
      for (int j = 0; j < kFindChunks; ++j) {
        if (c0 + 32 * j >= nq) break;
        double incl, excl;
        warp_scan_d(m[j], incl, excl);
        run += __shfl_sync(0xffffffffu, incl, 31);
      }
    }
    Z = run;
    if (mode == 1 && !(Z > 0.0)) {
      mode = 0;
      st = 32;  // SV_ROW_RESID_ZERO
      continue;
    }
    break;
  }
  const double theta = dc.us * Z;
  const int half = mode ? 0 : 1;
  double run = 0.0, Pc = 0.0;
  int own = -1, last_pos = -1;
  for (int c0 = 0; c0 < nq; c0 += 32 * kFindChunks) {
    double mm[kFindChunks];
#pragma unroll
    for (int j = 0; j < kFindChunks; ++j) {
      const int q = c0 + 32 * j + lane;
      mm[j] = mc_half == half ? mc[j] : (q < nq ? __ldcg(sm + midx(half, q)) : 0.0);
    }
#pragma unroll
    for (int j = 0; j < kFindChunks; ++j) {
      const int cj = c0 + 32 * j;
      if (cj >= nq) break;
      const bool valid = cj + lane < nq;
      const double m = mm[j];
      double incl, excl;
      warp_scan_d(m, incl, excl);
      const double P = run + excl;
      const unsigned pos = __ballot_sync(0xffffffffu, valid && m > 0.0);
      if (pos) last_pos = cj + 31 - __clz(pos);
      if (own < 0) {
        const unsigned cross = __ballot_sync(0xffffffffu, valid && P + m > theta);
        if (cross) {
          const int l = __ffs(cross) - 1;
          own = cj + l;
          Pc = __shfl_sync(0xffffffffu, P, l);
        }
      }
      run += __shfl_sync(0xffffffffu, incl, 31);
    }
  }
  const bool exact = own >= 0;
  if (!exact) own = last_pos;
  int tok = -1;
  // the owning slice lives on rank own / nsl: only that rank locates the token (others: -1)
  const int own_rank = own >= 0 ? own / nsl : -1;
  own = own >= 0 ? own % nsl : -1;
  if (own >= 0 && own_rank == a.rank) {
    float r[EPT];
    double mine, mine_t;
    if (mode) slice_lane<T, 1, true>(a, sr, own, r, mine, mine_t);
    else slice_lane<T, 0, true>(a, sr, own, r, mine, mine_t);
    double incl, excl;
    warp_scan_d(mine, incl, excl);
    // crossing lane (exact), else the last lane with mass (fallback)
    const unsigned sel = exact ? __ballot_sync(0xffffffffu, Pc + incl > theta) : __ballot_sync(0xffffffffu, mine > 0.0);
    if (sel) {
      const int ls = exact ? __ffs(sel) - 1 : 31 - __clz(sel);
      if (lane == ls) {
        double cum = Pc + excl;
        int lastp = -1;
#pragma unroll
        for (int e = 0; e < EPT; ++e) {
          if (r[e] > 0.f) lastp = e;
          cum += (double)r[e];
          if (exact && tok < 0 && cum > theta) tok = e;
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

// Persistent warp-granular K5 over the B x nsl warp slices: per slice the residual mass and
// the target mass (the R10 fallback), each the lane-31 value of a fixed-order warp scan.
template <typename T>
__global__ void __launch_bounds__(kSampleThreads, 3) sv_resid_kernel(const __grid_constant__ VerifyArgs a) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  pdl_wait();
  pdl_trigger();
  const int64_t nwarps = (int64_t)gridDim.x * (kSampleThreads / 32);
  const int64_t items = (int64_t)a.B * a.nsl;
  for (int64_t it = (int64_t)blockIdx.x * (kSampleThreads / 32) + wid; it < items; it += nwarps) {
    const int64_t b = it / a.nsl, s = it - b * a.nsl;
    const Decision dc = a.dec[b];
    if (dc.st) continue;  // K4b wrote the sentinels
    const SampleRow<T> sr = sample_row<T>(a, dc, b);
    double mine, mine_t;
    if (dc.mode) slice_lane<T, 1, false>(a, sr, s, nullptr, mine, mine_t);
    else slice_lane<T, 0, false>(a, sr, s, nullptr, mine, mine_t);
    double incl, excl, incl_t, excl_t;
    warp_scan_d(mine, incl, excl);
    warp_scan_d(mine_t, incl_t, excl_t);
    if (lane == 31) {
      double *sm = a.smass + b * 2 * (int64_t)a.nsl;
      sm[s] = incl;
      sm[a.nsl + s] = incl_t;
    }
  }
}

}  // namespace

int64_t verify_ws_bytes(int64_t B, int k, int64_t splits, int nsl) {
  return ws_round(B * (k + 1) * splits * 8) + ws_round(B * (int64_t)sizeof(Decision)) + ws_round(B * nsl * 16);
}

// stage 0: K4 rows, 1: K4b decide, 2: K5 residual slices, 3: K5b token search
cudaError_t launch_verify_stage(int stage, const VerifyArgs &a, cudaStream_t st) {
  switch (stage) {
    case 0: {  // K4: persistent over the compacted (sequence, row <= gamma, split) items
      const void *fn = a.bf16 ? (const void *)sv_rows_kernel<__nv_bfloat16> : (const void *)sv_rows_kernel<float>;
      const int64_t need = ((int64_t)a.B * (a.k + 1) * a.splits + kRowsThreads / 32 - 1) / (kRowsThreads / 32);
      const int64_t grid = need < resident_grid(fn, kRowsThreads, 0) ? need : resident_grid(fn, kRowsThreads, 0);
      return a.bf16 ? launch_k(sv_rows_kernel<__nv_bfloat16>, dim3((unsigned)grid), dim3(kRowsThreads), 0, st, a)
                    : launch_k(sv_rows_kernel<float>, dim3((unsigned)grid), dim3(kRowsThreads), 0, st, a);
    }
    case 1:
      return a.bf16 ? launch_k(sv_decide_kernel<__nv_bfloat16>, dim3((unsigned)a.B), dim3(32 * (a.k + 1)), 0, st, a)
                    : launch_k(sv_decide_kernel<float>, dim3((unsigned)a.B), dim3(32 * (a.k + 1)), 0, st, a);
    case 2: {
      const void *fn = a.bf16 ? (const void *)sv_resid_kernel<__nv_bfloat16> : (const void *)sv_resid_kernel<float>;
      const int64_t need = ((int64_t)a.B * a.nsl + kSampleThreads / 32 - 1) / (kSampleThreads / 32);
      const int64_t grid = need < resident_grid(fn, kSampleThreads, 0) ? need : resident_grid(fn, kSampleThreads, 0);
      return a.bf16 ? launch_k(sv_resid_kernel<__nv_bfloat16>, dim3((unsigned)grid), dim3(kSampleThreads), 0, st, a)
                    : launch_k(sv_resid_kernel<float>, dim3((unsigned)grid), dim3(kSampleThreads), 0, st, a);
    }
    default: {
      const unsigned fgrid = (unsigned)((a.B + 7) / 8);
      return a.bf16 ? launch_k(sv_find_kernel<__nv_bfloat16>, dim3(fgrid), dim3(256), 0, st, a)
                    : launch_k(sv_find_kernel<float>, dim3(fgrid), dim3(256), 0, st, a);
    }
  }
}

cudaError_t launch_verify(const VerifyArgs &a, cudaStream_t st) {
  for (int stage = 0; stage < 4; ++stage) {
    const cudaError_t e = launch_verify_stage(stage, a, st);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace sv
