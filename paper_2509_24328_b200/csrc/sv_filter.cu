// sv_filter.cu -- NEXT-2: the SV path under the paper's sampling filters (P L731-743 Table 5:
// top_k 20 / top_p 0.8 / tau 0.7 for Qwen), applied to draft, companion and target alike before
// S / A and the accept test (S L73-81, L183, L238; DESIGN R21).  With top_k <= 32 every filtered
// distribution has at most 32 support entries, so after one selection pass per row the rest of
// the path runs on tiny lists:
//
//   KF1 sv_topk_kernel  one CTA per row: the minimum of the 32 half-warp maxima bounds the
//                       top_k-th largest key from below, so one more pass gathers the few keys
//                       above it, ranked by counting; on overflow: radix select of the top_k-th
//                       largest logit on the
//                       order-preserving key of the raw bits (bf16: 2 passes of 8 bits, fp32: 4),
//                       256-bin shared-memory histograms over the row (the first pass streams
//                       it from HBM, the rest hit L2), then one collection pass: keys above the
//                       threshold in any order, keys equal to it in VOCABULARY order until
//                       top_k entries are held (ties to the lower index, R21); the list is
//                       sorted by (logit desc, index asc), softmaxed in fp64 over the kept
//                       entries, cut by top_p (sequential fp64 cumulative >= top_p) and
//                       renormalised -> FList {n, idx[32], p[32]}.
//   KF2 sv_fscore_kernel one warp per (b, i): S = sum min(p'_d, p'_c) over the draft list,
//                       A = min(1, p'_c(t)/p'_d(t)), KL(p'_d || p'_c), profile lookup.
//   KF3 sv_fverify_kernel one warp per sequence: p'_t(t_i)/p'_d(t_i), Philox u_i, N_b, then
//                       the residual max(0, p'_t - p'_d) (or the bonus p'_t) over the <= 32
//                       entries sorted by vocabulary index, sequential fp64 Z and inverse CDF.
#include <float.h>

#include "sv_device.cuh"
#include "sv_internal.h"

namespace sv {

namespace {

constexpr int kTopKThreads = 512;  // 256: 0.18 ms, 1024: 0.25 ms at the headline (512: 0.17)
constexpr int kHistCopies = kTopKThreads / 32 < 16 ? kTopKThreads / 32 : 16;  // private histograms
constexpr int kTieCap = 2048;   // tie indices held for the ordered pick (power of two)
constexpr int kCandCap = 2048;  // fast-path candidates (ranked by counting: O(n^2 / threads))

template <typename T> struct KeyOf;
template <> struct KeyOf<__nv_bfloat16> {
  using K = uint32_t;
  static constexpr int kBits = 16;
  __device__ static K key(const __nv_bfloat16 *p, int64_t e) {
    const uint32_t b = *reinterpret_cast<const uint16_t *>(p + e);
    return (b & 0x8000u) ? (~b & 0xFFFFu) : (b | 0x8000u);
  }
  // +inf or NaN of either sign (R18): +inf / +NaN map to keys >= 0xFF80, -NaN to keys <= 0x007E
  __device__ static bool bad(K k) { return k >= 0xFF80u || k < 0x007Fu; }
  __device__ static float value(K k) { return __uint_as_float(value_bits(k)); }
  __device__ static uint32_t value_bits(K k) {  // fp32 bits of the logit of key k
    const uint32_t b = (k & 0x8000u) ? (k & 0x7FFFu) : (~k & 0xFFFFu);
    return b << 16;
  }
};
template <> struct KeyOf<float> {
  using K = uint32_t;
  static constexpr int kBits = 32;
  __device__ static K key(const float *p, int64_t e) {
    const uint32_t b = __float_as_uint(p[e]);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
  }
  __device__ static bool bad(K k) { return k >= 0xFF800000u || k < 0x007FFFFFu; }  // (as above)
  __device__ static float value(K k) { return __uint_as_float(value_bits(k)); }
  __device__ static uint32_t value_bits(K k) { return (k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k; }
};

// order-preserving keys of the 8 consecutive elements v0 .. v0+7 (L2-resident re-reads: plain
// vector loads when the row is 16-byte aligned; entries at or beyond V are left 0 -- callers mask)
template <typename T>
__device__ __forceinline__ void load8(const T *x, int v0, int V, bool vec, uint32_t (&kk)[8]) {
  using KO = KeyOf<T>;
  if (vec && v0 + 8 <= V) {
    uint4 w[sizeof(T) / 2];
#pragma unroll
    for (int q = 0; q < (int)(sizeof(T) / 2); ++q) w[q] = __ldg(reinterpret_cast<const uint4 *>(x + v0) + q);
    const T *e = reinterpret_cast<const T *>(w);
#pragma unroll
    for (int j = 0; j < 8; ++j) kk[j] = KO::key(e, j);
  } else {
#pragma unroll
    for (int j = 0; j < 8; ++j) kk[j] = v0 + j < V ? KO::key(x, v0 + j) : 0u;
  }
}

// Row r of the set the launch processes (draft / companion rows for the score, target rows
// 0..gamma_b for the verify); returns false for rows that are skipped.
__device__ __forceinline__ bool row_of(const FilterArgs &a, int64_t r, int which, const void *&base, int64_t &off,
                                       FList *&out) {
  if (which == 2) {  // target rows (b, i <= gamma_b)
    const int64_t b = r / (a.k + 1), i = r % (a.k + 1);
    const int g = a.gamma[b];
    if (g < 0 || g > a.k || i > g) return false;
    base = a.t;
    off = b * a.t_sb + i * a.t_si;
    out = a.tl + r;
    return true;
  }
  const int64_t b = r / a.k, i = r % a.k;
  base = which == 0 ? a.d : a.c;
  off = which == 0 ? b * a.d_sb + i * a.d_si : b * a.c_sb + i * a.c_si;
  out = (which == 0 ? a.dl : a.cl) + r;
  return true;
}

// kNuc: nucleus-only (top_k = 0) -- a separate instantiation so the top-k path's registers and
// schedule do not carry the normaliser's code; it runs 4 CTAs per SM (32 registers: nucleus step
// 0.455 -> 0.445 ms), the top-k path 3 (40 registers; 4 measured 5 % slower)
template <typename T, bool kNuc>
__global__ void __launch_bounds__(kTopKThreads, kNuc ? 4 : 3) sv_topk_kernel(const __grid_constant__ FilterArgs a, int which0) {
  const int which = which0 + (int)blockIdx.y;  // score: y = 0 draft rows, y = 1 companion rows
  using KO = KeyOf<T>;
  using K = typename KO::K;
  constexpr int NT = kTopKThreads;
  __shared__ uint32_t hist[256];
  __shared__ K s_prefix, s_mask;
  __shared__ int s_remaining, s_bad, s_ngt, s_ntie;
  __shared__ int s_tie[kTieCap];
  __shared__ unsigned long long s_cand[kCandCap];
  __shared__ uint32_t s_gmax[32];
  __shared__ double s_lsum[kTopKThreads / 32], s_lfull;
  __shared__ int s_ncand;
  __shared__ K c_key[32];
  __shared__ int c_idx[32];
  pdl_wait();
  pdl_trigger();
  const void *base;
  int64_t off;
  FList *out;
  if (!row_of(a, blockIdx.x, which, base, off, out)) return;
  const T *x = reinterpret_cast<const T *>(base) + off;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  // top_k = 0: nucleus-only (top_p over the FULL distribution), supported when the nucleus has
  // at most 32 tokens -- the 32 largest are selected and the full-row normaliser is added below
  constexpr bool nucleus = kNuc;  // the launch picks kNuc = (a.top_k == 0)
  const int V = a.V, KK = min(nucleus ? 32 : a.top_k, V);
  if (tid == 0) {
    s_prefix = 0;
    s_mask = 0;
    s_remaining = KK;
    s_bad = 0;
    s_ngt = 0;
    s_ntie = 0;
  }
  bool fast = false;
  const double tau = (double)(which == 0 ? a.tau_d : which == 1 ? a.tau_c : a.tau_t);
  const float c2n = (float)(1.4426950408889634 / tau);
  float om = -FLT_MAX, ol = 0.f;
  // ---- fast path: the KK-th largest of the 512 thread maxima is a lower bound of the KK-th
  // largest key, so every top-KK element has key >= that bound; gather those few candidates
  // (second pass, an L2 hit) and sort them by (key desc, index asc).  Falls back to the radix
  // select when the candidates overflow kCandCap.
  {
    constexpr int EPU = 16 / sizeof(T);
    const bool vec = (reinterpret_cast<uintptr_t>(x) & 15) == 0;
    const int units = vec ? V / EPU : 0;
    K tmax = 0;
    int bad = 0;
    constexpr int UF = 4;  // independent 16-byte loads in flight per thread
    // nucleus-only: the full-row normaliser rides on this pass as a per-thread online sum
    // ol = sum 2^{(x - om) log2e / tau}, rescaled when a unit raises the running max om
    for (int u0 = tid; u0 < units; u0 += UF * NT) {
      uint4 w[UF];
#pragma unroll
      for (int q = 0; q < UF; ++q) {
        const int u = u0 + q * NT;
        w[q] = u < units ? ldg_stream(x + (size_t)u * EPU) : make_uint4(0u, 0u, 0u, 0u);
      }
#pragma unroll
      for (int q = 0; q < UF; ++q) {
        if (u0 + q * NT >= units) continue;
        const T *e = reinterpret_cast<const T *>(&w[q]);
        K um = 0;
        auto keys_max = [&]() {
#pragma unroll
          for (int j = 0; j < EPU; ++j) {
            const K kk = KO::key(e, j);
            um = kk > um ? kk : um;
            bad |= KO::bad(kk);
          }
        };
        if constexpr (sizeof(T) == 2) {
          // bf16: NaN-propagating packed maxima of the 8 values, then the keys of the 2 survivors
          // (for non-NaN values the float order is the key order except +-0, whose keys differ
          // by one: either survivor is an element of the unit, so the group bound stays valid; a
          // NaN of either sign or +inf survives and flags the row)
          const __nv_bfloat162 *h2 = reinterpret_cast<const __nv_bfloat162 *>(&w[q]);
          const __nv_bfloat162 m2 = __hmax2_nan(__hmax2_nan(h2[0], h2[1]), __hmax2_nan(h2[2], h2[3]));
          const uint32_t mb = *reinterpret_cast<const uint32_t *>(&m2);
          const __nv_bfloat16 lo = __ushort_as_bfloat16((unsigned short)(mb & 0xFFFFu));
          const __nv_bfloat16 hi = __ushort_as_bfloat16((unsigned short)(mb >> 16));
          const K k0 = KO::key(&lo, 0), k1 = KO::key(&hi, 0);
          um = k0 > k1 ? k0 : k1;
          bad |= KO::bad(k0) | KO::bad(k1);
        } else {
          keys_max();
        }
        tmax = um > tmax ? um : tmax;
        if (nucleus) {
          const float umv = KO::value(um);
          if (umv > om) {
            ol *= ex2((om - umv) * c2n);
            om = umv;
          }
          const float nm = -om * c2n;
          if constexpr (sizeof(T) == 2) {  // packed FFMA2 arguments, fixed FADD2 tree per unit
            f2 xv[EPU / 2];
            unit_pairs<T>(w[q], xv);
            const f2 cc{c2n, c2n}, nm2{nm, nm};
            f2 ev[EPU / 2];
#pragma unroll
            for (int p2 = 0; p2 < EPU / 2; ++p2) ev[p2] = ex2x2(fma2(xv[p2], cc, nm2));
            const f2 t = add2(add2(ev[0], ev[1]), add2(ev[2], ev[3]));
            ol += t.x + t.y;
          } else {
#pragma unroll
            for (int j = 0; j < EPU; ++j) ol += ex2(fmaf(KO::value(KO::key(e, j)), c2n, nm));
          }
        }
      }
    }
    for (int e = units * EPU + tid; e < V; e += NT) {
      const K kk = KO::key(x, e);
      tmax = kk > tmax ? kk : tmax;
      bad |= KO::bad(kk);
      if (nucleus) {
        const float v = KO::value(kk);
        if (v > om) {
          ol *= ex2((om - v) * c2n);
          om = v;
        }
        ol += ex2(fmaf(v, c2n, -om * c2n));
      }
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) s_bad = 1;
    __syncthreads();
    // lower bound: the minimum of the maxima of 32 thread groups (NT/32 lanes each) -- 32 distinct
    // elements are >= it, so the KK-th largest (KK <= 32) is too (no sort of the maxima needed)
    constexpr int GL = NT / 32;
    static_assert(GL >= 1 && GL <= 32, "32 groups of lanes");
    K gmax = tmax;
#pragma unroll
    for (int o = GL / 2; o > 0; o >>= 1) {
      const K v = __shfl_xor_sync(0xffffffffu, gmax, o);
      gmax = v > gmax ? v : gmax;
    }
    if ((lane & (GL - 1)) == 0) s_gmax[tid / GL] = gmax;
    __syncthreads();
    K lb = s_gmax[0];
#pragma unroll 8
    for (int g = 1; g < 32; ++g) lb = s_gmax[g] < lb ? s_gmax[g] : lb;
    if (tid == 0) s_ncand = 0;
    __syncthreads();
    for (int u0 = tid; u0 < units; u0 += UF * NT) {
      uint4 w[UF];
#pragma unroll
      for (int q = 0; q < UF; ++q) {
        const int u = u0 + q * NT;
        w[q] = u < units ? ldg_stream(x + (size_t)u * EPU) : make_uint4(0u, 0u, 0u, 0u);
      }
#pragma unroll
      for (int q = 0; q < UF; ++q) {
        const int u = u0 + q * NT;
        if (u >= units) continue;
        const T *e = reinterpret_cast<const T *>(&w[q]);
        if constexpr (sizeof(T) == 2) {  // skip units whose packed maximum is below the bound
          const __nv_bfloat162 *h2 = reinterpret_cast<const __nv_bfloat162 *>(&w[q]);
          const __nv_bfloat162 m2 = __hmax2_nan(__hmax2_nan(h2[0], h2[1]), __hmax2_nan(h2[2], h2[3]));
          const uint32_t mb = *reinterpret_cast<const uint32_t *>(&m2);
          const __nv_bfloat16 lo = __ushort_as_bfloat16((unsigned short)(mb & 0xFFFFu));
          const __nv_bfloat16 hi = __ushort_as_bfloat16((unsigned short)(mb >> 16));
          const K k0 = KO::key(&lo, 0), k1 = KO::key(&hi, 0);
          if ((k0 > k1 ? k0 : k1) + 1u < lb) continue;  // (+1: -0 and +0 are one key apart)
        }
#pragma unroll
        for (int j = 0; j < EPU; ++j) {
          const K kk = KO::key(e, j);
          if (kk >= lb) {
            const int slot = atomicAdd(&s_ncand, 1);
            if (slot < kCandCap)
              s_cand[slot] = ((unsigned long long)kk << 32) | (0xFFFFFFFFu - (uint32_t)(u * EPU + j));
          }
        }
      }
    }
    for (int e = units * EPU + tid; e < V; e += NT) {
      const K kk = KO::key(x, e);
      if (kk >= lb) {
        const int slot = atomicAdd(&s_ncand, 1);
        if (slot < kCandCap) s_cand[slot] = ((unsigned long long)kk << 32) | (0xFFFFFFFFu - (uint32_t)e);
      }
    }
    __syncthreads();
    const int nc = s_ncand;
    if (nc <= kCandCap) {  // rank by counting on the unique composite (key desc, index asc)
      for (int j = tid; j < nc; j += NT) {
        const unsigned long long cj = s_cand[j];
        int rank = 0;
        for (int i = 0; i < nc; ++i) rank += s_cand[i] > cj;
        if (rank < KK) {
          c_key[rank] = (K)(cj >> 32);
          c_idx[rank] = (int)(0xFFFFFFFFu - (uint32_t)cj);
        }
      }
      fast = true;
    }
    __syncthreads();
  }
  if (!fast) {
    // ---- radix select of the KK-th largest key, 8 bits per pass from the top
    for (int shift = KO::kBits - 8; shift >= 0; shift -= 8) {
      for (int j = tid; j < 256; j += NT) hist[j] = 0u;
      __syncthreads();
      const K prefix = s_prefix, mask = s_mask;
      int bad = 0;
      for (int e = tid; e < V; e += NT) {
        const K kk = KO::key(x, e);
        bad |= KO::bad(kk);
        if ((kk & mask) == prefix) atomicAdd(&hist[(kk >> shift) & 255u], 1u);
      }
      if (shift == KO::kBits - 8 && __any_sync(0xffffffffu, bad) && lane == 0) s_bad = 1;
      __syncthreads();
      if (tid == 0) {
        int rem = s_remaining, cum = 0, d = 255;
        for (; d > 0; --d) {
          if (cum + (int)hist[d] >= rem) break;
          cum += (int)hist[d];
        }
        s_remaining = rem - cum;  // still to take inside digit d
        s_prefix = prefix | ((K)d << shift);
        s_mask = mask | ((K)255u << shift);
      }
      __syncthreads();
    }
    const K theta = s_prefix;
    const int need = s_remaining;  // entries equal to theta to take, lowest indices first
    // ---- collection: keys > theta (< top_k of them, any order) and the indices of keys ==
    // theta (up to kTieCap, any order); the `need` lowest tie indices are then taken in order
    for (int e = tid; e < V; e += NT) {
      const K kk = KO::key(x, e);
      if (kk > theta) {
        const int slot = atomicAdd(&s_ngt, 1);
        c_key[slot] = kk;
        c_idx[slot] = e;
      } else if (kk == theta) {
        const int slot = atomicAdd(&s_ntie, 1);
        if (slot < kTieCap) s_tie[slot] = e;
      }
    }
    __syncthreads();
    const int ntie = s_ntie;
    if (ntie <= kTieCap) {  // bitonic sort of the tie indices (padded with INT32_MAX)
      int np2 = 1;
      while (np2 < ntie) np2 <<= 1;
      for (int j = ntie + tid; j < np2; j += NT) s_tie[j] = INT32_MAX;
      __syncthreads();
      for (int size = 2; size <= np2; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
          for (int j = tid; j < np2; j += NT) {
            const int o = j ^ stride;
            if (o > j) {
              const bool up = (j & size) == 0;
              const int u = s_tie[j], v = s_tie[o];
              if ((u > v) == up) {
                s_tie[j] = v;
                s_tie[o] = u;
              }
            }
          }
          __syncthreads();
        }
      }
      if (tid < need) {
        c_key[KK - need + tid] = theta;
        c_idx[KK - need + tid] = s_tie[tid];
      }
    } else {  // pathological tie counts: one ordered pass (warp 0, vocabulary order)
      if (wid == 0) {
        int taken = 0;
        for (int e0 = 0; e0 < V && taken < need; e0 += 32) {
          const int e = e0 + lane;
          const bool eq = e < V && KO::key(x, e) == theta;
          const unsigned m = __ballot_sync(0xffffffffu, eq);
          const int rank = taken + __popc(m & ((1u << lane) - 1u));
          if (eq && rank < need) {
            c_key[KK - need + rank] = theta;
            c_idx[KK - need + rank] = e;
          }
          taken += __popc(m);
        }
      }
    }
    __syncthreads();
  }
  if (nucleus) {  // full-row normaliser sum_v 2^{(x_v - x_max) log2e / tau}: merge of the pass-1
                  // online sums (fp64 block sum)
    K kmax = c_key[0];
    for (int j = 1; j < KK; ++j) kmax = c_key[j] > kmax ? c_key[j] : kmax;
    const float xmax = KO::value(kmax);
    const float lsum = (xmax > -FLT_MAX && ol > 0.f) ? ol * ex2((om - xmax) * c2n) : 0.f;
    double v = warp_sum_d((double)lsum);
    if (lane == 0) s_lsum[wid] = v;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < NT / 32; ++w) t += s_lsum[w];
      s_lfull = t;
    }
    __syncthreads();
  }
  __shared__ int s_wide;
  __shared__ double s_y0;
  if (wid == 0) {
    // ---- sort by (key desc, index asc), softmax (fp64), top_p, renormalise
    const K mk = lane < KK ? c_key[lane] : (K)0;
    const int mi = lane < KK ? c_idx[lane] : INT32_MAX;
    int rank = 0;
    for (int l = 0; l < KK; ++l) {
      const K ok = __shfl_sync(0xffffffffu, mk, l);
      const int oi = __shfl_sync(0xffffffffu, mi, l);
      rank += (ok > mk) || (ok == mk && oi < mi);
    }
    __syncwarp();
    if (lane < KK) {
      c_key[rank] = mk;
      c_idx[rank] = mi;
    }
    __syncwarp();
    const double y = lane < KK ? (double)KO::value(c_key[lane]) / tau : -INFINITY;
    const double y0 = __shfl_sync(0xffffffffu, y, 0);
    int st = s_bad ? 1 /*SV_ROW_NAN*/ : 0;
    if (!st && !(y0 > -INFINITY)) st = 2; /*SV_ROW_ALL_NEG_INF*/
    double p = (lane < KK && !st) ? exp(y - y0) : 0.0;
    double tot = 0.0;  // sequential in sorted order (the oracle's order); nucleus: the full row
    if (nucleus) tot = s_lfull;
    else
      for (int l = 0; l < KK; ++l) tot += __shfl_sync(0xffffffffu, p, l);
    p = p / tot;
    int n = KK;
    bool wide = false;
    double s = 1.0;
    if (a.top_p < 1.f) {
      double c = 0.0;
      bool cut = false;
      for (int l = 0; l < KK; ++l) {
        c += __shfl_sync(0xffffffffu, p, l);
        if (c >= (double)a.top_p) {
          n = l + 1;
          cut = true;
          break;
        }
      }
      wide = nucleus && !cut && !st;  // nucleus larger than 32 tokens: threshold form below
      s = 0.0;
      for (int l = 0; l < n; ++l) s += __shfl_sync(0xffffffffu, p, l);
      p = p / s;
    }
    if (st || wide) n = 0;
    if (lane < n) {
      out->idx[lane] = c_idx[lane];
      out->p[lane] = p;
    }
    if (lane == 0) {
      out->n = n;
      out->st = st;
      out->wide = wide;
      out->tau = tau;
      out->y0 = y0;
      out->tot = tot;
      if (!wide) {
        out->s = s;
        out->th_key = n ? (uint32_t)c_key[n - 1] : 0xFFFFFFFFu;
        out->th_idx = n ? c_idx[n - 1] : -1;
      }
      s_wide = wide;
      s_y0 = y0;
    }
  }
  __syncthreads();
  if (!s_wide) return;
  // ---- nucleus larger than 32 tokens (threshold form).  Digit histograms (8 bits per level from
  // the top) of counts and 2^-31 fixed-point masses (native 32-bit shared atomics, per-warp
  // copies) bound the cumulative mass from below and above; they locate a band of keys [L, U)
  // that surely holds the cut, refined digit by digit until it has at most kCandCap keys.  The
  // keys >= U are surely inside the nucleus: their exact fp64 mass c_U is summed in a fixed order;
  // the band is gathered, sorted by (key desc, index asc) and the cut taken as the oracle does
  // (p_j = exp(y_j - y0) / tot, sequential cumulative from c_U until >= top_p).  Deterministic.
  {
    __shared__ unsigned s_msum[256];
    __shared__ unsigned long long s_am, s_ahi, s_L, s_U;
    __shared__ double s_cu;
    __shared__ int s_state;  // 0 refine, 1 gather with L = s_prefix, 2 fall back
    __shared__ double s_pm[kCandCap];
    const double y0 = s_y0, tot = s_lfull;
    const float c2 = (float)(1.4426950408889634 / tau), nm = -KO::value(c_key[0]) * c2;
    const float scale31 = (float)(2147483648.0 / tot);
    const unsigned long long target = (unsigned long long)((double)a.top_p * 2147483648.0);
    const bool vec = (reinterpret_cast<uintptr_t>(x) & 15) == 0;
    if (tid == 0) {
      s_prefix = 0;
      s_mask = 0;
      s_am = 0ull;
      s_ahi = 0ull;
      s_state = 0;
      s_ncand = 0;
    }
    // per-warp private histograms (counts in the candidate buffer, masses in the p buffer -- both
    // free until the gather): same-address contention stays inside a warp
    unsigned *wc = reinterpret_cast<unsigned *>(s_cand) + (wid % kHistCopies) * 256;
    unsigned *wmass = reinterpret_cast<unsigned *>(s_pm) + (wid % kHistCopies) * 256;
    static_assert(kCandCap * 2 >= kHistCopies * 256, "private histograms must fit");
    for (int shift = KO::kBits - 8; shift >= 0; shift -= 8) {
      for (int j = lane; j < 256; j += 32) {
        wc[j] = 0u;
        wmass[j] = 0u;
      }
      __syncthreads();
      const K prefix = s_prefix, mask = s_mask;
      for (int v0 = tid * 8; v0 < V; v0 += NT * 8) {
        uint32_t kk[8];
        load8(x, v0, V, vec, kk);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (v0 + j < V && (kk[j] & mask) == prefix) {
            const unsigned d = (kk[j] >> shift) & 255u;
            atomicAdd(&wc[d], 1u);
            const unsigned mf = __float2uint_rz(ex2(fmaf(KO::value(kk[j]), c2, nm)) * scale31);
            if (mf) atomicAdd(&wmass[d], mf);
          }
        }
      }
      __syncthreads();
      if (tid < 256) {
        const unsigned *c0 = reinterpret_cast<const unsigned *>(s_cand);
        const unsigned *m0 = reinterpret_cast<const unsigned *>(s_pm);
        unsigned c = 0u, m = 0u;
        for (int w = 0; w < kHistCopies; ++w) {
          c += c0[w * 256 + tid];
          m += m0[w * 256 + tid];
        }
        hist[tid] = c;
        s_msum[tid] = m;
      }
      __syncthreads();
      if (tid == 0) {
        // lower / upper bounds of the cumulative mass from the top (truncation: each element's
        // fixed-point mass is low by < 1 unit, so hi = lo + count bounds it from above; eps covers
        // the fp32 ex2 terms).  Digits above da are surely inside the nucleus, digits from ds up
        // surely contain it: the cut lies in the band [ds, da].
        const unsigned long long eps = 4295ull;  // 2e-6 in 2^-31 units
        unsigned long long lo = s_am, hi = s_ahi, lo_a = 0ull, hi_a = 0ull;
        int da = -1, ds = -1;
        for (int d = 255; d >= 0; --d) {
          const unsigned long long lo0 = lo, hi0 = hi;
          lo += s_msum[d];
          hi += (unsigned long long)s_msum[d] + hist[d];
          if (da < 0 && hi + eps >= target) {
            da = d;
            lo_a = lo0;
            hi_a = hi0;
          }
          if (lo >= target + eps) {
            ds = d;
            break;
          }
        }
        unsigned cnt = 0u;
        for (int d = ds; d >= 0 && d <= da; ++d) cnt += hist[d];
        const unsigned long long base = (unsigned long long)prefix;
        if (ds < 0) s_state = 2;  // top_p + margin not reached (top_p ~ 1): fall back
        else if (cnt <= (unsigned)kCandCap) {
          s_state = 1;
          s_L = base | ((unsigned long long)ds << shift);
          s_U = base + ((unsigned long long)(da + 1) << shift);
        } else if (ds == da && shift > 0) {  // one uncertain digit: refine inside it
          s_am = lo_a;
          s_ahi = hi_a;
          s_prefix = prefix | ((K)ds << shift);
          s_mask = mask | ((K)255u << shift);
        } else s_state = 2;  // more than kCandCap keys in the uncertain band
      }
      __syncthreads();
      if (s_state) break;
    }
    if (s_state == 1) {
      const unsigned long long L = s_L, U = s_U;
      const double itot = 1.0 / tot;
      double cu = 0.0;  // exact mass of the keys >= U (all inside the nucleus), fixed-order sum
      for (int v0 = tid * 8; v0 < V; v0 += NT * 8) {
        uint32_t kk[8];
        load8(x, v0, V, vec, kk);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (v0 + j >= V) continue;
          if (kk[j] >= U) {
            cu += (double)ex2(fmaf(KO::value((K)kk[j]), c2, nm)) * itot;  // MUFU terms (~1e-7)
          } else if (kk[j] >= L) {
            const int slot = atomicAdd(&s_ncand, 1);
            s_cand[slot] = ((unsigned long long)kk[j] << 32) | (0xFFFFFFFFu - (uint32_t)(v0 + j));
          }
        }
      }
      cu = warp_sum_d(cu);
      if (lane == 0) s_lsum[wid] = cu;
      __syncthreads();
      if (tid == 0) {
        double t = 0.0;
        for (int w = 0; w < NT / 32; ++w) t += s_lsum[w];
        s_cu = t;
      }
      const int nc = s_ncand;
      int np2 = 1;
      while (np2 < nc) np2 <<= 1;
      for (int j = nc + tid; j < np2; j += NT) s_cand[j] = 0ull;
      __syncthreads();
      for (int size = 2; size <= np2; size <<= 1) {  // bitonic sort, descending composite
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
          for (int j = tid; j < np2; j += NT) {
            const int o = j ^ stride;
            if (o > j) {
              const bool down = (j & size) == 0;
              const unsigned long long u = s_cand[j], v = s_cand[o];
              if ((u < v) == down) {
                s_cand[j] = v;
                s_cand[o] = u;
              }
            }
          }
          __syncthreads();
        }
      }
      for (int j = tid; j < nc; j += NT) {
        double pj = exp((double)KO::value((K)(s_cand[j] >> 32)) / tau - y0);
        s_pm[j] = pj / tot;
      }
      __syncthreads();
      if (tid == 0) {
        double c = s_cu;
        int n = -1;
        for (int j = 0; j < nc; ++j) {
          c += s_pm[j];
          if (c >= (double)a.top_p) {
            n = j;
            break;
          }
        }
        if (n < 0) s_state = 2;  // rounding: the bound was not conservative enough
        else {
          out->th_key = (uint32_t)(s_cand[n] >> 32);
          out->th_idx = (int)(0xFFFFFFFFu - (uint32_t)s_cand[n]);
          out->s = c;
        }
      }
      __syncthreads();
      if (s_state == 1) return;
    }
  }
  // ---- fallback (nuclei of more than kCandCap tokens, top_p ~ 1): mass-weighted radix select
  // of the cut key theta on the order-preserving key, 8 bits per pass from the top: per digit the
  // mass sum exp(y_v - y0) / tot of the keys under the current prefix, in 2^-60 fixed point
  // (integer shared atomics: order-independent, exact bin sums, deterministic), into 8
  // privatised histograms in the (now free) candidate buffer.  The cut digit is the first, from
  // the top, whose cumulative mass reaches top_p.
  {
    constexpr double kFix = 1152921504606846976.0;  // 2^60
    unsigned long long *wm = s_cand;
    __shared__ unsigned long long s_cab;
    __shared__ int s_all, s_m;
    __shared__ double s_s;
    const double y0 = s_y0, tot = s_lfull;
    const unsigned long long tp_fix = (unsigned long long)((double)a.top_p * kFix);
    // per-element mass with the normaliser's own fp32 terms: 2^{(x - x_max) log2e / tau} / tot
    const float c2 = (float)(1.4426950408889634 / tau), nm = -KO::value(c_key[0]) * c2;
    const float scale = (float)(kFix / tot);
    const bool vec = (reinterpret_cast<uintptr_t>(x) & 15) == 0;
    if (tid == 0) {
      s_prefix = 0;
      s_mask = 0;
      s_cab = 0ull;
      s_all = 0;
      s_ntie = 0;
    }
    for (int shift = KO::kBits - 8; shift >= 0; shift -= 8) {
      for (int j = tid; j < kCandCap; j += NT) wm[j] = 0ull;
      __syncthreads();
      const K prefix = s_prefix, mask = s_mask;
      unsigned long long *mine = wm + (wid & 7) * 256;
      for (int v0 = tid * 8; v0 < V; v0 += NT * 8) {
        uint32_t kk[8];
        load8(x, v0, V, vec, kk);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (v0 + j < V && (kk[j] & mask) == prefix) {
            const unsigned long long mf = __float2ull_rz(ex2(fmaf(KO::value(kk[j]), c2, nm)) * scale);
            if (mf) atomicAdd(mine + ((kk[j] >> shift) & 255u), mf);
          }
        }
      }
      __syncthreads();
      if (tid < 256) {
        unsigned long long t = 0ull;
#pragma unroll
        for (int c = 0; c < 8; ++c) t += wm[c * 256 + tid];
        wm[tid] = t;
      }
      __syncthreads();
      if (tid == 0) {
        unsigned long long c = s_cab;
        int d = 255;
        for (; d >= 0; --d) {
          if (c + wm[d] >= tp_fix) break;
          c += wm[d];
        }
        if (d < 0) s_all = 1;  // the whole distribution rounds below top_p: keep every token
        s_cab = c;
        s_prefix = prefix | ((K)(d < 0 ? 0 : d) << shift);
        s_mask = mask | ((K)255u << shift);
      }
      __syncthreads();
      if (s_all) break;
    }
    if (s_all) {
      if (tid == 0) {
        out->th_key = 0u;
        out->th_idx = INT32_MAX;
        out->s = (double)s_cab / kFix;
      }
      return;
    }
    const K theta = s_prefix;
    for (int e = tid; e < V; e += NT)
      if (KO::key(x, e) == theta) {
        const int slot = atomicAdd(&s_ntie, 1);
        if (slot < kTieCap) s_tie[slot] = e;
      }
    __syncthreads();
    const int ntie = s_ntie;
    if (tid == 0) {  // the oracle's sequential cumulative over the tie group (index order)
      const double pth = exp((double)KO::value(theta) / tau - y0) / tot;
      double c = (double)s_cab / kFix;
      int m = 0;
      while (m < ntie) {
        c += pth;
        ++m;
        if (c >= (double)a.top_p) break;
      }
      s_m = m;
      s_s = c;
    }
    __syncthreads();
    const int m = s_m;
    if (ntie <= kTieCap) {  // bitonic sort of the tie indices; the m-th smallest closes the nucleus
      int np2 = 1;
      while (np2 < ntie) np2 <<= 1;
      for (int j = ntie + tid; j < np2; j += NT) s_tie[j] = INT32_MAX;
      __syncthreads();
      for (int size = 2; size <= np2; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
          for (int j = tid; j < np2; j += NT) {
            const int o = j ^ stride;
            if (o > j) {
              const bool up = (j & size) == 0;
              const int u = s_tie[j], v = s_tie[o];
              if ((u > v) == up) {
                s_tie[j] = v;
                s_tie[o] = u;
              }
            }
          }
          __syncthreads();
        }
      }
      if (tid == 0) out->th_idx = s_tie[m - 1];
    } else if (wid == 0) {  // pathological tie counts: one ordered pass (vocabulary order)
      int taken = 0;
      for (int e0 = 0; e0 < V && taken < m; e0 += 32) {
        const int e = e0 + lane;
        const bool eq = e < V && KO::key(x, e) == theta;
        const unsigned msk = __ballot_sync(0xffffffffu, eq);
        const int rank = taken + __popc(msk & ((1u << lane) - 1u));
        if (eq && rank == m - 1) out->th_idx = e;
        taken += __popc(msk);
      }
    }
    if (tid == 0) {
      out->th_key = (uint32_t)theta;
      out->s = s_s;
    }
  }
}

// threshold form of a row (every FList carries it, see sv_internal.h)
struct Thr {
  uint32_t key;
  int32_t idx;
  double tau, y0, tot, s;
};
__device__ __forceinline__ Thr load_thr(const FList *L) { return Thr{L->th_key, L->th_idx, L->tau, L->y0, L->tot, L->s}; }

// p'(v) of a row in threshold form: the kept set and the same fp64 operations as the list entries
// (exp(y - y0), / tot, / s), so list values are reproduced bit for bit
template <typename T>
__device__ __forceinline__ double thr_pk(uint32_t kk, int v, const Thr &L) {
  using KO = KeyOf<T>;
  if (kk < L.key || (kk == L.key && v > L.idx)) return 0.0;
  double p = exp((double)KO::value(kk) / L.tau - L.y0);
  p = p / L.tot;
  return p / L.s;
}
template <typename T>
__device__ __forceinline__ double thr_p(const T *x, int v, const Thr &L) {
  return thr_pk<T>(KeyOf<T>::key(x, v), v, L);
}

// bulk form for full-row passes: log p'(v) = x_v / tau - c with c = y0 + log(tot s) (no divisions;
// the same values up to rounding)
struct ThrF {
  uint32_t key;
  int32_t idx;
  double itau, c;
};
__device__ __forceinline__ ThrF make_thrf(const Thr &L) { return ThrF{L.key, L.idx, 1.0 / L.tau, L.y0 + log(L.tot * L.s)}; }
template <typename T>
__device__ __forceinline__ bool thr_kept(uint32_t kk, int v, const ThrF &L) {
  return kk > L.key || (kk == L.key && v <= L.idx);
}
template <typename T>
__device__ __forceinline__ double thr_logp(uint32_t kk, const ThrF &L) {
  return (double)KeyOf<T>::value(kk) * L.itau - L.c;
}

__device__ __forceinline__ double block_sum_d(double v, double *red) {  // fixed order: warps, then 0..nw-1
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum_d(v);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < nw; ++w) t += red[w];
  return t;
}

// p of vocabulary index v in a list (0 when absent); every lane returns the same value
__device__ __forceinline__ double list_p(const FList *L, int n, int v) {
  const int lane = threadIdx.x & 31;
  const bool hit = lane < n && L->idx[lane] == v;
  const unsigned m = __ballot_sync(0xffffffffu, hit);
  const double mine = hit ? L->p[lane] : 0.0;
  return m ? __shfl_sync(0xffffffffu, mine, __ffs(m) - 1) : 0.0;
}

// the score outputs of row r (lane / thread 0 of the row's owner)
__device__ __forceinline__ void write_fscore(const FilterArgs &a, int64_t r, int st, double S, double A, double KL,
                                             double pdt) {
  const float nanf_ = __int_as_float(0x7fc00000);
  float phat = 0.f;
  if (!st && a.p_hat) {  // bin = number of interior edges strictly below the value (R9)
    const float Sf = (float)S, Af = (float)A;
    int si = 0, ai = 0;
    for (int j = 1; j < a.n_s; ++j) si += a.s_edges[j] < Sf;
    for (int j = 1; j < a.n_a; ++j) ai += a.a_edges[j] < Af;
    phat = a.cells[si * a.n_a + ai];
  }
  if (a.S) a.S[r] = st ? nanf_ : (float)S;
  if (a.A) a.A[r] = st ? nanf_ : (float)A;
  if (a.KL) a.KL[r] = st ? nanf_ : (float)KL;
  if (a.p_hat) a.p_hat[r] = phat;
  if (a.dpt) a.dpt[r] = (st & ~8) ? nanf_ : (float)pdt;
  if (a.status) a.status[r] = st;
}

__global__ void __launch_bounds__(256) sv_fscore_kernel(const __grid_constant__ FilterArgs a) {
  pdl_wait();
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (r >= (int64_t)a.B * a.k) return;
  const FList *Ld = a.dl + r, *Lc = a.cl + r;
  if (Ld->wide || Lc->wide) return;  // sv_fwide_score_kernel
  const int nd = Ld->n, nc = Lc->n;
  int st = Ld->st | Lc->st;
  const int t = a.tok[r];
  if (t < 0 || t >= a.V) st |= 4; /*SV_ROW_BAD_TOKEN*/
  // S over the draft list (sorted order, sequential fp64), KL, p(t)
  const int vd = lane < nd ? Ld->idx[lane] : -1;
  const double pd = lane < nd ? Ld->p[lane] : 0.0;
  double pcv = 0.0;
  for (int l = 0; l < nc; ++l) {  // companion p at this lane's draft index
    const int ci = Lc->idx[l];
    if (ci == vd) pcv = Lc->p[l];
  }
  const double mn = fmin(pd, pcv);
  const double klt = pd > 0.0 ? (pcv > 0.0 ? pd * log(pd / pcv) : INFINITY) : 0.0;
  double S = 0.0, KL = 0.0;
  for (int l = 0; l < nd; ++l) {
    S += __shfl_sync(0xffffffffu, mn, l);
    KL += __shfl_sync(0xffffffffu, klt, l);
  }
  const double pdt = (st & 4) ? 0.0 : list_p(Ld, nd, t), pct = (st & 4) ? 0.0 : list_p(Lc, nc, t);
  if (!st && pdt == 0.0) st |= 8; /*SV_ROW_DRAFT_ZERO*/
  const double A = st ? 0.0 : fmin(1.0, pct / pdt);
  if (lane == 0) write_fscore(a, r, st, S, A, KL, pdt);
}

// KF2w: rows where the draft or the companion nucleus exceeds 32 tokens -- one cluster of
// kWideSplit CTAs per (b, i), CTA y streams the vocabulary slice y of both rows in threshold form
// (S = sum min(p'_d, p'_c), KL over p'_d > 0); the slices' sums meet in rank 0 over DSMEM and are
// added in slice order.  (One CTA per row took ~67 us for the few wide rows of a launch.)
constexpr int kWideSplit = 8;
template <typename T>
__global__ void __launch_bounds__(256) sv_fwide_score_kernel(const __grid_constant__ FilterArgs a) {
  pdl_wait();  // (no early launch_dependents: a cluster grid, see K1c in sv_score.cu)
  __shared__ double red[16];
  __shared__ double part[2];
  cg::cluster_group cl = cg::this_cluster();
  const int64_t r = blockIdx.x / kWideSplit;
  const int y = (int)(blockIdx.x % kWideSplit);
  const FList *Ld = a.dl + r, *Lc = a.cl + r;
  if (!Ld->wide && !Lc->wide) return;  // the whole cluster (same row) leaves
  const int64_t b = r / a.k, i = r % a.k;
  const T *xd = reinterpret_cast<const T *>(a.d) + b * a.d_sb + i * a.d_si;
  const T *xc = reinterpret_cast<const T *>(a.c) + b * a.c_sb + i * a.c_si;
  const Thr ld = load_thr(Ld), lc = load_thr(Lc);
  int st = Ld->st | Lc->st;
  const int t = a.tok[r];
  if (t < 0 || t >= a.V) st |= 4;
  double S = 0.0, KL = 0.0;
  const bool vec = ((reinterpret_cast<uintptr_t>(xd) | reinterpret_cast<uintptr_t>(xc)) & 15) == 0;
  // slice y: [vb, ve), boundaries multiples of 8
  const int vb = (int)(((int64_t)a.V * y / kWideSplit) & ~7ll);
  const int ve = y + 1 == kWideSplit ? a.V : (int)(((int64_t)a.V * (y + 1) / kWideSplit) & ~7ll);
  // per kept draft entry: log p' in fp64 (x / tau - c), p' = 2^{log p' log2 e} on the fp32 MUFU
  // (relative error ~1e-6, inside the north_star tolerance), KL term p'_d (log p'_d - log p'_c)
  const ThrF fd = make_thrf(ld), fc = make_thrf(lc);
  if (!st)
    for (int v0 = vb + threadIdx.x * 8; v0 < ve; v0 += blockDim.x * 8) {
      uint32_t kd[8], kc[8];
      load8(xd, v0, a.V, vec, kd);
      load8(xc, v0, a.V, vec, kc);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (v0 + j >= ve || !thr_kept<T>(kd[j], v0 + j, fd)) continue;
        const double lpd = thr_logp<T>(kd[j], fd);
        const double pd = (double)ex2((float)(lpd * 1.4426950408889634));
        if (pd > 0.0) {
          if (thr_kept<T>(kc[j], v0 + j, fc)) {
            const double lpc = thr_logp<T>(kc[j], fc);
            const double pc = (double)ex2((float)(lpc * 1.4426950408889634));
            S += fmin(pd, pc);
            KL += pd * (lpd - lpc);
          } else
            KL = INFINITY;
        }
      }
    }
  S = block_sum_d(S, red);
  KL = block_sum_d(KL, red);
  if (threadIdx.x == 0) {
    part[0] = S;
    part[1] = KL;
  }
  cl.sync();  // every slice's sums are in its shared memory
  if (y == 0 && threadIdx.x == 0) {
    S = 0.0;
    KL = 0.0;
    for (int q = 0; q < kWideSplit; ++q) {  // slice order
      const double *pq = cl.map_shared_rank(part, (unsigned)q);
      S += pq[0];
      KL += pq[1];
    }
  }
  cl.sync();  // (no CTA leaves while rank 0 reads its shared memory)
  if (y != 0 || threadIdx.x != 0) return;
  const double pdt = (st & 4) ? 0.0 : thr_p(xd, t, ld), pct = (st & 4) ? 0.0 : thr_p(xc, t, lc);
  if (!st && pdt == 0.0) st |= 8;
  const double A = st ? 0.0 : fmin(1.0, pct / pdt);
  write_fscore(a, r, st, S, A, KL, pdt);
}

template <typename T>
cudaError_t launch_fwide_score(const FilterArgs &a, unsigned rows, cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(rows * kWideSplit);
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  at[1].id = cudaLaunchAttributeClusterDimension;
  at[1].val.clusterDim.x = kWideSplit;
  at[1].val.clusterDim.y = 1;
  at[1].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, sv_fwide_score_kernel<T>, a);
}

constexpr int kPendingWide = -2;  // out_tok marker: the residual / bonus sample needs a full-row pass

template <typename T>
__global__ void __launch_bounds__(32 * 16) sv_fverify_kernel(const __grid_constant__ FilterArgs a) {
  pdl_wait();
  pdl_trigger();
  // one CTA of k warps per sequence: warp i evaluates draft position i's accept test (its list
  // lookups are warp-cooperative), warp 0 then takes the first rejection / error in position order
  // -- the same decisions as a sequential walk -- and draws the token
  __shared__ double s_ratio[16];
  __shared__ int s_rst[16], s_rej[16];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, k = a.k;
  const int64_t b = blockIdx.x;
  const int g = a.gamma[b];
  int st = (g < 0 || g > k) ? 64 /*BAD_GAMMA*/ : 0;
  const int gg = st ? -1 : g;
  const uint64_t off = a.offset;
  if (wid < gg) {
    const int i = wid;
    const int64_t rd = b * k + i, rt = b * (k + 1) + i;
    const FList *Ldr = a.dl + rd, *Ltr = a.tl + rt;
    const int t = a.tok[rd];
    int rst = Ldr->st | Ltr->st;
    if (t < 0 || t >= a.V) rst |= 4;
    if (Ldr->wide && !a.d) rst |= 256; /*SV_ROW_FILTER_UNSUPPORTED: wide draft row, no draft logits*/
    double pdt = 0.0, ptt = 0.0;
    if (!(rst & (4 | 256))) {
      pdt = Ldr->wide ? thr_p(reinterpret_cast<const T *>(a.d) + b * a.d_sb + i * a.d_si, t, load_thr(Ldr))
                      : list_p(Ldr, Ldr->n, t);
      ptt = Ltr->wide ? thr_p(reinterpret_cast<const T *>(a.t) + b * a.t_sb + i * a.t_si, t, load_thr(Ltr))
                      : list_p(Ltr, Ltr->n, t);
    }
    if (!rst && pdt == 0.0) rst |= 8;
    const double ratio = rst ? 0.0 : ptt / pdt;
    const uint4 w = sv_philox(a.seed, off, a.seq_base + b, i);
    if (lane == 0) {
      s_rst[i] = rst;
      s_ratio[i] = ratio;
      s_rej[i] = !rst && !(u24(w.x) < ratio);
    }
  }
  __syncthreads();
  if (wid != 0) return;
  // the walk in position order: an error stops it (its bits), else the first rejection sets N
  double ratio_mine = 0.0;
  int N = st ? 0 : gg;
  for (int i = 0; i < gg; ++i) {
    if (s_rst[i]) {
      st |= s_rst[i];
      break;
    }
    if (lane == i) ratio_mine = s_ratio[i];
    if (s_rej[i]) {
      N = i;
      break;
    }
  }
  if (a.ratio && lane < k) a.ratio[b * k + lane] = (!st && lane < N + (N < gg ? 1 : 0)) ? (float)fmin(1.0, ratio_mine)
                                                                                          : __int_as_float(0x7fc00000);
  const int64_t rt = b * (k + 1) + (st ? 0 : N);
  const FList *Lt = a.tl + rt;
  const FList *LdN = (!st && N < gg) ? a.dl + b * k + N : nullptr;
  if (!st && LdN && LdN->wide && !a.d) st |= 256;
  if (st) {
    if (lane == 0) {
      a.n_accept[b] = 0;
      a.out_tok[b] = -1;
      if (a.resid) a.resid[b] = __int_as_float(0x7fc00000);
      if (a.status) a.status[b] = st;
    }
    return;
  }
  if (Lt->st) st |= Lt->st;
  if (Lt->wide || (LdN && LdN->wide)) {  // sv_fwide_sample_kernel draws the token
    if (lane == 0) {
      a.n_accept[b] = N;
      a.out_tok[b] = kPendingWide;
      if (a.status) a.status[b] = st;
    }
    return;
  }
  // residual (N < gamma) or bonus (N == gamma) over the target list of row N
  const int nt = Lt->n;
  const int vi = lane < nt ? Lt->idx[lane] : INT32_MAX;
  double r = lane < nt ? Lt->p[lane] : 0.0;
  if (LdN) {
    double pdv = 0.0;
    for (int l = 0; l < LdN->n; ++l)
      if (LdN->idx[l] == vi) pdv = LdN->p[l];
    r = fmax(0.0, r - pdv);
  }
  // entries in vocabulary order (rank by index), then sequential Z and inverse CDF (R11)
  int rank = 0;
  for (int l = 0; l < nt; ++l) rank += __shfl_sync(0xffffffffu, vi, l) < vi;
  __shared__ double s_r[8][32], s_pt[8][32];
  __shared__ int s_v[8][32];
  const int w8 = 0;  // warp 0 of the sequence's CTA
  if (lane < nt) {
    s_r[w8][rank] = r;
    s_pt[w8][rank] = Lt->p[lane];
    s_v[w8][rank] = vi;
  }
  __syncwarp();
  if (lane == 0) {
    double Z = 0.0;
    for (int l = 0; l < nt; ++l) Z += s_r[w8][l];
    if (LdN && !(Z > 0.0)) {  // R10: a zero residual (rounding only) samples p_t of row N instead
      st |= 32;               /*SV_ROW_RESID_ZERO*/
      Z = 0.0;
      for (int l = 0; l < nt; ++l) {
        s_r[w8][l] = s_pt[w8][l];
        Z += s_r[w8][l];
      }
    }
    const double us = u24(sv_philox(a.seed, off, a.seq_base + b, N).y);
    const double th = us * Z;
    double cum = 0.0;
    int tok = -1, lastp = -1;
    for (int l = 0; l < nt; ++l) {
      if (!(s_r[w8][l] > 0.0)) continue;
      lastp = s_v[w8][l];
      cum += s_r[w8][l];
      if (cum > th) {
        tok = s_v[w8][l];
        break;
      }
    }
    if (tok < 0) tok = lastp;
    a.n_accept[b] = N;
    a.out_tok[b] = tok;
    if (a.resid) a.resid[b] = (float)Z;
    if (a.status) a.status[b] = st;
  }
}

// KF3w: the residual max(0, p'_t - p'_d) (or the bonus p'_t) of sequences whose row N has a
// nucleus wider than 32 tokens -- one CTA per sequence, full-row pass in threshold form: every
// thread sums a contiguous vocabulary chunk (fp64, sequential), a fixed-order prefix over the
// chunks gives Z and the chunk holding the crossing of u_s Z, which is rescanned (R11)
template <typename T>
__global__ void __launch_bounds__(512) sv_fwide_sample_kernel(const __grid_constant__ FilterArgs a) {
  pdl_wait();
  pdl_trigger();
  constexpr int NT = 512;
  __shared__ double s_sum[NT], s_pre[NT];
  __shared__ int s_last[NT];
  __shared__ int s_j;
  __shared__ double s_Z, s_th;
  const int64_t b = blockIdx.x;
  if (a.out_tok[b] != kPendingWide) return;
  const int tid = threadIdx.x, lane = tid & 31, k = a.k, V = a.V;
  const int N = a.n_accept[b], g = a.gamma[b];
  const Thr lt = load_thr(a.tl + b * (k + 1) + N);
  const T *xt = reinterpret_cast<const T *>(a.t) + b * a.t_sb + (int64_t)N * a.t_si;
  bool resid = N < g;
  const FList *LdN = a.dl + b * k + N;
  const bool dwide = resid && LdN->wide;  // else the <= 32 draft entries, walked in index order
  const Thr ld = dwide ? load_thr(LdN) : lt;
  const T *xd = dwide ? reinterpret_cast<const T *>(a.d) + b * a.d_sb + (int64_t)N * a.d_si : xt;
  __shared__ int s_di[32];
  __shared__ double s_dp[32];
  const int nd = (resid && !dwide) ? LdN->n : 0;
  if (tid < nd) {
    const int vi = LdN->idx[tid];
    int rank = 0;
    for (int l = 0; l < nd; ++l) rank += LdN->idx[l] < vi;
    s_di[rank] = vi;
    s_dp[rank] = LdN->p[tid];
  }
  __syncthreads();
  // contiguous chunks of a multiple of 8 elements (vector loads of 8 keys)
  const int chunk = (((V + NT - 1) / NT) + 7) & ~7, v0 = min(V, tid * chunk), v1 = min(V, v0 + chunk);
  const bool vec = ((reinterpret_cast<uintptr_t>(xt) | reinterpret_cast<uintptr_t>(xd)) & 15) == 0;
  int q = 0;  // first draft entry with index >= v (list-mode draft rows; v ascends within a pass)
  const ThrF ft = make_thrf(lt), fd = make_thrf(ld);
  auto rv = [&](int v, uint32_t kt, uint32_t kd) {
    const double pt = thr_kept<T>(kt, v, ft) ? exp(thr_logp<T>(kt, ft)) : 0.0;
    if (!resid || !(pt > 0.0)) return pt;
    if (dwide) return fmax(0.0, pt - (thr_kept<T>(kd, v, fd) ? exp(thr_logp<T>(kd, fd)) : 0.0));
    while (q < nd && s_di[q] < v) ++q;
    return fmax(0.0, pt - ((q < nd && s_di[q] == v) ? s_dp[q] : 0.0));
  };
  __shared__ int s_retry;
  double sum;
  int lastp;
pass_again:  // R10: when the residual mass is 0 (rounding only), the pass is redone over p_t
  sum = 0.0;
  lastp = -1;
  q = 0;
  for (int w0 = v0; w0 < v1; w0 += 8) {
    uint32_t kt[8], kd[8];
    load8(xt, w0, V, vec, kt);
    if (dwide) load8(xd, w0, V, vec, kd);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (w0 + j >= v1) break;
      const double r = rv(w0 + j, kt[j], dwide ? kd[j] : 0u);
      if (r > 0.0) {
        sum += r;
        lastp = w0 + j;
      }
    }
  }
  s_sum[tid] = sum;
  s_last[tid] = lastp;
  __syncthreads();
  if (tid < 32) {  // warp 0: prefix over the chunks (lane l: chunks 16 l .. 16 l + 15 in order)
    constexpr int PER = NT / 32;
    double ls = 0.0;
#pragma unroll
    for (int j = 0; j < PER; ++j) ls += s_sum[lane * PER + j];
    const double incl = warp_incl_scan_d(ls, lane);
    double p = __shfl_up_sync(0xffffffffu, incl, 1);
    if (lane == 0) p = 0.0;
    const double c = __shfl_sync(0xffffffffu, incl, 31);
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      s_pre[lane * PER + j] = p;
      p += s_sum[lane * PER + j];
    }
    const double us = u24(sv_philox(a.seed, a.offset, a.seq_base + b, N).y);
    const double th = us * c;
    int myj = -1;
    for (int j = 0; j < PER; ++j) {
      const int idx = lane * PER + j;
      if (s_sum[idx] > 0.0 && s_pre[idx] + s_sum[idx] > th) {
        myj = idx;
        break;
      }
    }
    const unsigned m = __ballot_sync(0xffffffffu, myj >= 0);
    const int jc = m ? __shfl_sync(0xffffffffu, myj, __ffs(m) - 1) : -1;
    if (lane == 0) {
      s_retry = resid && !(c > 0.0);
      s_j = jc;
      s_Z = c;
      s_th = th;
    }
  }
  __syncthreads();
  if (s_retry) {
    resid = false;
    if (tid == 0 && a.status) a.status[b] |= 32;  // SV_ROW_RESID_ZERO
    __syncthreads();
    goto pass_again;
  }
  const int jc = s_j;
  if (jc < 0) {  // rounding left no crossing (or Z = 0): the last positive entry (R11 fallback)
    if (tid == 0) {
      int tok = -1;
      for (int j = NT - 1; j >= 0 && tok < 0; --j) tok = s_last[j];
      const double Z = s_Z;
      a.out_tok[b] = tok;
      if (a.resid) a.resid[b] = (float)Z;
      if (a.status && !(Z > 0.0)) a.status[b] |= 32;
    }
    return;
  }
  if (tid >= 32) return;
  // warp 0 rescans chunk jc: lane l takes a contiguous sub-range (multiple of 8 elements), sums
  // it sequentially in fp64; a fixed-order warp scan finds the crossing lane, which walks its
  // sub-range from its prefix (R11); if rounding leaves no crossing, the last positive element
  const double th = s_th;
  const int c0 = min(V, jc * chunk), c1 = min(V, c0 + chunk);
  const int per = ((((c1 - c0) + 31) / 32) + 7) & ~7;
  const int l0 = min(c1, c0 + lane * per), l1 = min(c1, l0 + per);
  double ls = 0.0;
  int llast = -1;
  q = 0;
  for (int w0 = l0; w0 < l1; w0 += 8) {
    uint32_t kt[8], kd[8];
    load8(xt, w0, V, vec, kt);
    if (dwide) load8(xd, w0, V, vec, kd);
    for (int j = 0; j < 8 && w0 + j < l1; ++j) {
      const double r = rv(w0 + j, kt[j], dwide ? kd[j] : 0u);
      if (r > 0.0) {
        ls += r;
        llast = w0 + j;
      }
    }
  }
  const double incl = warp_incl_scan_d(ls, lane);
  double excl = __shfl_up_sync(0xffffffffu, incl, 1);
  if (lane == 0) excl = 0.0;
  const double base = s_pre[jc];
  const unsigned cross = __ballot_sync(0xffffffffu, ls > 0.0 && base + incl > th);
  int tok = s_last[jc];
  if (cross) {
    const int lc = __ffs(cross) - 1;
    if (lane == lc) {
      double cum = base + excl;
      bool found = false;
      q = 0;
      for (int w0 = l0; w0 < l1 && !found; w0 += 8) {
        uint32_t kt[8], kd[8];
        load8(xt, w0, V, vec, kt);
        if (dwide) load8(xd, w0, V, vec, kd);
        for (int j = 0; j < 8 && w0 + j < l1; ++j) {
          const double r = rv(w0 + j, kt[j], dwide ? kd[j] : 0u);
          if (!(r > 0.0)) continue;
          cum += r;
          if (cum > th) {
            tok = w0 + j;
            found = true;
            break;
          }
        }
      }
      if (!found) tok = llast;
    }
    tok = __shfl_sync(0xffffffffu, tok, lc);
  }
  if (lane != 0) return;
  a.out_tok[b] = tok;
  if (a.resid) a.resid[b] = (float)s_Z;
}

cudaError_t launch_topk(const FilterArgs &a, dim3 grid, int which0, cudaStream_t st) {
  const dim3 blk(kTopKThreads);
  if (a.top_k == 0)
    return a.bf16 ? launch_k(sv_topk_kernel<__nv_bfloat16, true>, grid, blk, 0, st, a, which0)
                  : launch_k(sv_topk_kernel<float, true>, grid, blk, 0, st, a, which0);
  return a.bf16 ? launch_k(sv_topk_kernel<__nv_bfloat16, false>, grid, blk, 0, st, a, which0)
                : launch_k(sv_topk_kernel<float, false>, grid, blk, 0, st, a, which0);
}

}  // namespace

cudaError_t launch_filter_score(const FilterArgs &a, cudaStream_t st) {
  const unsigned rows = (unsigned)((int64_t)a.B * a.k);
  cudaError_t e = launch_topk(a, dim3(rows, 2), 0, st);
  if (e != cudaSuccess) return e;
  e = launch_k(sv_fscore_kernel, dim3((rows + 7) / 8), dim3(256), 0, st, a);
  if (e != cudaSuccess || a.top_k != 0) return e;  // wide rows exist only without top_k
  return a.bf16 ? launch_fwide_score<__nv_bfloat16>(a, rows, st) : launch_fwide_score<float>(a, rows, st);
}

cudaError_t launch_filter_verify(const FilterArgs &a, cudaStream_t st) {
  const unsigned rows = (unsigned)((int64_t)a.B * (a.k + 1));
  cudaError_t e = launch_topk(a, dim3(rows), 2, st);
  if (e != cudaSuccess) return e;
  const dim3 gv((unsigned)((a.B + 7) / 8));
  const dim3 gq((unsigned)a.B), bq(32 * (a.k > 0 ? a.k : 1));  // one CTA of k warps per sequence
  e = a.bf16 ? launch_k(sv_fverify_kernel<__nv_bfloat16>, gq, bq, 0, st, a)
             : launch_k(sv_fverify_kernel<float>, gq, bq, 0, st, a);
  if (e != cudaSuccess || a.top_k != 0) return e;
  return a.bf16 ? launch_k(sv_fwide_sample_kernel<__nv_bfloat16>, dim3((unsigned)a.B), dim3(512), 0, st, a)
                : launch_k(sv_fwide_sample_kernel<float>, dim3((unsigned)a.B), dim3(512), 0, st, a);
}

}  // namespace sv
