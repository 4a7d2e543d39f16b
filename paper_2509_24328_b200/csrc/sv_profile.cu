// sv_profile.cu -- NEXT-4: the offline (S, A) -> acceptance profile and its information-gain
// report, on the GPU (P L176: "perform a profiling run ... compute the average token
// acceptance probability for each bin combination" with adaptive binning; S L275-310; the
// Table 2 layout P L347-368).  Input: N records (S, A, X) as produced by sv_score (S, A) and
// sd_verify (X = accept_ratio = min(1, p_t(t)/p_d(t)), the true acceptance probability P L150).
//
//   K_sort   bitonic sort of S and A (padded to a power of two with +inf): shared-memory tiles
//            for the strides below 4096, one global pass per larger stride.
//   K_edges  equal-frequency edges (interior edge j = the ceil(j n / n_bins)-th order statistic,
//            first = min, last = max, duplicates collapsed: S L278, L281), one thread per axis.
//   K_bin    per record: right-closed bins (R9: index = #interior edges < value), integer counts
//            and fixed-point (2^32) sums of X per cell, joint (s, a, x) histogram for the report.
//            Integer atomics only: the result is deterministic.
//   K_final  cell means with the S L296 fallbacks pre-filled (empty cell -> S-row mean -> global
//            mean) and the plug-in entropies H(X), H(X|S), H(X|A), H(X|S,A), I(X; S,A) in bits
//            (X in x_bins equal-width bins on [0, 1], S L328), fp64 in a fixed order.
#include <float.h>

#include "sv_device.cuh"
#include "sv_internal.h"

namespace sv {

namespace {

// Sort: bitonic network over P = next power of two >= N (padding +inf), ascending, on both axes
// at once (blockIdx.y = 0: S, 1: A).  Tiles of kSortTile elements run every stage with a stride
// below the tile in shared memory; the larger strides are one global pass each.  Equal values are
// interchangeable for the order statistics, so no stability is needed.
constexpr int kSortThreads = 512;
constexpr int kSortTile = 4096;

__device__ __forceinline__ float *sort_buf(const ProfileArgs &a) { return blockIdx.y == 0 ? a.s_sorted : a.a_sorted; }

__global__ void __launch_bounds__(kSortThreads) sv_sort_load_kernel(const ProfileArgs a, int P) {
  pdl_wait();
  pdl_trigger();
  const float *x = blockIdx.y == 0 ? a.S : a.A;
  float *buf = sort_buf(a);
  for (int i = blockIdx.x * kSortThreads + threadIdx.x; i < P; i += gridDim.x * kSortThreads)
    buf[i] = i < a.N ? x[i] : __int_as_float(0x7f800000);
}

// stages (size, stride) with stride < kSortTile inside one shared-memory tile: from size = 2 up
// to size_hi when `full`, else only the strides below the tile of the single size `size_hi`
__global__ void __launch_bounds__(kSortThreads) sv_sort_tile_kernel(const ProfileArgs a, int size_hi, int full, int P) {
  __shared__ float t[kSortTile];
  pdl_wait();
  pdl_trigger();
  float *buf = sort_buf(a);
  const int n = min(kSortTile, P), base = blockIdx.x * n;
  for (int j = threadIdx.x; j < n; j += kSortThreads) t[j] = buf[base + j];
  __syncthreads();
  for (int size = full ? 2 : size_hi; size <= size_hi; size <<= 1) {
    for (int stride = min(size, n) >> 1; stride > 0; stride >>= 1) {
      for (int j = threadIdx.x; j < n; j += kSortThreads) {
        const int o = j ^ stride;
        if (o > j) {
          const bool up = ((base + j) & size) == 0;
          const float u = t[j], v = t[o];
          if ((u > v) == up) {
            t[j] = v;
            t[o] = u;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int j = threadIdx.x; j < n; j += kSortThreads) buf[base + j] = t[j];
}

__global__ void __launch_bounds__(kSortThreads) sv_sort_global_kernel(const ProfileArgs a, int size, int stride, int P) {
  pdl_wait();
  pdl_trigger();
  float *buf = sort_buf(a);
  for (int j = blockIdx.x * kSortThreads + threadIdx.x; j < P; j += gridDim.x * kSortThreads) {
    const int o = j ^ stride;
    if (o > j) {
      const bool up = (j & size) == 0;
      const float u = buf[j], v = buf[o];
      if ((u > v) == up) {
        buf[j] = v;
        buf[o] = u;
      }
    }
  }
}

// equal-frequency edges of one sorted axis with the duplicate collapse (matches
// oracle/profile.py adaptive_edges); returns the number of bins
__device__ int build_edges(const float *xs, int n, int n_bins, float *edges) {
  int ne = 0;
  edges[ne++] = xs[0];
  for (int j = 1; j < n_bins; ++j) {
    const int64_t r = ((int64_t)j * n + n_bins - 1) / n_bins;  // ceil(j n / n_bins)
    const float e = xs[r - 1];
    if (e > edges[ne - 1]) edges[ne++] = e;
  }
  if (xs[n - 1] > edges[ne - 1] || ne == 1) edges[ne++] = xs[n - 1];
  return ne - 1;
}

__global__ void sv_edges_kernel(const ProfileArgs a) {
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x == 0) *a.n_s = build_edges(a.s_sorted, a.N, a.n_s_bins, a.s_edges);
  if (threadIdx.x == 32) *a.n_a = build_edges(a.a_sorted, a.N, a.n_a_bins, a.a_edges);
}

__device__ __forceinline__ int bin_index(const float *edges, int nb, float v) {
  int idx = 0;  // number of interior edges strictly below v (R9), clamped
  for (int j = 1; j < nb; ++j) idx += edges[j] < v;
  return idx;
}

__global__ void __launch_bounds__(256) sv_bin_kernel(const ProfileArgs a) {
  __shared__ float se[kProfMaxBins + 1], ae[kProfMaxBins + 1];
  __shared__ int ns, na;
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x == 0) {
    ns = *a.n_s;
    na = *a.n_a;
  }
  __syncthreads();
  for (int j = threadIdx.x; j <= ns; j += blockDim.x) se[j] = a.s_edges[j];
  for (int j = threadIdx.x; j <= na; j += blockDim.x) ae[j] = a.a_edges[j];
  __syncthreads();
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < a.N; r += gridDim.x * blockDim.x) {
    const int si = bin_index(se, ns, a.S[r]), ai = bin_index(ae, na, a.A[r]);
    const double x = (double)a.X[r];
    int xb = (int)(x * a.x_bins);
    xb = xb < 0 ? 0 : (xb > a.x_bins - 1 ? a.x_bins - 1 : xb);
    const int cell = si * na + ai;
    atomicAdd(a.counts + cell, 1);
    atomicAdd(a.xsum + cell, (unsigned long long)llrint(x * 4294967296.0));  // fixed point 2^-32
    atomicAdd(a.joint + cell * a.x_bins + xb, 1);
  }
}

// one CTA: counts / joint histogram staged in shared memory, cell means with the fallbacks,
// then the entropy terms in parallel (one thread per S bin, A bin or cell) and their sums in a
// fixed order by thread 0 (deterministic)
constexpr int kFinalThreads = 256;
__global__ void __launch_bounds__(kFinalThreads) sv_prof_final_kernel(const ProfileArgs a, int joint_in_smem) {
  extern __shared__ __align__(16) uint8_t dyn[];  // [nc] u64 X sums, [nc] counts, [nc xb] joint
  __shared__ double term_s[kProfMaxBins], term_a[kProfMaxBins];
  __shared__ double term_c[kProfMaxBins * kProfMaxBins];
  __shared__ double hx, rmean[kProfMaxBins];
  pdl_wait();
  pdl_trigger();
  const int tid = threadIdx.x;
  const int ns = *a.n_s, na = *a.n_a, xb = a.x_bins, N = a.N, nc = ns * na;
  unsigned long long *sx = reinterpret_cast<unsigned long long *>(dyn);
  int *scnt = reinterpret_cast<int *>(sx + kProfMaxBins * kProfMaxBins);
  int *sj = joint_in_smem ? scnt + kProfMaxBins * kProfMaxBins : a.joint;
  for (int c = tid; c < nc; c += kFinalThreads) {
    sx[c] = a.xsum[c];
    scnt[c] = a.counts[c];
  }
  if (joint_in_smem)
    for (int j = tid; j < nc * xb; j += kFinalThreads) sj[j] = a.joint[j];
  __syncthreads();
  const double scale = 1.0 / 4294967296.0;
  // cell means with the S L296 fallbacks: integer sums (exact, any order), one thread per S row
  unsigned long long gsum = 0;
  for (int c = 0; c < nc; ++c) gsum += sx[c];
  const double gmean = (double)gsum * scale / (double)N;
  for (int i = tid; i < ns; i += kFinalThreads) {
    unsigned long long rs = 0;
    long long rn = 0;
    for (int j = 0; j < na; ++j) {
      rs += sx[i * na + j];
      rn += scnt[i * na + j];
    }
    rmean[i] = rn > 0 ? (double)rs * scale / (double)rn : gmean;
  }
  __syncthreads();
  for (int c = tid; c < nc; c += kFinalThreads)
    a.cells[c] = scnt[c] > 0 ? (double)sx[c] * scale / (double)scnt[c] : rmean[c / na];
  if (!a.info) return;
  auto ent = [&](auto count_of, int tot) {  // H over the x bins of one group, bits
    double h = 0.0;
    for (int x = 0; x < xb; ++x) {
      const int v = count_of(x);
      if (v > 0) {
        const double p = (double)v / (double)tot;
        h -= p * log2(p);
      }
    }
    return h;
  };
  for (int i = tid; i < ns; i += kFinalThreads) {  // S bin i: n_i / N * H(X | S = i)
    int tot = 0;
    for (int j = 0; j < na * xb; ++j) tot += sj[i * na * xb + j];
    term_s[i] = tot > 0 ? (double)tot / N * ent([&](int x) {
      int v = 0;
      for (int j = 0; j < na; ++j) v += sj[(i * na + j) * xb + x];
      return v;
    }, tot) : 0.0;
  }
  for (int j = tid; j < na; j += kFinalThreads) {  // A bin j
    int tot = 0;
    for (int i = 0; i < ns; ++i)
      for (int x = 0; x < xb; ++x) tot += sj[(i * na + j) * xb + x];
    term_a[j] = tot > 0 ? (double)tot / N * ent([&](int x) {
      int v = 0;
      for (int i = 0; i < ns; ++i) v += sj[(i * na + j) * xb + x];
      return v;
    }, tot) : 0.0;
  }
  for (int c = tid; c < nc; c += kFinalThreads) {  // cell c
    const int tot = scnt[c];
    term_c[c] = tot > 0 ? (double)tot / N * ent([&](int x) { return sj[c * xb + x]; }, tot) : 0.0;
  }
  if (tid == 0) {
    hx = ent([&](int x) {
      int v = 0;
      for (int c = 0; c < nc; ++c) v += sj[c * xb + x];
      return v;
    }, N);
  }
  __syncthreads();
  if (tid == 0) {
    double hs = 0.0, ha = 0.0, hsa = 0.0;
    for (int i = 0; i < ns; ++i) hs += term_s[i];
    for (int j = 0; j < na; ++j) ha += term_a[j];
    for (int c = 0; c < nc; ++c) hsa += term_c[c];
    a.info[0] = hx;
    a.info[1] = hs;
    a.info[2] = ha;
    a.info[3] = hsa;
    a.info[4] = hx - hsa;
  }
}

}  // namespace

cudaError_t launch_profile(const ProfileArgs &a, cudaStream_t st) {
  cudaError_t e;
  int P = 1;
  while (P < a.N) P <<= 1;
  const unsigned gblocks = (unsigned)((P + kSortThreads - 1) / kSortThreads < 512 ? (P + kSortThreads - 1) / kSortThreads : 512);
  if ((e = launch_k(sv_sort_load_kernel, dim3(gblocks, 2), dim3(kSortThreads), 0, st, a, P)) != cudaSuccess) return e;
  const int tile = P < kSortTile ? P : kSortTile;
  const dim3 tgrid((unsigned)(P / tile), 2);
  if ((e = launch_k(sv_sort_tile_kernel, tgrid, dim3(kSortThreads), 0, st, a, tile, 1, P)) != cudaSuccess) return e;
  for (int size = 2 * tile; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride >= tile; stride >>= 1)
      if ((e = launch_k(sv_sort_global_kernel, dim3(gblocks, 2), dim3(kSortThreads), 0, st, a, size, stride, P)) !=
          cudaSuccess)
        return e;
    if ((e = launch_k(sv_sort_tile_kernel, tgrid, dim3(kSortThreads), 0, st, a, size, 0, P)) != cudaSuccess) return e;
  }
  if ((e = launch_k(sv_edges_kernel, dim3(1), dim3(64), 0, st, a)) != cudaSuccess) return e;
  const int grid = (int)((a.N + 255) / 256 < 1184 ? (a.N + 255) / 256 : 1184);
  if ((e = launch_k(sv_bin_kernel, dim3((unsigned)grid), dim3(256), 0, st, a)) != cudaSuccess) return e;
  const size_t base = (size_t)kProfMaxBins * kProfMaxBins * 12;
  const size_t joint = (size_t)a.n_s_bins * a.n_a_bins * a.x_bins * 4;
  const int jsm = base + joint <= 160 * 1024;
  const size_t smem = base + (jsm ? joint : 0);
  if ((e = cudaFuncSetAttribute(sv_prof_final_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) !=
      cudaSuccess)
    return e;
  return launch_k(sv_prof_final_kernel, dim3(1), dim3(kFinalThreads), smem, st, a, jsm);
}

}  // namespace sv
