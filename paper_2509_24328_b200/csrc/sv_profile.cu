// sv_profile.cu -- NEXT-4: the offline (S, A) -> acceptance profile and its information-gain
// report, on the GPU (P L176: "perform a profiling run ... compute the average token
// acceptance probability for each bin combination" with adaptive binning; S L275-310; the
// Table 2 layout P L347-368).  Input: N records (S, A, X) as produced by sv_score (S, A) and
// sd_verify (X = accept_ratio = min(1, p_t(t)/p_d(t)), the true acceptance probability P L150).
//
//   K_rank   stable ranks by all-pairs comparison through shared-memory tiles (rank_i =
//            #{x_j < x_i} + #{j < i : x_j == x_i}, unique), then a scatter sorts S and A exactly.
//            O(N^2 / lanes): ~0.2-0.5 ms at N = 65536 -- an offline step, chosen for exactness
//            and determinism over a radix sort.
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

constexpr int kRankThreads = 256;
constexpr int kRankTile = 4096;

// blockIdx.y selects the array (0 = S, 1 = A)
__global__ void __launch_bounds__(kRankThreads) sv_rank_kernel(const ProfileArgs a) {
  __shared__ float tile[kRankTile];
  pdl_wait();
  pdl_trigger();
  const float *x = blockIdx.y == 0 ? a.S : a.A;
  float *sorted = blockIdx.y == 0 ? a.s_sorted : a.a_sorted;
  const int i = blockIdx.x * kRankThreads + threadIdx.x;
  const float xi = i < a.N ? x[i] : 0.f;
  int rank = 0;
  for (int t0 = 0; t0 < a.N; t0 += kRankTile) {
    const int n = min(kRankTile, a.N - t0);
    __syncthreads();
    for (int j = threadIdx.x; j < n; j += kRankThreads) tile[j] = x[t0 + j];
    __syncthreads();
    if (i < a.N) {
      const int jlim = i - t0;  // tile entries with global index < i
#pragma unroll 8
      for (int j = 0; j < n; ++j) {
        const float xj = tile[j];
        rank += (xj < xi) | ((xj == xi) & (j < jlim));
      }
    }
  }
  if (i < a.N) sorted[rank] = xi;
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

__device__ double entropy_bits(const int *c, int n, int stride, int total) {
  double h = 0.0;
  for (int j = 0; j < n; ++j) {
    const int v = c[j * stride];
    if (v > 0) {
      const double p = (double)v / (double)total;
      h -= p * log2(p);
    }
  }
  return h;
}

// one thread: cell means with fallbacks, then the entropies (small tables, fixed order)
__global__ void sv_prof_final_kernel(const ProfileArgs a) {
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const int ns = *a.n_s, na = *a.n_a, xb = a.x_bins, N = a.N;
  unsigned long long gsum = 0;
  for (int c = 0; c < ns * na; ++c) gsum += a.xsum[c];
  const double scale = 1.0 / 4294967296.0;
  const double gmean = (double)gsum * scale / (double)N;
  for (int i = 0; i < ns; ++i) {
    unsigned long long rs = 0;
    long long rn = 0;
    for (int j = 0; j < na; ++j) {
      rs += a.xsum[i * na + j];
      rn += a.counts[i * na + j];
    }
    const double rmean = rn > 0 ? (double)rs * scale / (double)rn : gmean;
    for (int j = 0; j < na; ++j) {
      const int c = a.counts[i * na + j];
      a.cells[i * na + j] = c > 0 ? (double)a.xsum[i * na + j] * scale / (double)c : rmean;
    }
  }
  if (!a.info) return;
  // H(X): marginal over x bins; conditionals as sum over keys (in key order) of
  // n_key / N * H(X | key)
  int *tmp = a.scratch;  // [x_bins]
  for (int x = 0; x < xb; ++x) tmp[x] = 0;
  for (int c = 0; c < ns * na; ++c)
    for (int x = 0; x < xb; ++x) tmp[x] += a.joint[c * xb + x];
  const double hx = entropy_bits(tmp, xb, 1, N);
  double hs = 0.0, ha = 0.0, hsa = 0.0;
  for (int i = 0; i < ns; ++i) {  // H(X | S)
    int tot = 0;
    for (int x = 0; x < xb; ++x) {
      tmp[x] = 0;
      for (int j = 0; j < na; ++j) tmp[x] += a.joint[(i * na + j) * xb + x];
      tot += tmp[x];
    }
    if (tot > 0) hs += (double)tot / N * entropy_bits(tmp, xb, 1, tot);
  }
  for (int j = 0; j < na; ++j) {  // H(X | A)
    int tot = 0;
    for (int x = 0; x < xb; ++x) {
      tmp[x] = 0;
      for (int i = 0; i < ns; ++i) tmp[x] += a.joint[(i * na + j) * xb + x];
      tot += tmp[x];
    }
    if (tot > 0) ha += (double)tot / N * entropy_bits(tmp, xb, 1, tot);
  }
  for (int c = 0; c < ns * na; ++c) {  // H(X | S, A)
    const int tot = a.counts[c];
    if (tot > 0) hsa += (double)tot / N * entropy_bits(a.joint + c * xb, xb, 1, tot);
  }
  a.info[0] = hx;
  a.info[1] = hs;
  a.info[2] = ha;
  a.info[3] = hsa;
  a.info[4] = hx - hsa;
}

}  // namespace

cudaError_t launch_profile(const ProfileArgs &a, cudaStream_t st) {
  cudaError_t e;
  if ((e = launch_k(sv_rank_kernel, dim3((unsigned)((a.N + kRankThreads - 1) / kRankThreads), 2), dim3(kRankThreads),
                    0, st, a)) != cudaSuccess)
    return e;
  if ((e = launch_k(sv_edges_kernel, dim3(1), dim3(64), 0, st, a)) != cudaSuccess) return e;
  const int grid = (int)((a.N + 255) / 256 < 1184 ? (a.N + 255) / 256 : 1184);
  if ((e = launch_k(sv_bin_kernel, dim3((unsigned)grid), dim3(256), 0, st, a)) != cudaSuccess) return e;
  return launch_k(sv_prof_final_kernel, dim3(1), dim3(32), 0, st, a);
}

}  // namespace sv
