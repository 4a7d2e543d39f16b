// sv_greedy.cu -- NEXT-1: the paper's batch-level greedy schedule (P L247-252; S L402-417).
//
// Greedy (paper): start from gamma_q = 0 for every query; repeatedly add the candidate
// token with the largest marginal gain in expected accepted tokens (query q's next token
// has gain P_{q, gamma_q + 1} = prod_{i <= gamma_q + 1} p_hat_{q,i}; ties -> lower query,
// S L405) while batch goodput (sum_q (E_q + 1)) / L[sum_q (gamma_q + 1)] strictly improves.
// Because P_{q,j} is non-increasing in j, that sequence of additions is exactly the list
// of all B*k candidates sorted by (gain desc, query asc, position asc) (DESIGN R16), so
// one CTA: (1) computes the gains, (2) bitonic-sorts them in shared memory, (3) one thread
// walks the sorted prefix in the greedy's own fp64 association until goodput stops
// improving, (4) gamma_q / E_q are read off the selected prefix.
#include <float.h>

#include "sv_device.cuh"
#include "sv_internal.h"

namespace sv {

namespace {

constexpr int kGreedyThreads = 1024;
constexpr int kGreedyMax = 8192;  // B * k candidates

__device__ __forceinline__ bool before(double ga, int ia, double gb, int ib) {
  return ga > gb || (ga == gb && ia < ib);
}

__global__ void __launch_bounds__(kGreedyThreads) sv_greedy_kernel(const ScheduleArgs a, int npow2) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) uint8_t smem[];
  double *g = reinterpret_cast<double *>(smem);
  int *id = reinterpret_cast<int *>(g + npow2);
  __shared__ int s_stop;
  __shared__ double s_G;
  const int B = a.B, k = a.k, N = B * k, tid = threadIdx.x;

  // (1) gains: per-sequence prefix products (thread per sequence, sequential fp64)
  for (int q = tid; q < B; q += blockDim.x) {
    double P = 1.0;
    int st = 0;
    for (int j = 0; j < k; ++j) {
      float v = a.p_hat[(int64_t)q * k + j];
      if (!(fabsf(v) <= FLT_MAX)) {
        v = 0.f;
        st |= 16;
      }
      P = __dmul_rn(P, (double)v);
      g[q * k + j] = P;
      id[q * k + j] = q * k + j;
    }
    if (a.status) a.status[q] = st;
  }
  for (int x = N + tid; x < npow2; x += blockDim.x) {
    g[x] = -1.0;
    id[x] = INT_MAX;
  }
  __syncthreads();
  // (2) bitonic sort, order = before()
  for (int size = 2; size <= npow2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int x = tid; x < npow2; x += blockDim.x) {
        const int y = x ^ stride;
        if (y > x) {
          const bool up = (x & size) == 0;
          const bool sw = up ? before(g[y], id[y], g[x], id[x]) : before(g[x], id[x], g[y], id[y]);
          if (sw) {
            const double tg = g[x];
            g[x] = g[y];
            g[y] = tg;
            const int ti = id[x];
            id[x] = id[y];
            id[y] = ti;
          }
        }
      }
      __syncthreads();
    }
  }
  // (3) walk the sorted prefix with the greedy's stop rule
  if (tid == 0) {
    double num = 0.0;
    for (int q = 0; q < B; ++q) num = __dadd_rn(num, 1.0);
    int64_t n = B;
    double G = __ddiv_rn(num, a.L[n]);
    int m = 0;
    while (m < N && n + 1 < a.n_lat) {
      const double num2 = __dadd_rn(num, g[m]);
      const double G2 = __ddiv_rn(num2, a.L[n + 1]);
      if (!(G2 > G)) break;
      num = num2;
      G = G2;
      ++n;
      ++m;
    }
    s_stop = m;
    s_G = G;
  }
  __syncthreads();
  // (4) per-sequence gamma and E (selected gains of a sequence are its first gamma_q
  //     positions, in position order)
  const int stop = s_stop;
  for (int q = tid; q < B; q += blockDim.x) {
    int gam = 0;
    for (int x = 0; x < stop; ++x) gam += (id[x] / k == q) ? 1 : 0;
    double E = 0.0, P = 1.0;
    for (int j = 0; j < gam; ++j) {
      float v = a.p_hat[(int64_t)q * k + j];
      if (!(fabsf(v) <= FLT_MAX)) v = 0.f;
      P = __dmul_rn(P, (double)v);
      E = __dadd_rn(E, P);
    }
    a.gamma[q] = gam;
    if (a.exp_accept) a.exp_accept[q] = (float)E;
    if (a.goodput) a.goodput[q] = (float)s_G;
  }
}

}  // namespace

cudaError_t launch_schedule_greedy(const ScheduleArgs &a, cudaStream_t st) {
  int npow2 = 1;
  while (npow2 < a.B * a.k) npow2 <<= 1;
  if (npow2 > kGreedyMax) return cudaErrorInvalidValue;
  const size_t smem = (size_t)npow2 * (sizeof(double) + sizeof(int));
  cudaError_t e = cudaFuncSetAttribute(sv_greedy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return launch_k(sv_greedy_kernel, dim3(1), dim3(kGreedyThreads), smem, st, a, npow2);
}

}  // namespace sv
