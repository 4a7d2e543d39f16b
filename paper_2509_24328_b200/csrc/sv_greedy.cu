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
  double *Ls = g + npow2 + 2;                        // L[B .. B + N + 1]: the walk's latencies
  float *ph = reinterpret_cast<float *>(Ls + npow2 + 2);  // p_hat staged once
  int *id = reinterpret_cast<int *>(ph + npow2);
  __shared__ int s_stop;
  __shared__ double s_G;
  const int B = a.B, k = a.k, N = B * k, tid = threadIdx.x;

  // (0) stage p_hat and the latencies the walk can reach (coalesced, all threads)
  // the latencies the walk can reach, L[B .. B + mmax], must be positive and finite (as in the
  // per-row mode); otherwise every sequence gets the sentinel gamma = 0 and SV_ROW_BAD_LATENCY
  __shared__ int s_badlat;
  if (tid == 0) s_badlat = 0;
  __syncthreads();
  const int mmax = (int)min((int64_t)N, (int64_t)a.n_lat - 1 - B);  // n + 1 < n_lat
  for (int x = tid; x < N; x += blockDim.x) ph[x] = a.p_hat[x];
  for (int x = tid; x <= N + 1; x += blockDim.x) {
    const double v = (int64_t)B + x < a.n_lat ? a.L[B + x] : 1.0;
    Ls[x] = v;
    if (x <= max(mmax, 0) && !(v > 0.0 && v <= DBL_MAX)) s_badlat = 1;
  }
  __syncthreads();
  if (s_badlat) {
    for (int q = tid; q < B; q += blockDim.x) {
      a.gamma[q] = 0;
      if (a.exp_accept) a.exp_accept[q] = 0.f;
      if (a.goodput) a.goodput[q] = __int_as_float(0x7fc00000);
      if (a.status) a.status[q] = 128;  // SV_ROW_BAD_LATENCY
    }
    return;
  }
  // (1) gains: per-sequence prefix products (thread per sequence, sequential fp64)
  for (int q = tid; q < B; q += blockDim.x) {
    double P = 1.0;
    int st = 0;
    for (int j = 0; j < k; ++j) {
      float v = ph[q * k + j];
      if (!(v >= 0.f && v <= 1.f)) {  // not a probability: used as 0 (SV_ROW_PHAT_BAD, DESIGN R22)
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
  // (3) the greedy's stop rule on the sorted prefix: the running numerators B + G_m in the
  //     greedy's own association (one thread, sequential fp64, written over the sorted gains),
  //     then every
  //     goodput (B + G_m) / L[B + m] in parallel and the first m whose successor is not strictly
  //     better (block min).  Identical operations to the sequential walk, so identical bits.
  if (tid == 0) {
    double num = 0.0;
    for (int q = 0; q < B; ++q) num = __dadd_rn(num, 1.0);
    double prev = g[0];
    g[0] = num;  // g[m] <- numerator before candidate m (g has npow2 + 2 slots)
    for (int m = 0; m < N; ++m) {
      const double gm = prev;
      prev = g[m + 1];
      num = __dadd_rn(num, gm);
      g[m + 1] = num;
    }
    s_stop = N;  // default: every candidate taken (or the latency table ends first)
  }
  __syncthreads();
  for (int m = tid; m < mmax; m += blockDim.x) {
    const double G = __ddiv_rn(g[m], Ls[m]), G2 = __ddiv_rn(g[m + 1], Ls[m + 1]);
    if (!(G2 > G)) atomicMin(&s_stop, m);
  }
  __syncthreads();
  if (tid == 0) {
    const int stop = min(s_stop, mmax < 0 ? 0 : mmax);
    s_stop = stop;
    s_G = __ddiv_rn(g[stop], Ls[stop]);
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
      float v = ph[q * k + j];
      if (!(v >= 0.f && v <= 1.f)) v = 0.f;
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
  const size_t smem = (size_t)npow2 * (2 * sizeof(double) + sizeof(float) + sizeof(int)) + 4 * sizeof(double);
  // raise the shared-memory opt-in once per device and size (a host API call, not per launch)
  static size_t attr_smem[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || smem > attr_smem[dev]) {
    cudaError_t e = cudaFuncSetAttribute(sv_greedy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < 64) attr_smem[dev] = smem;
  }
  return launch_k(sv_greedy_kernel, dim3(1), dim3(kGreedyThreads), smem, st, a, npow2);
}

}  // namespace sv
