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
#include "sd_verify_dev.cuh"

#ifndef SV_K4_MINB
#define SV_K4_MINB 4  // K4 CTAs per SM (64 registers)
#endif
#ifndef SV_K5_MINB
#define SV_K5_MINB 5  // K5 CTAs per SM (48 registers, no spills; 3 and 4 measured slower)
#endif

namespace sv {

SV_TRACE_DECL

namespace {

// K4b sv_decide_kernel: one CTA of k+1 warps per sequence.  Warp i <= gamma_b merges row i's
// split partials in a fixed order (lane-strided sequential, then butterfly) into (M_i, L_i);
// warp 0 then runs the accept tests: p_t(t_i), ratio_i = p_t(t_i) / p_d(t_i), u_i, N_b =
// first rejection, and writes the Decision for K5 (+ n_accept, accept_ratio).
template <typename T>
__global__ void __launch_bounds__(32 * (SV_MAX_K_DEV + 1)) sv_decide_kernel(const __grid_constant__ VerifyArgs a) {
  __shared__ float s_M[SV_MAX_K_DEV + 1];
  __shared__ double s_L[SV_MAX_K_DEV + 1];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t b = blockIdx.x;
  DecidePre pre{};
  if (wid == 0) pre = decide_prefetch<T>(a, b);  // inputs written >= 2 launches earlier (see there)
  pdl_wait();
  pdl_trigger();
  SV_TRACE_START(3);
  const int g = a.gamma[b];
  if (g >= 0 && g <= a.k && wid <= g) {
    float M;
    double L;
    merge_row_warp(a, b, wid, M, L);
    if (lane == 0) {
      s_M[wid] = M;
      s_L[wid] = L;
    }
  }
  __syncthreads();
  if (wid != 0) return;
  const bool in = g >= 0 && g <= a.k && lane <= g;
  decide_warp<T>(a, b, g, in ? s_M[lane] : kMFloor, in ? s_L[lane] : 0.0, pre);
  SV_TRACE_END(3);
}

// Persistent warp-granular K4 over the items (b, i <= gamma_b, split), in sequence order.
template <typename T>
__global__ void __launch_bounds__(kRowsThreads, SV_K4_MINB) sv_rows_kernel(const __grid_constant__ VerifyArgs a) {
  constexpr int NT = kRowsThreads, NW = NT / 32;
  __shared__ int s_pref[NT + 1];
  __shared__ int s_wtot[NW];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  pdl_wait();
  pdl_trigger();
  SV_TRACE_START(2);
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
  SV_TRACE_END(2);
}

template <typename T>
__global__ void __launch_bounds__(256) sv_find_kernel(const __grid_constant__ VerifyArgs a) {
  pdl_wait();
  pdl_trigger();
  SV_TRACE_START(5);
  const int64_t b = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (b < a.B) find_seq<T>(a, b);
  SV_TRACE_END(5);
}

// Persistent warp-granular K5 over the B x nsl warp slices: per slice the residual mass and
// the target mass (the R10 fallback), each the lane-31 value of a fixed-order warp scan.
template <typename T>
__global__ void __launch_bounds__(kSampleThreads, SV_K5_MINB) sv_resid_kernel(const __grid_constant__ VerifyArgs a) {
  const int wid = threadIdx.x >> 5;
  pdl_wait();
  pdl_trigger();
  SV_TRACE_START(4);
  const int64_t nwarps = (int64_t)gridDim.x * (kSampleThreads / 32);
  const int64_t items = (int64_t)a.B * a.nsl;
  for (int64_t it = (int64_t)blockIdx.x * (kSampleThreads / 32) + wid; it < items; it += nwarps) {
    const int64_t b = it / a.nsl;
    const Decision dc = a.dec[b];
    if (!dc.st) resid_item<T>(a, dc, b, it - b * a.nsl);  // (bad sequences: K4b wrote the sentinels)
  }
  SV_TRACE_END(4);
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

// SV_EXP_VERIFY_STAGES: build-time experiment knob (scripts/k1_ab.py variants time the chain
// stage by stage); the product always launches all four stages.
#ifndef SV_EXP_VERIFY_STAGES
#define SV_EXP_VERIFY_STAGES 4
#endif
cudaError_t launch_verify(const VerifyArgs &a, cudaStream_t st) {
  for (int stage = 0; stage < SV_EXP_VERIFY_STAGES; ++stage) {
    const cudaError_t e = launch_verify_stage(stage, a, st);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace sv

SV_TRACE_READER(verify)
