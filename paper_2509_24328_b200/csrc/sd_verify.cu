// sd_verify.cu -- steps a5-a6: standard SD verification and the correction / bonus sample
// (P L29 citing Leviathan et al.; S L148-165, L82-90; DESIGN R1, R10-R13).
//
// One fused kernel, one thread-block CLUSTER per sequence b; CTA r owns vocabulary chunk r of
// every row of that sequence (same cluster-size rule as sv_score: a function of (V, dtype)).
//   rows    : stream the chunk of target rows 0..gamma_b from HBM (rows > gamma_b are never
//             read; 16-byte loads, L2 evict_last) -> per-row raw max m and l = sum 2^{(x-m)c}
//   exchange: the last warp (highest id, favoured by the arbiter) pushes the per-row (m, l) into
//             every CTA of the cluster over DSMEM (remote mbarrier arrive, release.cluster); every
//             CTA merges them in rank order -> identical p_t(t_i), ratio_i = p_t/p_d, Philox u_i,
//             N_b = first rejection, u_s = word 1 of position N_b
//   sample  : r_v = max(0, p_t - p_d) of row N_b (T chunk re-read from L2, D chunk from HBM) or
//             p_t of row gamma_b (bonus), summed in fp64 in a fixed (lane, round, warp, rank)
//             order; chunk masses exchanged over DSMEM; the CTA whose range holds u_s * Z locates
//             the token by warp scan + in-lane sequential scan (smallest j with cum_j > u_s Z).
// No workspace, no atomics, no second launch: the decision chain (partials -> N_b -> row N_b)
// stays inside the cluster.  Every reduction order depends on (V, dtype) only.
#include <float.h>

#include "../../include/sv.h"
#include "sv_device.cuh"
#include "sv_internal.h"

namespace sv {

namespace {

constexpr int NT = kVerifyThreads, NW = NT / 32, G = kVerifyGroup;
constexpr int KR = SV_MAX_K + 1;  // target rows per sequence, at most

struct VSmem {
  uint64_t bar_rows;                // all ranks' row partials landed (count cs)
  uint64_t bar_mass[2];             // all ranks' chunk masses landed, per sampling pass (count cs)
  float rowpart[kMaxCluster][KR][2];  // (m, l) of every row, pushed by every rank
  float myrow[KR][2];               // this CTA's row partials
  double zslot[2][kMaxCluster];     // chunk masses, per pass, pushed by every rank
  double wsum[NW];
  float fscr[2 * NW];
  double dscr[NW];
  // decision, broadcast to the CTA
  int N, st, gg, owner, w_star;
  float Mt, dm;
  double Lt, dl, us, Z, Pc, Zc, Q;
};

__device__ __forceinline__ uint32_t remote(const void *p, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void remote_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void st_remote_f32(uint32_t addr, float v) {
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
__device__ __forceinline__ void st_remote_f64(uint32_t addr, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
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
__device__ __forceinline__ void cluster_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.aligned;" ::: "memory"); }
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint4 ldg_hint(const void *p, uint64_t pol) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p), "l"(pol));
  return r;
}

template <typename T>
__device__ __forceinline__ float unit_max(const uint4 &v) {
  if constexpr (sizeof(T) == 2) {
    const __nv_bfloat162 *p = reinterpret_cast<const __nv_bfloat162 *>(&v);
    const __nv_bfloat162 m = __hmax2(__hmax2(p[0], p[1]), __hmax2(p[2], p[3]));
    return fmaxf(__low2float(m), __high2float(m));
  } else {
    return fmaxf(fmaxf(__uint_as_float(v.x), __uint_as_float(v.y)), fmaxf(__uint_as_float(v.z), __uint_as_float(v.w)));
  }
}

// (m, l) of the thread's share of one target-row chunk: groups of G units in flight together,
// exact online rescale between groups, element-wise remainder.
template <typename T>
__device__ __forceinline__ void row_thread(const T *x, int n, bool vec, float c, uint64_t pol, float &m, float &l) {
  constexpr int EPU = Elem<T>::kPerUnit;
  const int tid = threadIdx.x;
  const int units = vec ? n / EPU : 0;
  m = kMFloor;
  l = 0.f;
  for (int u0 = tid; u0 < units; u0 += G * NT) {
    uint4 r[G];
#pragma unroll
    for (int q = 0; q < G; ++q)
      if (u0 + q * NT < units) r[q] = ldg_hint(x + (size_t)(u0 + q * NT) * EPU, pol);
    float gm = m;
#pragma unroll
    for (int q = 0; q < G; ++q)
      if (u0 + q * NT < units) gm = fmaxf(gm, unit_max<T>(r[q]));
    if (gm > m) {
      l *= ex2((m - gm) * c);
      m = gm;
    }
    const float nm = -m * c;
    const f2 c2{c, c}, nm2{nm, nm};
    f2 acc{0.f, 0.f};
#pragma unroll
    for (int q = 0; q < G; ++q)
      if (u0 + q * NT < units) {
        float xs[EPU];
        Elem<T>::unit(r[q], xs);
#pragma unroll
        for (int j = 0; j < EPU; j += 2) acc = add2(acc, ex2x2(fma2(f2{xs[j], xs[j + 1]}, c2, nm2)));
      }
    l += acc.x + acc.y;
  }
  for (int e = units * EPU + tid; e < n; e += NT) {
    const float xe = Elem<T>::load(x + e);
    if (xe > m) {
      l *= ex2((m - xe) * c);
      m = xe;
    }
    l += ex2(fmaf(xe, c, -m * c));
  }
}

// Residual / target mass of the sampled row, element by element in a fixed order.
template <typename T>
struct SampleCtx {
  const T *t, *d;  // chunk of target row N and draft row N (global)
  int n;
  bool vec;        // both chunks 16-byte aligned
  bool resid;
  float ct, cd, nmt, nmd, ilt, ild;
  __device__ __forceinline__ float r_at(int e) const {
    const float pt = ex2(fmaf(Elem<T>::load(t + e), ct, nmt)) * ilt;
    if (!resid) return pt;
    const float pd = ex2(fmaf(Elem<T>::load(d + e), cd, nmd)) * ild;
    return fmaxf(0.f, pt - pd);
  }
  // fp64 mass of one 16-byte unit (elements in order)
  __device__ __forceinline__ double unit_mass(int u) const {
    constexpr int EPU = Elem<T>::kPerUnit;
    double v = 0.0;
    const int e0 = u * EPU;
    if (vec && e0 + EPU <= n) {
      float xt[EPU], xd[EPU];
      Elem<T>::unit(ldg_stream(t + e0), xt);
      if (resid) Elem<T>::unit(ldg_stream(d + e0), xd);
#pragma unroll
      for (int j = 0; j < EPU; ++j) {
        const float pt = ex2(fmaf(xt[j], ct, nmt)) * ilt;
        const float r = resid ? fmaxf(0.f, pt - ex2(fmaf(xd[j], cd, nmd)) * ild) : pt;
        v += (double)r;
      }
    } else {
      for (int e = e0; e < min(n, e0 + EPU); ++e) v += (double)r_at(e);
    }
    return v;
  }
};

template <typename T>
__global__ void __launch_bounds__(kVerifyThreads, kVerifyMinBlocks) sv_verify_kernel(const VerifyArgs a) {
  __shared__ VSmem sm;
  cg::cluster_group cluster = cg::this_cluster();
  const int cs = a.cs;
  const int rank = (int)cluster.block_rank();
  const int64_t b = blockIdx.x / cs;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const bool ctl = wid == NW - 1;
  const int k = a.k;
  const float nanf_ = __int_as_float(0x7fc00000);
  if (tid == 0) {
    mbar_init(&sm.bar_rows, cs);
    mbar_init(&sm.bar_mass[0], cs);
    mbar_init(&sm.bar_mass[1], cs);
    fence_mbar_init();
  }
  __syncthreads();
  cluster_arrive_relaxed();  // (0) started, barriers initialised: peers may push after wait (0)

  const int g = a.gamma[b];
  const int gg = (g < 0 || g > k) ? -1 : g;  // -1: bad gamma (SV_ROW_BAD_GAMMA)
  const int64_t v0 = (int64_t)rank * a.chunk;
  const int n = (int)max((int64_t)0, min(a.chunk, (int64_t)a.V - v0));
  const T *trow0 = reinterpret_cast<const T *>(a.t) + b * a.t_sb + v0;

  // control warp: per-row token data for the accept tests, loaded now (latency hidden)
  int tok_i = 0;
  float xt_i = 0.f, dpt_i = 0.f, dl_i = 0.f;
  if (ctl && lane < gg) {
    const int64_t ri = b * k + lane;
    tok_i = a.tok[ri];
    dpt_i = a.dpt[ri];
    dl_i = a.dl[ri];
    if (tok_i >= 0 && tok_i < a.V)
      xt_i = Elem<T>::load(reinterpret_cast<const T *>(a.t) + b * a.t_sb + (int64_t)lane * a.t_si + tok_i);
  }

  // ---- rows 0..gamma: chunk (m, l) partials
  const uint64_t pol_keep = l2_policy_evict_last();
  for (int i = 0; i <= gg; ++i) {
    const T *x = trow0 + (int64_t)i * a.t_si;
    float m, l;
    row_thread<T>(x, n, (reinterpret_cast<uintptr_t>(x) & 15) == 0, a.ct, pol_keep, m, l);
    const float Mw = warp_max(m);
    if (lane == 0) sm.fscr[wid] = Mw;
    __syncthreads();
    float M = sm.fscr[0];
#pragma unroll
    for (int q = 1; q < NW; ++q) M = fmaxf(M, sm.fscr[q]);
    const double lw = warp_sum_d((double)l * ex2((m - M) * a.ct));
    if (lane == 0) sm.dscr[wid] = lw;
    __syncthreads();
    if (tid == 0) {
      double L = 0.0;
      for (int q = 0; q < NW; ++q) L += sm.dscr[q];
      sm.myrow[i][0] = M;
      sm.myrow[i][1] = (float)L;
    }
  }
  __syncthreads();
  cluster_wait();  // (0)

  // ---- exchange + decision (control warp)
  if (ctl) {
    for (int q = lane; q < cs * (gg + 1); q += 32) {  // push (rank -> peer p, row i)
      const int p = q / (gg + 1), i = q % (gg + 1);
      st_remote_f32(remote(&sm.rowpart[rank][i][0], p), sm.myrow[i][0]);
      st_remote_f32(remote(&sm.rowpart[rank][i][1], p), sm.myrow[i][1]);
    }
    __syncwarp();
    if (lane < cs) remote_arrive(remote(&sm.bar_rows, lane));
    wait_cluster(&sm.bar_rows, 0);  // always: every peer arrives, even with nothing to push
    // lane i merges row i over the ranks in rank order
    float Mi = kMFloor;
    double Li = 0.0;
    int lst = 0;
    bool acc = true;
    double ratio = 0.0;
    if (lane <= gg) {
      for (int r = 0; r < cs; ++r) Mi = fmaxf(Mi, sm.rowpart[r][lane][0]);
      for (int r = 0; r < cs; ++r) Li += (double)sm.rowpart[r][lane][1] * ex2((sm.rowpart[r][lane][0] - Mi) * a.ct);
      if (!(Li == Li) || !(Mi < FLT_MAX) || !(Li < 1e300)) lst |= SV_ROW_NAN;
      else if (!(Li > 0.0)) lst |= SV_ROW_ALL_NEG_INF;
      if (lane < gg) {
        if (!(dl_i == dl_i)) lst |= SV_ROW_NAN;
        else if (!(dl_i > 0.f)) lst |= SV_ROW_ALL_NEG_INF;
        if (tok_i < 0 || tok_i >= a.V) {
          lst |= SV_ROW_BAD_TOKEN;
        } else if (!lst) {
          if (!(dpt_i > 0.f)) {
            lst |= (dpt_i == 0.f) ? SV_ROW_DRAFT_ZERO : SV_ROW_NAN;
          } else {
            const double pt = exp2_acc((double)xt_i * a.ct - (double)(Mi * a.ct) - log2_acc(Li));
            ratio = pt / (double)dpt_i;
            acc = u24(sv_philox(a.seed, a.offset, a.seq_base + b, lane).x) < ratio;
          }
        }
      }
    }
    int st = gg < 0 ? SV_ROW_BAD_GAMMA : 0;
    const unsigned rej = __ballot_sync(0xffffffffu, lane < gg && !acc);
    const int N = st ? 0 : (rej ? (__ffs(rej) - 1) : gg);
    int all = lst;
    if (lane == gg && N != gg) all = 0;  // row gamma's target status counts only if it is sampled
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) all |= __shfl_xor_sync(0xffffffffu, all, o);
    st |= all;
    const float MN = __shfl_sync(0xffffffffu, Mi, st ? 0 : N);
    const double LN = __shfl_sync(0xffffffffu, Li, st ? 0 : N);
    if (rank == 0 && lane < k && a.ratio) a.ratio[b * k + lane] = (!st && lane < gg) ? (float)fmin(1.0, ratio) : nanf_;
    if (lane == 0) {
      sm.N = N;
      sm.st = st;
      sm.gg = gg;
      sm.Mt = MN;
      sm.Lt = LN;
      const bool resid = !st && N < gg;
      sm.dm = resid ? a.dm[b * k + N] : 0.f;
      sm.dl = resid ? (double)a.dl[b * k + N] : 1.0;
      sm.us = st ? 0.0 : u24(sv_philox(a.seed, a.offset, a.seq_base + b, N).y);
    }
  }
  __syncthreads();
  const int N = sm.N;
  int st = sm.st;
  if (st) {
    if (rank == 0 && tid == 0) {
      a.n_accept[b] = 0;
      a.out_tok[b] = -1;
      if (a.resid) a.resid[b] = nanf_;
      if (a.status) a.status[b] = st;
    }
    return;  // every push into this CTA has landed (bar_rows), none follows
  }

  // ---- sample row N: residual (rejected) or target (bonus)
  const bool resid0 = N < sm.gg;
  SampleCtx<T> cx;
  cx.t = trow0 + (int64_t)N * a.t_si;
  cx.d = reinterpret_cast<const T *>(a.d) + b * a.d_sb + (int64_t)N * a.d_si + v0;
  cx.n = n;
  cx.vec = ((reinterpret_cast<uintptr_t>(cx.t) | reinterpret_cast<uintptr_t>(cx.d)) & 15) == 0;
  cx.ct = a.ct;
  cx.cd = a.cd;
  cx.nmt = -(sm.Mt * a.ct);
  cx.ilt = (float)(1.0 / sm.Lt);
  cx.nmd = -(sm.dm * a.cd);
  cx.ild = (float)(1.0 / sm.dl);
  constexpr int EPU = Elem<T>::kPerUnit;
  const int units = (n + EPU - 1) / EPU;
  const int Uw = (units + NW - 1) / NW;
  const int wbeg = min(units, wid * Uw), wend = min(units, (wid + 1) * Uw);

  for (int pass = 0; pass < 2; ++pass) {
    cx.resid = resid0 && pass == 0;
    // per-warp mass: rounds of 32 units, lane value = in-unit sequential fp64 sum, round total
    // = lane 31 of the inclusive warp scan, accumulated round by round
    double R = 0.0;
    for (int base = wbeg; base < wend; base += 32) {
      const int u = base + lane;
      const double v = (u < wend) ? cx.unit_mass(u) : 0.0;
      const double incl = warp_incl_scan_d(v, lane);
      R += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) sm.wsum[wid] = R;
    __syncthreads();
    if (ctl) {
      double zc = 0.0;
      for (int w = 0; w < NW; ++w) zc += sm.wsum[w];
      if (lane < cs) {
        st_remote_f64(remote(&sm.zslot[pass][rank], lane), zc);
        remote_arrive(remote(&sm.bar_mass[pass], lane));
      }
      wait_cluster(&sm.bar_mass[pass], 0);
      // walk the ranks in order (identical bits everywhere)
      const double zr = lane < cs ? sm.zslot[pass][lane] : 0.0;
      double Zs = 0.0;
      for (int r = 0; r < cs; ++r) Zs += __shfl_sync(0xffffffffu, zr, r);
      const double th = sm.us * Zs;
      double P = 0.0, Pc = 0.0, Zc = -1.0;
      int own = -1, last_pos = -1;
      for (int r = 0; r < cs; ++r) {
        const double z = __shfl_sync(0xffffffffu, zr, r);
        if (z > 0.0) last_pos = r;
        if (own < 0 && P + z > th) {
          own = r;
          Pc = P;
          Zc = z;
        }
        P += z;
      }
      if (own < 0) {  // rounding: no crossing -> last CTA with mass
        own = last_pos;
        Pc = 0.0;
        Zc = -1.0;
      }
      if (lane == 0) {
        sm.Z = Zs;
        sm.Pc = Pc;
        sm.Zc = Zc;
        sm.owner = own;
      }
    }
    __syncthreads();
    const double Z = sm.Z;
    if (cx.resid && !(Z > 0.0)) {  // DESIGN R10: residual mass 0 -> sample p_t instead
      st |= SV_ROW_RESID_ZERO;
      continue;
    }
    const double theta = sm.us * Z;
    if (rank == sm.owner) {
      // level 2: the warp whose range crosses theta (fixed order)
      if (tid == 0) {
        int w_star = -1, w_last = -1;
        double Q = sm.Pc, Qs = 0.0;
        const bool exact = sm.Zc >= 0.0;
        for (int w = 0; w < NW; ++w) {
          if (sm.wsum[w] > 0.0) w_last = w;
          if (w_star < 0 && exact && Q + sm.wsum[w] > theta) {
            w_star = w;
            Qs = Q;
          }
          Q += sm.wsum[w];
        }
        if (w_star < 0) {
          w_star = w_last;
          Qs = -1.0;  // fallback marker: take the last positive element of that warp
        }
        sm.w_star = w_star;
        sm.Q = Qs;
      }
      __syncthreads();
      if (wid == sm.w_star) {
        // level 3: rounds of the warp; level 4: in-lane sequential scan
        const bool exact = sm.Q >= 0.0;
        double Rq = sm.Q;
        int tok = -1, last_u = -1;
        for (int base = wbeg; base < wend && tok < 0; base += 32) {
          const int u = base + lane;
          const double v = (u < wend) ? cx.unit_mass(u) : 0.0;
          const double incl = warp_incl_scan_d(v, lane);
          const unsigned pos = __ballot_sync(0xffffffffu, v > 0.0);
          if (pos) last_u = base + 31 - __clz(pos);
          const unsigned cross = exact ? __ballot_sync(0xffffffffu, Rq + incl > theta) : 0u;
          if (cross) {
            const int ls = __ffs(cross) - 1;
            const double excl = __shfl_sync(0xffffffffu, incl, ls > 0 ? ls - 1 : 0);
            if (lane == ls) {
              double cum = Rq + (ls > 0 ? excl : 0.0);
              const int e0 = u * EPU, e1 = min(n, e0 + EPU);
              int lastp = -1;
              for (int e = e0; e < e1; ++e) {
                const float r = cx.r_at(e);
                if (r > 0.f) lastp = e;
                cum += (double)r;
                if (cum > theta) {
                  tok = e;
                  break;
                }
              }
              if (tok < 0) tok = lastp;
            }
            tok = __shfl_sync(0xffffffffu, tok, ls);
            break;
          }
          Rq += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (tok < 0 && last_u >= 0 && lane == 0) {  // fallback: last positive element
          const int e0 = last_u * EPU, e1 = min(n, e0 + EPU);
          for (int e = e0; e < e1; ++e)
            if (cx.r_at(e) > 0.f) tok = e;
        }
        if (lane == 0) a.out_tok[b] = (int)(v0 + tok);
      }
    }
    if (rank == 0 && tid == 0) {
      a.n_accept[b] = N;
      if (a.resid) a.resid[b] = (float)Z;
      if (a.status) a.status[b] = st;
    }
    break;
  }
  // every push into this CTA (row partials, chunk masses of the final pass) has landed
}

template <typename T>
cudaError_t launch_verify_t(const VerifyArgs &a, cudaStream_t st) {
  const void *fn = (const void *)sv_verify_kernel<T>;
  if (a.cs > 8) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((int64_t)a.B * a.cs));
  cfg.blockDim = dim3(kVerifyThreads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = a.cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, sv_verify_kernel<T>, a);
}

}  // namespace

cudaError_t launch_verify(const VerifyArgs &a, cudaStream_t st) {
  return a.bf16 ? launch_verify_t<__nv_bfloat16>(a, st) : launch_verify_t<float>(a, st);
}

}  // namespace sv
