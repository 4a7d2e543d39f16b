// sd_verify.cu -- K4 + K5: steps a5-a6 (standard SD verification and the correction /
// bonus sample; P L29 citing Leviathan et al.; S L148-165, L82-90; DESIGN R1, R10-R13).
//
// K4 sv_rows_kernel: one CTA per (target row, vocabulary split).  Rows i > gamma_b exit at
//   once, so only the verified target rows are streamed from HBM.  16 independent 16-byte
//   streaming loads per thread are issued before any use (64 KB in flight per CTA), then
//   the split's raw max m and l = sum 2^{(x - m) log2e / tau_t} are reduced (per-unit
//   fp32 sums, fp64 per thread and per block) and written as one (m, l) partial.
// K5 sv_sample_kernel: one CTA cluster per sequence.
//   prologue (every CTA, identically): merge the (m, l) partials of rows 0..gamma_b in
//   split order, p_t(t_i), ratio_i = p_t(t_i) / p_d(t_i), Philox u_i, N_b = first
//   rejection; u_s = word 1 of position N_b.
//   body: CTA r bulk-copies its vocabulary chunk of the target row N_b (and of the draft
//   row N_b when rejected) into smem, computes r_v = max(0, p_t - p_d) (or p_t for the
//   bonus), and sums it in fp64 in a fixed (lane, round, warp, rank) order.  The chunk
//   sums are exchanged through DSMEM; the CTA whose range contains u_s * Z locates the
//   token by warp scan + in-lane sequential scan (smallest j with cum_j > u_s Z).
#include <float.h>

#include "sv_device.cuh"
#include "sv_internal.h"

namespace sv {

namespace {

// ------------------------------------------------------------------ K4
template <typename T>
__global__ void __launch_bounds__(kRowsThreads, 4) sv_rows_kernel(const VerifyArgs a) {
  constexpr int NT = kRowsThreads, EPU = Elem<T>::kPerUnit, U = kRowUnitsPerThread;
  __shared__ float fscr[NT / 32];
  __shared__ double dscr[NT / 32];
  const int64_t cta = blockIdx.x;
  const int64_t row = cta / a.splits, split = cta % a.splits;
  const int64_t b = row / (a.k + 1), i = row % (a.k + 1);
  const int g = a.gamma[b];
  if (g < 0 || g > a.k || i > g) return;
  const int64_t v0 = split * a.rows_chunk;
  const int n = (int)min(a.rows_chunk, (int64_t)a.V - v0);
  const T *src = reinterpret_cast<const T *>(a.t) + b * a.t_sb + i * a.t_si + v0;
  const int tid = threadIdx.x;
  const float c = a.ct;
  float m = kMFloor;
  double l = 0.0;
  if ((reinterpret_cast<uintptr_t>(src) & 15) == 0) {
    const int units = n / EPU;
    uint4 r[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int u = tid + j * NT;
      if (u < units) r[j] = ldg_stream(src + (size_t)u * EPU);
    }
    const int tail = n - units * EPU;
    float xt = kMFloor;
    if (tid < tail) xt = Elem<T>::load(src + units * EPU + tid);
#pragma unroll
    for (int j = 0; j < U; ++j) {
      if (tid + j * NT < units) {
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
      if (tid + j * NT < units) {
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
    if (tid < tail) l += ex2(fmaf(xt, c, nm));
  } else {  // unaligned row start (edge cases): element-wise online loop
    for (int e = tid; e < n; e += NT) {
      const float x = Elem<T>::load(src + e);
      if (x > m) {
        l *= ex2((m - x) * c);
        m = x;
      }
      l += ex2(fmaf(x, c, -m * c));
    }
  }
  const float M = block_max<NT>(m, fscr);
  double v = l * ex2((m - M) * c);
  v = warp_sum_d(v);
  if ((tid & 31) == 0) dscr[tid >> 5] = v;
  __syncthreads();
  if (tid == 0) {
    double s = dscr[0];
    for (int w = 1; w < NT / 32; ++w) s += dscr[w];
    a.partials[row * a.splits + split] = make_float2(M, (float)s);
  }
}

// ------------------------------------------------------------------ K5
struct SampleSmemTail {
  uint64_t bar;
  int N, st, gamma, mode;
  float Mt, dm;
  double Lt, dl, us;
  double wsum[kSampleThreads / 32];
  double zslot[2];  // this CTA's chunk mass, per pass
  int found_tok;
};

template <typename T>
struct SampleCtx {
  const T *st_, *sd_;
  int n, units, NW;
  bool resid;
  float ct, cd, nmt, nmd, ilt, ild;
  __device__ __forceinline__ float r_at(int e) const {
    const float pt = ex2(fmaf(Elem<T>::load(st_ + e), ct, nmt)) * ilt;
    if (!resid) return pt;
    const float pd = ex2(fmaf(Elem<T>::load(sd_ + e), cd, nmd)) * ild;
    return fmaxf(0.f, pt - pd);
  }
  // fp64 mass of one 16-byte unit (elements in order)
  __device__ __forceinline__ double unit_mass(int u) const {
    constexpr int EPU = Elem<T>::kPerUnit;
    double v = 0.0;
    const int e0 = u * EPU;
    if (e0 + EPU <= n) {
      float xt[EPU], xd[EPU];
      Elem<T>::unit(*reinterpret_cast<const uint4 *>(st_ + e0), xt);
      if (resid) Elem<T>::unit(*reinterpret_cast<const uint4 *>(sd_ + e0), xd);
#pragma unroll
      for (int j = 0; j < EPU; ++j) {
        const float pt = ex2(fmaf(xt[j], ct, nmt)) * ilt;
        float r = pt;
        if (resid) r = fmaxf(0.f, pt - ex2(fmaf(xd[j], cd, nmd)) * ild);
        v += (double)r;
      }
    } else {
      for (int e = e0; e < n; ++e) v += (double)r_at(e);
    }
    return v;
  }
};

template <typename T>
__global__ void __launch_bounds__(kSampleThreads) sv_sample_kernel(const VerifyArgs a) {
  constexpr int NT = kSampleThreads, NW = NT / 32, EPU = Elem<T>::kPerUnit;
  cg::cluster_group cluster = cg::this_cluster();
  const int cs = a.cs;
  const int rank = (int)cluster.block_rank();
  const int64_t b = blockIdx.x / cs;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int k = a.k;
  extern __shared__ __align__(128) uint8_t smem[];
  const size_t cbytes = (size_t)a.chunk * sizeof(T);
  T *s_t = reinterpret_cast<T *>(smem);
  T *s_d = reinterpret_cast<T *>(smem + cbytes);
  SampleSmemTail *tl = reinterpret_cast<SampleSmemTail *>(smem + 2 * cbytes);
  const float nanf_ = __int_as_float(0x7fc00000);

  // ---------------- prologue (warp 0): merge row partials, accept tests, N_b
  if (wid == 0) {
    const int g = a.gamma[b];
    int st = (g < 0 || g > k) ? 64 /*BAD_GAMMA*/ : 0;
    const int gg = st ? -1 : g;
    float Mi = kMFloor;
    double Li = 0.0;
    int lst = 0;
    bool acc = true;
    double ratio = 0.0;
    if (lane <= gg) {
      const float2 *pp = a.partials + ((int64_t)b * (k + 1) + lane) * a.splits;
      for (int s = 0; s < a.splits; ++s) Mi = fmaxf(Mi, pp[s].x);
      for (int s = 0; s < a.splits; ++s) Li += (double)pp[s].y * ex2((pp[s].x - Mi) * a.ct);
      if (!(Li == Li) || !(Mi < FLT_MAX) || !(Li < 1e300)) lst |= 1;
      else if (!(Li > 0.0)) lst |= 2;
      if (lane < gg) {
        const int64_t ri = b * k + lane;
        const int t = a.tok[ri];
        const float dl = a.dl[ri], dpt = a.dpt[ri];
        if (!(dl == dl)) lst |= 1;
        else if (!(dl > 0.f)) lst |= 2;
        if (t < 0 || t >= a.V) lst |= 4;
        else if (!lst) {
          if (!(dpt > 0.f)) {
            lst |= (dpt == 0.f) ? 8 : 1;
          } else {
            const T *trow = reinterpret_cast<const T *>(a.t) + b * a.t_sb + lane * a.t_si;
            const float xt = Elem<T>::load(trow + t);
            const double pt = exp2((double)xt * a.ct - (double)(Mi * a.ct)) / Li;
            ratio = pt / (double)dpt;
            const uint4 w = sv_philox(a.seed, a.offset, a.seq_base + b, lane);
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
    if (rank == 0 && lane < k) {
      float out = nanf_;
      if (!st && lane < gg) out = (float)fmin(1.0, ratio);
      if (a.ratio) a.ratio[b * k + lane] = out;
    }
    if (lane == 0) {
      tl->N = N;
      tl->st = st;
      tl->gamma = gg;
      tl->Mt = MN;
      tl->Lt = LN;
      if (!st && N < gg) {
        tl->dm = a.dm[b * k + N];
        tl->dl = (double)a.dl[b * k + N];
      } else {
        tl->dm = 0.f;
        tl->dl = 1.0;
      }
      tl->us = st ? 0.0 : u24(sv_philox(a.seed, a.offset, a.seq_base + b, N).y);
      tl->mode = (!st && N < gg) ? 1 : 0;  // 1 = residual, 0 = target (bonus)
      tl->found_tok = -1;
      mbar_init(&tl->bar, 1);
      fence_mbar_init();
    }
  }
  __syncthreads();
  const int N = tl->N;
  int st = tl->st;
  if (st) {
    if (rank == 0 && tid == 0) {
      a.n_accept[b] = 0;
      a.out_tok[b] = -1;
      if (a.resid) a.resid[b] = nanf_;
      if (a.status) a.status[b] = st;
    }
    return;  // uniform over the whole cluster: no cluster barrier was entered
  }
  const bool resid0 = tl->mode == 1;

  // ---------------- load this CTA's chunk of target row N (+ draft row N)
  const int64_t v0 = (int64_t)rank * a.chunk;
  const int n = (int)max((int64_t)0, min(a.chunk, (int64_t)a.V - v0));
  const T *gt = reinterpret_cast<const T *>(a.t) + b * a.t_sb + (int64_t)N * a.t_si + v0;
  const T *gd = reinterpret_cast<const T *>(a.d) + b * a.d_sb + (int64_t)N * a.d_si + v0;
  const int units_full = n / EPU;
  const bool bulk = units_full > 0 && (reinterpret_cast<uintptr_t>(gt) & 15) == 0 &&
                    (!resid0 || (reinterpret_cast<uintptr_t>(gd) & 15) == 0);
  const int bulk_units = bulk ? units_full : 0;
  if (tid == 0 && bulk) {
    const uint32_t bytes = (uint32_t)bulk_units * 16u;
    mbar_arrive_expect_tx(&tl->bar, resid0 ? 2u * bytes : bytes);
    bulk_g2s(s_t, gt, bytes, &tl->bar);
    if (resid0) bulk_g2s(s_d, gd, bytes, &tl->bar);
  }
  for (int e = bulk_units * EPU + tid; e < n; e += NT) {
    s_t[e] = gt[e];
    if (resid0) s_d[e] = gd[e];
  }
  __syncthreads();
  if (bulk) mbar_wait(&tl->bar, 0);

  SampleCtx<T> cx;
  cx.st_ = s_t;
  cx.sd_ = s_d;
  cx.n = n;
  cx.units = (n + EPU - 1) / EPU;
  cx.NW = NW;
  cx.ct = a.ct;
  cx.cd = a.cd;
  cx.nmt = -(tl->Mt * a.ct);
  cx.ilt = (float)(1.0 / tl->Lt);
  cx.nmd = -(tl->dm * a.cd);
  cx.ild = (float)(1.0 / tl->dl);
  const int Uw = (cx.units + NW - 1) / NW;
  const int wbeg = min(cx.units, wid * Uw), wend = min(cx.units, (wid + 1) * Uw);

  for (int pass = 0; pass < 2; ++pass) {
    cx.resid = resid0 && pass == 0;
    // per-warp mass: rounds of 32 units, lane value = in-unit sequential fp64 sum,
    // round total = lane 31 of the inclusive warp scan, summed round by round
    double R = 0.0;
    for (int base = wbeg; base < wend; base += 32) {
      const int u = base + lane;
      const double v = (u < wend) ? cx.unit_mass(u) : 0.0;
      const double incl = warp_incl_scan_d(v, lane);
      R += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) tl->wsum[wid] = R;
    __syncthreads();
    if (tid == 0) {
      double z = 0.0;
      for (int w = 0; w < NW; ++w) z += tl->wsum[w];
      tl->zslot[pass] = z;
    }
    cluster.sync();  // chunk masses of this pass visible cluster-wide
    // warp 0 fetches the chunk masses (lane r <- rank r) and walks them in rank order
    __shared__ double s_Z, s_Pc, s_Zc;
    __shared__ int s_owner;
    if (wid == 0) {
      const double zr = lane < cs ? cluster.map_shared_rank(tl->zslot, lane)[pass] : 0.0;
      double Zs = 0.0;
      for (int r = 0; r < cs; ++r) Zs += __shfl_sync(0xffffffffu, zr, r);
      const double th = tl->us * Zs;
      double P = 0.0, Pc_ = 0.0, Zc_ = -1.0;
      int own = -1, last_pos = -1;
      for (int r = 0; r < cs; ++r) {
        const double z = __shfl_sync(0xffffffffu, zr, r);
        if (z > 0.0) last_pos = r;
        if (own < 0 && P + z > th) {
          own = r;
          Pc_ = P;
          Zc_ = z;
        }
        P += z;
      }
      if (own < 0) {  // rounding: no crossing -> last CTA with mass
        own = last_pos;
        Pc_ = 0.0;
        Zc_ = -1.0;
      }
      if (lane == 0) {
        s_Z = Zs;
        s_Pc = Pc_;
        s_Zc = Zc_;
        s_owner = own;
      }
    }
    __syncthreads();
    const double Z = s_Z, Pc = s_Pc, Zc = s_Zc;
    const int owner = s_owner;
    if (cx.resid && !(Z > 0.0)) {  // DESIGN R10: residual mass 0 -> sample p_t instead
      st |= 32;
      cluster.sync();  // keep zslot[0] alive until every CTA has read it
      continue;
    }
    const double theta = tl->us * Z;
    if (rank == owner) {
      // level 2: the warp whose range crosses theta (thread 0, fixed order)
      __shared__ int s_w;
      __shared__ double s_Q;
      if (tid == 0) {
        int w_star = -1, w_last = -1;
        double Q = Pc, Qs = 0.0;
        const bool exact = Zc >= 0.0;
        for (int w = 0; w < NW; ++w) {
          if (tl->wsum[w] > 0.0) w_last = w;
          if (w_star < 0 && exact && Q + tl->wsum[w] > theta) {
            w_star = w;
            Qs = Q;
          }
          Q += tl->wsum[w];
        }
        if (w_star < 0) {
          w_star = w_last;
          Qs = -1.0;  // fallback marker: take the last positive element of that warp
        }
        s_w = w_star;
        s_Q = Qs;
      }
      __syncthreads();
      if (wid == s_w) {
        // level 3: rounds of the warp; level 4: in-lane sequential scan
        const bool exact = s_Q >= 0.0;
        double Rq = s_Q;
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
    cluster.sync();  // no CTA exits while others may still read its zslot
    break;
  }
}

}  // namespace

cudaError_t launch_verify(const VerifyArgs &a, cudaStream_t st) {
  // K4
  {
    const int64_t grid = (int64_t)a.B * (a.k + 1) * a.splits;
    if (a.bf16)
      sv_rows_kernel<__nv_bfloat16><<<(unsigned)grid, kRowsThreads, 0, st>>>(a);
    else
      sv_rows_kernel<float><<<(unsigned)grid, kRowsThreads, 0, st>>>(a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  // K5
  const int elem = a.bf16 ? 2 : 4;
  const size_t smem = 2 * (size_t)a.chunk * elem + sizeof(SampleSmemTail);
  const void *fn = a.bf16 ? (const void *)sv_sample_kernel<__nv_bfloat16> : (const void *)sv_sample_kernel<float>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (a.cs > 8) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((int64_t)a.B * a.cs));
  cfg.blockDim = dim3(kSampleThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = a.cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (a.bf16) return cudaLaunchKernelEx(&cfg, sv_sample_kernel<__nv_bfloat16>, a);
  return cudaLaunchKernelEx(&cfg, sv_sample_kernel<float>, a);
}

}  // namespace sv
