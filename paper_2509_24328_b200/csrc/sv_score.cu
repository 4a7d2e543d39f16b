// sv_score.cu -- K1: steps a1-a3 of the SV hot path (P L159 S/A, P L164 divergence,
// north_star KL, P L176 profile lookup).
//
// Design (DESIGN.md §5 K1).  A row pair (draft row + companion row of one (b, i)) is cut into
// nch vocabulary chunks of kScoreBytes per tensor; a work item is one (row, chunk).  A
// persistent grid of co-resident CTAs (2 per SM) walks the items in "waves": wave j covers
// rows [j R, (j+1) R) with R = G / nch, CTA c owning chunk c % nch of row j R + c / nch, so all
// chunks of a row are in flight together.  Every CTA keeps a 3-slot shared-memory ring fed by
// the bulk-copy (TMA) engine one wave ahead, and in wave j runs
//   phase 1 on its item of wave j (smem slot j % 3): thread maxima (packed bf16x2 max),
//     l = sum 2^{(x - m) log2e / tau}, KL partial w = sum e_d (a_d - a_c) with packed fp32x2
//     FFMA2 / FADD2, block merge in fixed order, publish 5 partials + release-increment the
//     row counter; the CTA whose increment completes the row merges the nch partials in chunk
//     order and publishes the row's normalisers (Lambda = m c + log2 l);
//   phase 2 on its item of wave j - 1 (slot (j - 1) % 3, still resident): acquire the row's
//     Lambdas, S_q = sum 2^{min(x_d c_d - Lambda_d, x_c c_c - Lambda_c)} (one MUFU per pair);
//     the CTA that completes the row runs the epilogue (S, A, KL in fp64, profile lookup,
//     draft normalisers for sd_verify) and resets the row's counters.
// Every logit crosses HBM once and never leaves the SM that loaded it; no clusters, so all 148
// SMs work whatever the GPC layout.  Phase 2 only waits on phase-1 work of an earlier wave,
// which never waits, so the co-resident (cooperative) grid cannot deadlock.  All reduction
// orders depend on (V, dtype) only: results are bitwise identical for any B, grid size or GPU
// count.
#include <float.h>

#include "sv_device.cuh"
#include "sv_internal.h"

namespace sv {

namespace {

constexpr int NT = kScoreThreads, NW = NT / 32;

#ifdef SV_TRACE
__device__ unsigned long long *g_trace = nullptr;  // debug builds only: [cta][wave][5] timestamps
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define TR(jj, k)                                                                         \
  if (g_trace && threadIdx.x == 0 && (jj) < 64) g_trace[((size_t)blockIdx.x * 64 + (jj)) * 5 + (k)] = gtime();
#else
#define TR(jj, k)
#endif
constexpr int UPT = kScoreBytes / 16 / NT;  // 16-byte units per thread per tensor per item

struct ScoreWs {
  int32_t *cnt1, *cnt2;  // [rows] phase-1 / phase-2 arrivals (zero at rest)
  RowState *rs;          // [rows]
  ItemPart *part;        // [rows * nch]
  float *spart;          // [rows * nch]
};

__device__ __forceinline__ ScoreWs carve(const ScoreArgs &a) {
  ScoreWs w;
  const int64_t rows = (int64_t)a.B * a.k;
  uint8_t *p = reinterpret_cast<uint8_t *>(a.ws);
  w.cnt1 = reinterpret_cast<int32_t *>(p);
  w.cnt2 = w.cnt1 + rows;
  w.rs = reinterpret_cast<RowState *>(p + score_ws_row_offset(rows));
  w.part = reinterpret_cast<ItemPart *>(p + score_ws_part_offset(rows));
  w.spart = reinterpret_cast<float *>(p + score_ws_spart_offset(rows, a.nch));
  return w;
}

__device__ __forceinline__ int ld_acquire(const int32_t *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int32_t *p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

struct Item {
  int64_t row;
  int q;      // chunk index
  bool valid;
};

struct Sched {
  int64_t rows;
  int nch, R;  // chunks per row, rows per wave
  __device__ __forceinline__ Item item(int64_t wave) const {
    Item it;
    const int c = blockIdx.x;
    it.row = wave * R + c / nch;
    it.q = c % nch;
    it.valid = wave >= 0 && c < R * nch && it.row < rows;
    return it;
  }
};

template <typename T>
struct Src {
  const T *d, *c;
  int n;     // elements in the chunk
  int bulk;  // elements moved by the bulk-copy engine (multiple of 16 B)
};

template <typename T>
__device__ __forceinline__ Src<T> src_of(const ScoreArgs &a, const Item &it) {
  const int64_t b = it.row / a.k, i = it.row % a.k, v0 = (int64_t)it.q * a.chunk;
  Src<T> s;
  s.d = reinterpret_cast<const T *>(a.d) + b * a.d_sb + i * a.d_si + v0;
  s.c = reinterpret_cast<const T *>(a.c) + b * a.c_sb + i * a.c_si + v0;
  s.n = (int)min(a.chunk, (int64_t)a.V - v0);
  const bool al = ((reinterpret_cast<uintptr_t>(s.d) | reinterpret_cast<uintptr_t>(s.c)) & 15) == 0;
  s.bulk = al ? (s.n * (int)sizeof(T)) / 16 * 16 / (int)sizeof(T) : 0;
  return s;
}

struct BlockScratch {
  uint64_t bar[kScoreSlots];
  float fscr[2 * NW];
  double dscr[3 * NW];
  float lam[2];
  int flag;
};

// tid 0: start the bulk copy of an item into its slot (a row without 16-byte alignment
// just completes the barrier phase; its elements are copied by the threads in phase 1)
template <typename T>
__device__ __forceinline__ void issue(const ScoreArgs &a, const Item &it, T *slot, uint64_t *bar) {
  const Src<T> s = src_of<T>(a, it);
  if (s.bulk == 0) {
    mbar_arrive(bar);
    return;
  }
  const uint32_t bytes = (uint32_t)s.bulk * sizeof(T);
  fence_proxy_async();  // earlier generic-proxy reads of this slot precede the async writes
  mbar_arrive_expect_tx(bar, 2u * bytes);
  bulk_g2s(slot, s.d, bytes, bar);
  bulk_g2s(slot + a.chunk, s.c, bytes, bar);
}

// ---------------------------------------------------------------- phase 1 arithmetic
// One 16-byte unit of each tensor: packed bf16 max / sums with FFMA2 / FADD2.
struct P1 {
  f2 ld, lc;  // l_d, l_c partials, two lanes each
  f2 w;       // KL partial, two lanes
};

template <typename T>
__device__ __forceinline__ void p1_unit(const uint4 &ud, const uint4 &uc, f2 c2, f2 nm2, P1 &acc, f2 cdd, f2 ccc,
                                        f2 nmdd, f2 nmcc);

// bf16: 8 elements per unit; lane pairs (x_2j, x_2j+1) of one tensor share an FFMA2
template <>
__device__ __forceinline__ void p1_unit<__nv_bfloat16>(const uint4 &ud, const uint4 &uc, f2, f2, P1 &acc, f2 cdd,
                                                       f2 ccc, f2 nmdd, f2 nmcc) {
  const uint32_t wd[4] = {ud.x, ud.y, ud.z, ud.w}, wc[4] = {uc.x, uc.y, uc.z, uc.w};
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const f2 xd{bf_lo(wd[p]), bf_hi(wd[p])}, xc{bf_lo(wc[p]), bf_hi(wc[p])};
    const f2 ad = fma2(xd, cdd, nmdd), ac = fma2(xc, ccc, nmcc);
    const f2 ed = ex2x2(ad), ec = ex2x2(ac);
    acc.ld = add2(acc.ld, ed);
    acc.lc = add2(acc.lc, ec);
    acc.w = fma2(ed, sub2(ad, ac), acc.w);
  }
}
template <>
__device__ __forceinline__ void p1_unit<float>(const uint4 &ud, const uint4 &uc, f2, f2, P1 &acc, f2 cdd, f2 ccc,
                                               f2 nmdd, f2 nmcc) {
  const float xd4[4] = {__uint_as_float(ud.x), __uint_as_float(ud.y), __uint_as_float(ud.z), __uint_as_float(ud.w)};
  const float xc4[4] = {__uint_as_float(uc.x), __uint_as_float(uc.y), __uint_as_float(uc.z), __uint_as_float(uc.w)};
#pragma unroll
  for (int p = 0; p < 2; ++p) {
    const f2 xd{xd4[2 * p], xd4[2 * p + 1]}, xc{xc4[2 * p], xc4[2 * p + 1]};
    const f2 ad = fma2(xd, cdd, nmdd), ac = fma2(xc, ccc, nmcc);
    const f2 ed = ex2x2(ad), ec = ex2x2(ac);
    acc.ld = add2(acc.ld, ed);
    acc.lc = add2(acc.lc, ec);
    acc.w = fma2(ed, sub2(ad, ac), acc.w);
  }
}

// element-wise (tails / unaligned rows / guarded redo): p_d = 0 terms contribute 0 to w
__device__ __forceinline__ void p1_one(float xd, float xc, float cd, float cc, float nmd, float nmc, P1 &acc) {
  const float ad = fmaf(xd, cd, nmd), ac = fmaf(xc, cc, nmc);
  const float ed = ex2(ad);
  acc.ld.x += ed;
  acc.lc.x += ex2(ac);
  acc.w.x += ed > 0.f ? ed * (ad - ac) : 0.f;
}

__device__ __forceinline__ void umax(__nv_bfloat162 &m, const uint4 &v) {
  const __nv_bfloat162 *p = reinterpret_cast<const __nv_bfloat162 *>(&v);
  m = __hmax2(__hmax2(m, p[0]), __hmax2(p[1], __hmax2(p[2], p[3])));
}

template <typename T>
__device__ __forceinline__ void thread_max(const T *sd, const T *sc, int units, float &md, float &mc) {
  if constexpr (sizeof(T) == 2) {
    __nv_bfloat162 pd = __halves2bfloat162(__ushort_as_bfloat16(0xFF80), __ushort_as_bfloat16(0xFF80));
    __nv_bfloat162 pc = pd;
#pragma unroll
    for (int q = 0; q < UPT; ++q) {
      const int u = threadIdx.x + q * NT;
      if (u < units) {
        umax(pd, reinterpret_cast<const uint4 *>(sd)[u]);
        umax(pc, reinterpret_cast<const uint4 *>(sc)[u]);
      }
    }
    md = fmaxf(md, fmaxf(__low2float(pd), __high2float(pd)));
    mc = fmaxf(mc, fmaxf(__low2float(pc), __high2float(pc)));
  } else {
#pragma unroll
    for (int q = 0; q < UPT; ++q) {
      const int u = threadIdx.x + q * NT;
      if (u < units) {
        const float4 xd = reinterpret_cast<const float4 *>(sd)[u], xc = reinterpret_cast<const float4 *>(sc)[u];
        md = fmaxf(md, fmaxf(fmaxf(xd.x, xd.y), fmaxf(xd.z, xd.w)));
        mc = fmaxf(mc, fmaxf(fmaxf(xc.x, xc.y), fmaxf(xc.z, xc.w)));
      }
    }
  }
}

template <typename T>
__device__ void phase1(const ScoreArgs &a, const ScoreWs &ws, const Item &it, T *slot, BlockScratch &sh) {
  constexpr int EPU = Elem<T>::kPerUnit;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const float cd = a.cd, cc = a.cc;
  const Src<T> s = src_of<T>(a, it);
  T *sd = slot, *sc = slot + a.chunk;
  for (int e = s.bulk + tid; e < s.n; e += NT) {  // ragged tail / unaligned rows
    sd[e] = s.d[e];
    sc[e] = s.c[e];
  }
  if (s.bulk < s.n) __syncthreads();
  const int units = s.bulk / EPU, e0 = units * EPU;  // e0.. n-1 handled element-wise
  float md = kMFloor, mc = kMFloor;
  thread_max<T>(sd, sc, units, md, mc);
  for (int e = e0 + tid; e < s.n; e += NT) {
    md = fmaxf(md, Elem<T>::load(sd + e));
    mc = fmaxf(mc, Elem<T>::load(sc + e));
  }
  const float nmd = -md * cd, nmc = -mc * cc;
  const f2 cdd{cd, cd}, ccc{cc, cc}, nmdd{nmd, nmd}, nmcc{nmc, nmc};
  P1 acc{{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};
#pragma unroll
  for (int q = 0; q < UPT; ++q) {
    const int u = tid + q * NT;
    if (u < units)
      p1_unit<T>(reinterpret_cast<const uint4 *>(sd)[u], reinterpret_cast<const uint4 *>(sc)[u], f2{}, f2{}, acc, cdd,
                 ccc, nmdd, nmcc);
  }
  for (int e = e0 + tid; e < s.n; e += NT) p1_one(Elem<T>::load(sd + e), Elem<T>::load(sc + e), cd, cc, nmd, nmc, acc);
  float lf_d = acc.ld.x + acc.ld.y, lf_c = acc.lc.x + acc.lc.y, wf = acc.w.x + acc.w.y;
  if (wf != wf && lf_d == lf_d && lf_c == lf_c) {  // 0 * (-inf) from masked logits: guarded redo
    P1 g{{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};  // same elements per thread as the fast path
    for (int q = 0; q < UPT; ++q) {
      const int u = tid + q * NT;
      if (u < units)
        for (int j = 0; j < EPU; ++j)
          p1_one(Elem<T>::load(sd + u * EPU + j), Elem<T>::load(sc + u * EPU + j), cd, cc, nmd, nmc, g);
    }
    for (int e = e0 + tid; e < s.n; e += NT) p1_one(Elem<T>::load(sd + e), Elem<T>::load(sc + e), cd, cc, nmd, nmc, g);
    lf_d = g.ld.x;
    lf_c = g.lc.x;
    wf = g.w.x;
  }
  // ---- block merge (fixed warp / lane order)
  float Md = warp_max(md), Mc = warp_max(mc);
  if (lane == 0) {
    sh.fscr[wid] = Md;
    sh.fscr[NW + wid] = Mc;
  }
  __syncthreads();
  Md = sh.fscr[0];
  Mc = sh.fscr[NW];
#pragma unroll
  for (int q = 1; q < NW; ++q) {
    Md = fmaxf(Md, sh.fscr[q]);
    Mc = fmaxf(Mc, sh.fscr[NW + q]);
  }
  const float sdf = ex2((md - Md) * cd), scf = ex2((mc - Mc) * cc);
  const float delta = (Mc - mc) * cc - (Md - md) * cd;
  double ww = wf;
  if (lf_d > 0.f) ww += (double)lf_d * (double)delta;
  double v[3] = {(double)lf_d * sdf, (double)lf_c * scf, ww * sdf};
#pragma unroll
  for (int j = 0; j < 3; ++j) v[j] = warp_sum_d(v[j]);
  if (lane == 0)
#pragma unroll
    for (int j = 0; j < 3; ++j) sh.dscr[j * NW + wid] = v[j];
  __syncthreads();
  if (tid == 0) {
    ItemPart p;
    p.md = Md;
    p.mc = Mc;
    p.ld = sh.dscr[0];
    p.lc = sh.dscr[NW];
    p.w = sh.dscr[2 * NW];
    for (int q = 1; q < NW; ++q) {
      p.ld += sh.dscr[q];
      p.lc += sh.dscr[NW + q];
      p.w += sh.dscr[2 * NW + q];
    }
    ws.part[it.row * a.nch + it.q] = p;
    __threadfence();
    sh.flag = atomicAdd(ws.cnt1 + it.row, 1) == a.nch - 1;
    if (sh.flag) __threadfence();
  }
  __syncthreads();
  if (!sh.flag || wid != 0) return;
  // ---- this CTA completed the row's phase 1: merge in chunk order, publish the normalisers
  const ItemPart *pp = ws.part + it.row * a.nch;
  float GMd = kMFloor, GMc = kMFloor;
  for (int q = lane; q < a.nch; q += 32) {
    GMd = fmaxf(GMd, (float)__ldcg(&pp[q].md));
    GMc = fmaxf(GMc, (float)__ldcg(&pp[q].mc));
  }
  GMd = warp_max(GMd);
  GMc = warp_max(GMc);
  double L_d = 0.0, L_c = 0.0, W = 0.0;
  for (int q0 = 0; q0 < a.nch; q0 += 32) {
    double cl_d = 0.0, cl_c = 0.0, cw = 0.0;
    const int q = q0 + lane;
    if (q < a.nch) {
      const float rmd = (float)__ldcg(&pp[q].md), rmc = (float)__ldcg(&pp[q].mc);
      const double rld = __ldcg(&pp[q].ld), rlc = __ldcg(&pp[q].lc), rw = __ldcg(&pp[q].w);
      const float f_d = ex2((rmd - GMd) * cd), f_c = ex2((rmc - GMc) * cc);
      const float dl = (GMc - rmc) * cc - (GMd - rmd) * cd;
      double w_ = rw;
      if (rld > 0.0) w_ += rld * (double)dl;
      cl_d = rld * f_d;
      cl_c = rlc * f_c;
      cw = w_ * f_d;
    }
    const int m = min(32, a.nch - q0);
    for (int r = 0; r < m; ++r) {  // chunk order
      L_d += __shfl_sync(0xffffffffu, cl_d, r);
      L_c += __shfl_sync(0xffffffffu, cl_c, r);
      W += __shfl_sync(0xffffffffu, cw, r);
    }
  }
  if (lane == 0) {
    RowState *r = ws.rs + it.row;
    r->g[0] = GMd;
    r->g[1] = L_d;
    r->g[2] = GMc;
    r->g[3] = L_c;
    r->g[4] = W;
    const bool ok = L_d > 0.0 && L_c > 0.0 && L_d < 1e300 && L_c < 1e300 && GMd < FLT_MAX && GMc < FLT_MAX;
    r->lam[0] = ok ? (float)((double)GMd * cd + log2(L_d)) : __int_as_float(0x7fc00000);
    r->lam[1] = ok ? (float)((double)GMc * cc + log2(L_c)) : __int_as_float(0x7fc00000);
    __threadfence();
    st_release(ws.cnt1 + it.row, a.nch + 1);  // "merged" marker
  }
}

// Epilogue of one row (warp 0 of the CTA that completed the row's phase 2; fp64, independent
// pieces on separate lanes).  The draft-side outputs depend on the draft row alone.
template <typename T>
__device__ __noinline__ void epilogue(const ScoreArgs &a, const ScoreWs &ws, int64_t row) {
  const int lane = threadIdx.x & 31;
  const float cd = a.cd, cc = a.cc;
  const RowState *rsp = ws.rs + row;
  const float GMd = (float)__ldcg(&rsp->g[0]), GMc = (float)__ldcg(&rsp->g[2]);
  const double L_d = __ldcg(&rsp->g[1]), L_c = __ldcg(&rsp->g[3]), W = __ldcg(&rsp->g[4]);
  auto row_bits = [](double L, float M) {
    if (!(L == L) || !(L < 1e300) || !(M < FLT_MAX)) return 1; /*SV_ROW_NAN*/
    return (L > 0.0) ? 0 : 2;                                  /*SV_ROW_ALL_NEG_INF*/
  };
  const int d_st = row_bits(L_d, GMd), c_st = row_bits(L_c, GMc);
  const int32_t t = a.tok[row];
  const bool tok_ok = t >= 0 && t < a.V;
  int st = d_st | c_st | (tok_ok ? 0 : 4 /*SV_ROW_BAD_TOKEN*/);
  const int64_t b = row / a.k, i = row % a.k;
  // S partials in chunk order: lane-parallel loads, ordered shuffle sum
  double S = 0.0;
  for (int q0 = 0; q0 < a.nch; q0 += 32) {
    const int q = q0 + lane;
    const double sp = q < a.nch ? (double)__ldcg(ws.spart + row * a.nch + q) : 0.0;
    const int m = min(32, a.nch - q0);
    for (int r = 0; r < m; ++r) S += __shfl_sync(0xffffffffu, sp, r);
  }
  // lane 0: log2 p_d(t); lane 1: log2 p_c(t); lane 2: ln(L_d / L_c)
  double piece = 0.0;
  if (lane == 0 && !d_st && tok_ok) {
    const float x = Elem<T>::load(reinterpret_cast<const T *>(a.d) + b * a.d_sb + i * a.d_si + t);
    piece = (double)x * cd - (double)(GMd * cd) - log2(L_d);
  }
  if (lane == 1 && !st) {
    const float x = Elem<T>::load(reinterpret_cast<const T *>(a.c) + b * a.c_sb + i * a.c_si + t);
    piece = (double)x * cc - (double)(GMc * cc) - log2(L_c);
  }
  if (lane == 2 && !st) piece = log(L_d / L_c);
  const double argd = __shfl_sync(0xffffffffu, piece, 0);
  double piece2 = 0.0;  // lane 0: p_d(t); lane 1: p_c(t) / p_d(t)
  if (lane == 0 && !d_st && tok_ok) piece2 = exp2(argd);
  if (lane == 1 && !st) piece2 = exp2(piece - argd);
  const double pdt = __shfl_sync(0xffffffffu, piece2, 0);
  const double Ar = __shfl_sync(0xffffffffu, piece2, 1);
  const double lnr = __shfl_sync(0xffffffffu, piece, 2);
  if (!d_st && tok_ok && pdt == 0.0) st |= 8; /*SV_ROW_DRAFT_ZERO*/
  double A = 0.0, KL = 0.0;
  if (!st) {
    A = fmin(1.0, Ar);
    KL = 0.6931471805599453 * (W / L_d) - lnr;
    if (KL > 1e20) KL = __longlong_as_double(0x7ff0000000000000LL);  // p_c = 0 where p_d > 0
  }
  float phat = 0.f;
  if (!st && a.p_hat) {  // bin = number of interior edges strictly below the value (R9)
    const float Sf = (float)S, Af = (float)A;
    int si = 0, ai = 0;
    for (int j = lane + 1; j < a.n_s; j += 32) si += (a.s_edges[j] < Sf) ? 1 : 0;
    for (int j = lane + 1; j < a.n_a; j += 32) ai += (a.a_edges[j] < Af) ? 1 : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      si += __shfl_xor_sync(0xffffffffu, si, o);
      ai += __shfl_xor_sync(0xffffffffu, ai, o);
    }
    phat = a.cells[si * a.n_a + ai];
  }
  if (lane == 0) {
    const float nanf_ = __int_as_float(0x7fc00000);
    if (a.S) a.S[row] = st ? nanf_ : (float)S;
    if (a.A) a.A[row] = st ? nanf_ : (float)A;
    if (a.KL) a.KL[row] = st ? nanf_ : (float)KL;
    if (a.p_hat) a.p_hat[row] = phat;
    a.dm[row] = GMd;
    a.dl[row] = (d_st & 1) ? nanf_ : ((d_st & 2) ? 0.f : (float)L_d);
    a.dpt[row] = (d_st || !tok_ok) ? nanf_ : (float)pdt;
    if (a.status) a.status[row] = st;
    ws.cnt1[row] = 0;  // leave the counters zeroed for the next call
    ws.cnt2[row] = 0;
  }
}

template <typename T>
__device__ void phase2(const ScoreArgs &a, const ScoreWs &ws, const Item &it, const T *slot, BlockScratch &sh) {
  constexpr int EPU = Elem<T>::kPerUnit;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) {
    while (ld_acquire(ws.cnt1 + it.row) != a.nch + 1) __nanosleep(32);
#ifdef SV_TRACE
    if (g_trace) {
      const int64_t jj = it.row / ((gridDim.x) / a.nch) + 1;
      if (jj < 64) g_trace[((size_t)blockIdx.x * 64 + jj) * 5 + 3] = gtime();
    }
#endif
    const RowState *r = ws.rs + it.row;
    sh.lam[0] = __ldcg(&r->lam[0]);
    sh.lam[1] = __ldcg(&r->lam[1]);
  }
  __syncthreads();
  const float lamd = sh.lam[0], lamc = sh.lam[1];
  const float cd = a.cd, cc = a.cc;
  const Src<T> s = src_of<T>(a, it);
  const T *sd = slot, *sc = slot + a.chunk;
  float ssum = 0.f;
  if (lamd == lamd && lamc == lamc) {  // bad rows skip the S sweep
    const int units = s.bulk / EPU, e0 = units * EPU;
    const f2 cdd{cd, cd}, ccc{cc, cc}, ld2{-lamd, -lamd}, lc2{-lamc, -lamc};
    f2 acc{0.f, 0.f};
#pragma unroll
    for (int q = 0; q < UPT; ++q) {
      const int u = tid + q * NT;
      if (u < units) {
        const uint4 ud = reinterpret_cast<const uint4 *>(sd)[u], uc = reinterpret_cast<const uint4 *>(sc)[u];
        float xd[EPU], xc[EPU];
        Elem<T>::unit(ud, xd);
        Elem<T>::unit(uc, xc);
#pragma unroll
        for (int j = 0; j < EPU; j += 2) {
          const f2 ad = fma2(f2{xd[j], xd[j + 1]}, cdd, ld2), ac = fma2(f2{xc[j], xc[j + 1]}, ccc, lc2);
          acc = add2(acc, f2{ex2(fminf(ad.x, ac.x)), ex2(fminf(ad.y, ac.y))});
        }
      }
    }
    for (int e = e0 + tid; e < s.n; e += NT)
      acc.x += ex2(fminf(fmaf(Elem<T>::load(sd + e), cd, -lamd), fmaf(Elem<T>::load(sc + e), cc, -lamc)));
    ssum = acc.x + acc.y;
  }
  ssum = warp_sum(ssum);
  if (lane == 0) sh.fscr[wid] = ssum;
  __syncthreads();
  if (tid == 0) {
    float r = sh.fscr[0];
    for (int q = 1; q < NW; ++q) r += sh.fscr[q];
    ws.spart[it.row * a.nch + it.q] = r;
    __threadfence();
    sh.flag = atomicAdd(ws.cnt2 + it.row, 1) == a.nch - 1;
    if (sh.flag) __threadfence();  // acquire side: every chunk's S partial is visible
  }
  __syncthreads();
  if (sh.flag && wid == 0) epilogue<T>(a, ws, it.row);
}


template <typename T>
__global__ void __launch_bounds__(kScoreThreads, 2) sv_score_kernel(const ScoreArgs a, const int R) {
  __shared__ BlockScratch sh;
  extern __shared__ __align__(128) uint8_t smem[];
  T *ring = reinterpret_cast<T *>(smem);  // kScoreSlots x [draft chunk | companion chunk]
  const ScoreWs ws = carve(a);
  const Sched sc{(int64_t)a.B * a.k, a.nch, R};
  const int64_t waves = (sc.rows + R - 1) / R;
  auto slot = [&](int64_t j) { return ring + (size_t)(j % kScoreSlots) * 2 * a.chunk; };
  if (threadIdx.x == 0) {
    for (int s = 0; s < kScoreSlots; ++s) mbar_init(&sh.bar[s], 1);
    fence_mbar_init();
    const Item it0 = sc.item(0);
    if (it0.valid) issue<T>(a, it0, slot(0), &sh.bar[0]);
  }
  __syncthreads();
  for (int64_t j = 0; j <= waves; ++j) {
    const Item cur = sc.item(j), prev = sc.item(j - 1);
    if (threadIdx.x == 0) {  // prefetch the next wave's item (its slot held wave j - 2, done)
      const Item nxt = sc.item(j + 1);
      if (nxt.valid) issue<T>(a, nxt, slot(j + 1), &sh.bar[(j + 1) % kScoreSlots]);
    }
    TR(j, 0);
    if (cur.valid) {
      mbar_wait(&sh.bar[j % kScoreSlots], (uint32_t)((j / kScoreSlots) & 1));
      TR(j, 1);
      phase1<T>(a, ws, cur, slot(j), sh);
      TR(j, 2);
    }
    if (prev.valid) phase2<T>(a, ws, prev, slot(j - 1), sh);
    TR(j, 4);
  }
}

}  // namespace

cudaError_t launch_score(const ScoreArgs &a, cudaStream_t st) {
  const int elem = a.bf16 ? 2 : 4;
  const size_t smem = (size_t)kScoreSlots * 2 * a.chunk * elem;
  const void *fn = a.bf16 ? (const void *)sv_score_kernel<__nv_bfloat16> : (const void *)sv_score_kernel<float>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int64_t rows = (int64_t)a.B * a.k;
  int64_t grid = resident_grid(fn, kScoreThreads, (int)smem);  // co-resident: phase 2 waits on others
  // rows per wave: every chunk of a row is processed in the same wave
  int64_t R = grid / a.nch;
  if (R < 1) return cudaErrorInvalidConfiguration;  // V too large for the resident grid
  if (R > rows) R = rows;
  grid = R * a.nch;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kScoreThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // guarantees co-residency (or fails loudly)
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (a.bf16) return cudaLaunchKernelEx(&cfg, sv_score_kernel<__nv_bfloat16>, a, (int)R);
  return cudaLaunchKernelEx(&cfg, sv_score_kernel<float>, a, (int)R);
}

}  // namespace sv

#ifdef SV_TRACE
extern "C" __attribute__((visibility("default"))) int sv_debug_set_trace(void *buf) {
  return (int)cudaMemcpyToSymbol(sv::g_trace, &buf, sizeof(buf));
}
#endif
