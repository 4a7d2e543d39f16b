// sv_score_dev.cuh -- the device code of K1 (steps a1-a3): element arithmetic of both passes,
// block / row merges, the row epilogue (included by sv_score.cu, the K1 kernels).
#pragma once
#include <float.h>

#include "sv_device.cuh"
#include "sv_internal.h"

namespace sv {

namespace {

template <int NW>
struct Smem {
  double glob[5];  // merged (M_d, L_d, M_c, L_c, W)
  float lam[2];    // Lambda_d, Lambda_c
  float fscr[2 * NW];
  double dscr[5 * NW];  // per-warp pass-1 partials (ref_d, l_d, ref_c, l_c, w)
  double wglob[NW][5];  // P2: every warp merges the row's partials itself (no block barrier)
  float wlam[NW][2];
};

__device__ __forceinline__ uint4 ldg_hint(const void *p, uint64_t pol) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ void red_release_add(uint32_t *p, uint32_t v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t atom_add_acq_rel(uint32_t *p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Bounded: the producers are CTAs with lower linear indices (dispatched first), so the count is
// always reached unless the workspace invariant is broken (counters not zero at entry); then the
// kernel traps (a CUDA error the caller sees) instead of spinning forever.
__device__ __forceinline__ void wait_count(const uint32_t *p, uint32_t target) {
  for (uint32_t n = 0; ld_acquire(p) < target; ++n) {
    if (n > (1u << 26)) __trap();
    __nanosleep(100);
  }
}

// ---------------------------------------------------------------- element arithmetic
// Pass-1 output of one thread: sums of 2^{(x - r) c} (and the KL partial sum e_d (a_d - a_c))
// taken against the thread's references (r_d, r_c) in logit units.  Any references are exact
// for the merge (the block / row merges rescale by 2^{(r - M) c}); the pass only has to keep
// them close enough to the maxima that nothing overflows or vanishes.
struct P1Out {
  float rd, rc, ld, lc, w;
};

// Where this CTA's chunk of a row lives.
template <typename T>
struct Chunk {
  const T *d, *c;
  int n;      // elements
  int units;  // 16-byte units (0 when the chunk pair is not 16-byte aligned)
};
template <typename T>
__device__ __forceinline__ Chunk<T> chunk_of(const ScoreArgs &a, int64_t b, int64_t i, int rank) {
  const int64_t v0 = (int64_t)rank * a.chunk;
  Chunk<T> ch;
  ch.d = reinterpret_cast<const T *>(a.d) + b * a.d_sb + i * a.d_si + v0;
  ch.c = reinterpret_cast<const T *>(a.c) + b * a.c_sb + i * a.c_si + v0;
  ch.n = (int)max((int64_t)0, min(a.chunk, (int64_t)a.V - v0));
  const bool al = ((reinterpret_cast<uintptr_t>(ch.d) | reinterpret_cast<uintptr_t>(ch.c)) & 15) == 0;
  ch.units = al ? ch.n / Elem<T>::kPerUnit : 0;
  return ch;
}

// Sources of a chunk's 16-byte units: global memory (the vocab-sharded staging; L2 policy hint)
// or the CTA's shared-memory copy (K1: the chunk pair is bulk-copied once and read twice).
// Elements past the last whole unit (and the whole chunk when it is not 16-byte aligned) are
// always read from global memory through the Chunk pointers.
template <typename T>
struct GSrc {
  const T *d, *c;
  uint64_t pol;
  __device__ __forceinline__ uint4 ud(int u) const { return ldg_hint(d + (size_t)u * Elem<T>::kPerUnit, pol); }
  __device__ __forceinline__ uint4 uc(int u) const { return ldg_hint(c + (size_t)u * Elem<T>::kPerUnit, pol); }
};
struct SSrc {
  const uint4 *d, *c;  // shared memory
  __device__ __forceinline__ uint4 ud(int u) const { return d[u]; }
  __device__ __forceinline__ uint4 uc(int u) const { return c[u]; }
};

// The thread's first full group of a task's units, loaded ahead of time: a P2 task issues it
// before the merge of the row's P1 partials, and the persistent K1 issues the NEXT task's first
// group before the current task's tail (block merge / publish), so both latencies hide.
template <int G>
struct Pre {
  uint4 d[G], c[G];
  bool full;
};
template <typename T, int NT, int G, typename Src>
__device__ __forceinline__ void prefetch_first(const Src &src, const Chunk<T> &ch, Pre<G> &pre) {
  const int tid = threadIdx.x;
  pre.full = tid + (G - 1) * NT < ch.units;
  if (pre.full) {
#pragma unroll
    for (int q = 0; q < G; ++q) {
      pre.d[q] = src.ud(tid + q * NT);
      pre.c[q] = src.uc(tid + q * NT);
    }
  }
}

// ---- pass 1, fast path.  The thread's references are the maxima of its FIRST group (any value
// <= the true maximum keeps every term of the final sum >= 2^{-(max - r) c}, so nothing
// vanishes); no running maximum, no rescaling: a term can only overflow if a later logit
// exceeds the reference by ~88 / c nats, and then the sums are not finite and the thread redoes
// its share on the exact path below (also the path of NaN / +inf / masked inputs).
struct P1Fast {
  float rd, rc;
  f2 ld, lc, w;
};

template <typename T, int g>
__device__ __forceinline__ void fast_ref(P1Fast &t, const uint4 (&rd)[g], const uint4 (&rc)[g]) {
  float md = kMFloor, mc = kMFloor;
#pragma unroll
  for (int q = 0; q < g; ++q) {
    md = fmaxf(md, unit_max<T>(rd[q]));
    mc = fmaxf(mc, unit_max<T>(rc[q]));
  }
  t.rd = md;
  t.rc = mc;
}

// sums of one group of g units per tensor: 2 MUFU.EX2 per (d, c) pair, packed FFMA2 / FADD2
template <typename T, int g>
__device__ __forceinline__ void fast_group(P1Fast &t, const uint4 (&rd)[g], const uint4 (&rc)[g], f2 cdd, f2 ccc,
                                           f2 nrd, f2 nrc) {
  constexpr int EPU = Elem<T>::kPerUnit;
#pragma unroll
  for (int q = 0; q < g; ++q) {
    f2 xd[EPU / 2], xc[EPU / 2];
    unit_pairs<T>(rd[q], xd);
    unit_pairs<T>(rc[q], xc);
#pragma unroll
    for (int p = 0; p < EPU / 2; ++p) {
      const f2 ad = fma2(xd[p], cdd, nrd), ac = fma2(xc[p], ccc, nrc);
      const f2 ed = ex2x2(ad), ec = ex2x2(ac);
      t.ld = add2(t.ld, ed);
      t.lc = add2(t.lc, ec);
      t.w = fma2(ed, sub2(ad, ac), t.w);
    }
  }
}

// The thread's units u = tid + j NT in groups of G (all loads of a group issued together).
template <typename T, int NT, int G, typename Src>
__device__ __forceinline__ P1Fast pass1_fast(const Src &src, const Chunk<T> &ch, float cd, float cc,
                                             const Pre<G> *pre) {
  constexpr int EPU = Elem<T>::kPerUnit;
  const int tid = threadIdx.x;
  P1Fast t{kMFloor, kMFloor, {0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};
  const f2 cdd{cd, cd}, ccc{cc, cc};
  f2 nrd{0.f, 0.f}, nrc{0.f, 0.f};
  bool first = true;
  int u0 = tid;
  if (pre && pre->full) {
    fast_ref<T, G>(t, pre->d, pre->c);
    nrd = f2{-(t.rd * cd), -(t.rd * cd)};
    nrc = f2{-(t.rc * cc), -(t.rc * cc)};
    first = false;
    fast_group<T, G>(t, pre->d, pre->c, cdd, ccc, nrd, nrc);
    u0 += G * NT;
  }
  for (; u0 + (G - 1) * NT < ch.units; u0 += G * NT) {
    uint4 rd[G], rc[G];
#pragma unroll
    for (int q = 0; q < G; ++q) {
      rd[q] = src.ud(u0 + q * NT);
      rc[q] = src.uc(u0 + q * NT);
    }
    if (first) {
      fast_ref<T, G>(t, rd, rc);
      nrd = f2{-(t.rd * cd), -(t.rd * cd)};
      nrc = f2{-(t.rc * cc), -(t.rc * cc)};
      first = false;
    }
    fast_group<T, G>(t, rd, rc, cdd, ccc, nrd, nrc);
  }
  for (; u0 < ch.units; u0 += NT) {
    const uint4 rd[1] = {src.ud(u0)}, rc[1] = {src.uc(u0)};
    if (first) {
      fast_ref<T, 1>(t, rd, rc);
      nrd = f2{-(t.rd * cd), -(t.rd * cd)};
      nrc = f2{-(t.rc * cc), -(t.rc * cc)};
      first = false;
    }
    fast_group<T, 1>(t, rd, rc, cdd, ccc, nrd, nrc);
  }
  // element tail (< one unit; also the whole share of an unaligned chunk), from global memory
  const int e0 = ch.units * EPU;
  if (e0 + tid < ch.n) {
    if (first) {
      float md = kMFloor, mc = kMFloor;
      for (int e = e0 + tid; e < ch.n; e += NT) {
        md = fmaxf(md, Elem<T>::load(ch.d + e));
        mc = fmaxf(mc, Elem<T>::load(ch.c + e));
      }
      t.rd = md;
      t.rc = mc;
      nrd = f2{-(t.rd * cd), -(t.rd * cd)};
      nrc = f2{-(t.rc * cc), -(t.rc * cc)};
    }
    for (int e = e0 + tid; e < ch.n; e += NT) {
      const float ad = fmaf(Elem<T>::load(ch.d + e), cd, nrd.x), ac = fmaf(Elem<T>::load(ch.c + e), cc, nrc.x);
      const float ed = ex2(ad);
      t.ld.x += ed;
      t.lc.x += ex2(ac);
      t.w.x = fmaf(ed, ad - ac, t.w.x);
    }
  }
  return t;
}

// ---- pass 1, exact path (running maxima, lazy exact rescaling, guarded KL terms): the fallback
// of a thread whose fast sums are not finite.
struct P1State {
  float md, mc, rd, rc, ld, lc, w;
};
constexpr float kLazy = 8.f;

__device__ __forceinline__ void p1_rescale(P1State &t, float cd, float cc) {
  if ((t.md - t.rd) * cd > kLazy || (t.mc - t.rc) * cc > kLazy) {  // exact rescale to (md, mc)
    const float sdf = ex2((t.rd - t.md) * cd), scf = ex2((t.rc - t.mc) * cc);
    const float delta = (t.mc - t.rc) * cc - (t.md - t.rd) * cd;
    if (t.ld > 0.f) t.w = fmaf(t.ld, delta, t.w);
    t.w *= sdf;
    t.ld *= sdf;
    t.lc *= scf;
    t.rd = t.md;
    t.rc = t.mc;
  }
}

template <typename T>
__device__ __forceinline__ void exact_unit(P1State &t, const uint4 &ud, const uint4 &uc, float cd, float cc) {
  constexpr int EPU = Elem<T>::kPerUnit;
  t.md = fmaxf(t.md, unit_max<T>(ud));
  t.mc = fmaxf(t.mc, unit_max<T>(uc));
  p1_rescale(t, cd, cc);
  const float nmd = -t.rd * cd, nmc = -t.rc * cc;
  float xd[EPU], xc[EPU];
  Elem<T>::unit(ud, xd);
  Elem<T>::unit(uc, xc);
#pragma unroll
  for (int e = 0; e < EPU; ++e) {
    const float ad = fmaf(xd[e], cd, nmd), ac = fmaf(xc[e], cc, nmc);
    const float ed = ex2(ad);
    t.ld += ed;
    t.lc += ex2(ac);
    t.w += ed > 0.f ? ed * (ad - ac) : 0.f;  // p_d = 0 terms contribute 0 even against a_c = -inf
  }
}

template <typename T, int NT, typename Src>
__device__ __forceinline__ P1Out pass1_exact(const Src &src, const Chunk<T> &ch, float cd, float cc) {
  const int tid = threadIdx.x;
  P1State t{kMFloor, kMFloor, kMFloor, kMFloor, 0.f, 0.f, 0.f};
  for (int u = tid; u < ch.units; u += NT) exact_unit<T>(t, src.ud(u), src.uc(u), cd, cc);
  const int e0 = ch.units * Elem<T>::kPerUnit;
  for (int e = e0 + tid; e < ch.n; e += NT) {
    t.md = fmaxf(t.md, Elem<T>::load(ch.d + e));
    t.mc = fmaxf(t.mc, Elem<T>::load(ch.c + e));
  }
  p1_rescale(t, cd, cc);
  const float nmd = -t.rd * cd, nmc = -t.rc * cc;
  for (int e = e0 + tid; e < ch.n; e += NT) {
    const float ad = fmaf(Elem<T>::load(ch.d + e), cd, nmd), ac = fmaf(Elem<T>::load(ch.c + e), cc, nmc);
    const float ed = ex2(ad);
    t.ld += ed;
    t.lc += ex2(ac);
    t.w += ed > 0.f ? ed * (ad - ac) : 0.f;
  }
  return P1Out{t.rd, t.rc, t.ld, t.lc, t.w};  // sums against the (lazy) references
}

// The thread's pass-1 output: the fast path, or the exact path when its sums are not finite
// (overflow against the first-group reference, NaN / +inf logits, masked -inf terms in KL).
template <typename T, int NT, int G, typename Src>
__device__ __forceinline__ P1Out pass1_thread(const Src &src, const Chunk<T> &ch, float cd, float cc,
                                              const Pre<G> *pre = nullptr) {
  const P1Fast f = pass1_fast<T, NT, G>(src, ch, cd, cc, pre);
  const float ld = f.ld.x + f.ld.y, lc = f.lc.x + f.lc.y, w = f.w.x + f.w.y;
  if (ld < 1e36f && lc < 1e36f && w == w && fabsf(w) < 1e36f) return P1Out{f.rd, f.rc, ld, lc, w};
  return pass1_exact<T, NT>(src, ch, cd, cc);
}

// ---- pass 2: S_r = sum 2^{min(x_d c_d - Lambda_d, x_c c_c - Lambda_c)}, one exp per pair.
// A fixed NPOLY of every 4 packed pairs take 2^y on the FMA pipe (ex2_poly2: rel. err. ~2.4e-7,
// the MUFU's ~1.4e-7), the rest on the MUFU: the two pipes share the load.
template <typename T, int g, int NPOLY>
__device__ __forceinline__ void p2_group(f2 &acc, const uint4 (&rd)[g], const uint4 (&rc)[g], f2 cdd, f2 ccc, f2 nld,
                                         f2 nlc) {
  constexpr int EPU = Elem<T>::kPerUnit;
#pragma unroll
  for (int q = 0; q < g; ++q) {
    f2 xd[EPU / 2], xc[EPU / 2];
    unit_pairs<T>(rd[q], xd);
    unit_pairs<T>(rc[q], xc);
#pragma unroll
    for (int p = 0; p < EPU / 2; ++p) {
      const f2 ad = fma2(xd[p], cdd, nld), ac = fma2(xc[p], ccc, nlc);
      const f2 m{fminf(ad.x, ac.x), fminf(ad.y, ac.y)};
      const bool poly = (EPU == 8) ? (p < NPOLY) : (2 * p < NPOLY);
      acc = add2(acc, poly ? ex2_poly2(m) : ex2x2(m));
    }
  }
}

template <typename T, int NT, int G, int NPOLY, typename Src>
__device__ __forceinline__ float pass2_thread(const Src &src, const Chunk<T> &ch, float cd, float cc, float lamd,
                                              float lamc, const Pre<G> *pre = nullptr) {
  constexpr int EPU = Elem<T>::kPerUnit;
  const int tid = threadIdx.x;
  const f2 cdd{cd, cd}, ccc{cc, cc}, nld{-lamd, -lamd}, nlc{-lamc, -lamc};
  f2 acc{0.f, 0.f};
  int u0 = tid;
  if (pre && pre->full) {
    p2_group<T, G, NPOLY>(acc, pre->d, pre->c, cdd, ccc, nld, nlc);
    u0 += G * NT;
  }
  for (; u0 + (G - 1) * NT < ch.units; u0 += G * NT) {
    uint4 rd[G], rc[G];
#pragma unroll
    for (int q = 0; q < G; ++q) {
      rd[q] = src.ud(u0 + q * NT);
      rc[q] = src.uc(u0 + q * NT);
    }
    p2_group<T, G, NPOLY>(acc, rd, rc, cdd, ccc, nld, nlc);
  }
  for (; u0 < ch.units; u0 += NT) {
    const uint4 rd[1] = {src.ud(u0)}, rc[1] = {src.uc(u0)};
    p2_group<T, 1, NPOLY>(acc, rd, rc, cdd, ccc, nld, nlc);
  }
  for (int e = ch.units * EPU + tid; e < ch.n; e += NT)
    acc.x += ex2(fminf(fmaf(Elem<T>::load(ch.d + e), cd, -lamd), fmaf(Elem<T>::load(ch.c + e), cc, -lamc)));
  return acc.x + acc.y;
}

// Epilogue of one row (control warp of its epilogue CTA; independent pieces on separate lanes,
// fp64 range reduction + fp32 transcendentals).  The draft-side outputs depend on the draft row
// alone: a bad companion row does not poison them.
// S partials: entry j < G cs of this row is sarr[(j / cs) gstride + j % cs] (vocabulary order);
// xtok: NULL = load the token logits from the rows, else the owner's of xtok[g gstride2 + 0/1]
// over g (NaN = not owned; vocab-sharded staging).
// Inputs of a row's epilogue that do not depend on the passes (token, its logits, profile edges),
// loaded ahead by K1c's epilogue warp into shared memory (lane l's edges at [l]).
struct EpiPre {
  int32_t t;
  float x[2];
  float se[2][32], ae[2][32];
};
template <typename T>
__device__ __forceinline__ void epilogue_prefetch(const ScoreArgs &a, int64_t b, int64_t i, EpiPre &p) {
  const int lane = threadIdx.x & 31;
  const int32_t t = a.tok[b * a.k + i];
  const float inf = __int_as_float(0x7f800000);
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int j = lane + 1 + 32 * h;
    p.se[h][lane] = (a.p_hat && j < a.n_s) ? a.s_edges[j] : inf;
    p.ae[h][lane] = (a.p_hat && j < a.n_a) ? a.a_edges[j] : inf;
  }
  if (lane < 2) {
    float x = 0.f;
    if (t >= 0 && t < a.V)
      x = lane == 0 ? Elem<T>::load(reinterpret_cast<const T *>(a.d) + b * a.d_sb + i * a.d_si + t)
                    : Elem<T>::load(reinterpret_cast<const T *>(a.c) + b * a.c_sb + i * a.c_si + t);
    p.x[lane] = x;
  }
  if (lane == 0) p.t = t;
}

template <typename T>
__device__ __forceinline__ void epilogue(const ScoreArgs &a, int64_t b, int64_t i, const double *glob,
                                      const float *sarr, int cs, int G, int64_t gstride, const float *xtok,
                                      int64_t gstride2, const EpiPre *pre = nullptr, bool sarr_local = false) {
  const int64_t row = b * a.k + i;
  const int lane = threadIdx.x & 31;
  const float cd = a.cd, cc = a.cc;
  const float GMd = (float)glob[0], GMc = (float)glob[2];
  const double L_d = glob[1], L_c = glob[3], W = glob[4];
  auto row_bits = [](double L, float M) {
    if (!(L == L) || !(L < 1e300) || !(M < FLT_MAX)) return 1; /*SV_ROW_NAN*/
    return (L > 0.0) ? 0 : 2;                                  /*SV_ROW_ALL_NEG_INF*/
  };
  const int d_st = row_bits(L_d, GMd), c_st = row_bits(L_c, GMc);
  const int32_t t = pre ? pre->t : a.tok[row];
  const bool tok_ok = t >= 0 && t < a.V;
  int st = d_st | c_st | (tok_ok ? 0 : 4 /*SV_ROW_BAD_TOKEN*/);
  // profile edges j = lane + 1, lane + 33 (+inf past the end) -- loads issued early
  const float inf = __int_as_float(0x7f800000);
  float se[2], ae[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int j = lane + 1 + 32 * h;
    if (pre) {
      se[h] = pre->se[h][lane];
      ae[h] = pre->ae[h][lane];
    } else {
      se[h] = (a.p_hat && j < a.n_s) ? a.s_edges[j] : inf;
      ae[h] = (a.p_hat && j < a.n_a) ? a.a_edges[j] : inf;
    }
  }
  // lane 0: log2 p_d(t); lane 1: log2 p_c(t); lane 2: log2 L_d - log2 L_c; lane 3: S (rank order)
  double piece = 0.0;
  auto tok_logit = [&](int which) {  // 0 = draft, 1 = companion
    if (pre) return pre->x[which];
    if (!xtok) {
      return which == 0 ? Elem<T>::load(reinterpret_cast<const T *>(a.d) + b * a.d_sb + i * a.d_si + t)
                        : Elem<T>::load(reinterpret_cast<const T *>(a.c) + b * a.c_sb + i * a.c_si + t);
    }
    float x = __int_as_float(0x7fc00000);
    for (int g = 0; g < G; ++g) {
      const float v = __ldcg(xtok + g * gstride2 + which);
      if (x != x) x = v;
    }
    return x;
  };
  if (lane == 0 && !d_st && tok_ok) {
    const float x = tok_logit(0);
    piece = (double)x * cd - (double)(GMd * cd) - log2_acc(L_d);
  }
  if (lane == 1 && !st) {
    const float x = tok_logit(1);
    piece = (double)x * cc - (double)(GMc * cc) - log2_acc(L_c);
  }
  if (lane == 2 && !st) piece = log2_acc(L_d) - log2_acc(L_c);
  {  // S partials in blocks of 32 loaded in parallel (lane j: partial j0 + j), summed in order by lane 3
    const int ns = G * cs;
    for (int j0 = 0; j0 < ns; j0 += 32) {
      const int j = j0 + lane;
      const float *sp = sarr + (j / cs) * gstride + j % cs;
      const float v = j < ns ? (sarr_local ? *sp : __ldcg(sp)) : 0.f;  // local: shared memory (K1c)
      const int nr = min(32, ns - j0);
      for (int r = 0; r < nr; ++r) {
        const float x = __shfl_sync(0xffffffffu, v, r);
        if (lane == 3) piece += (double)x;
      }
    }
  }
  const double argd = __shfl_sync(0xffffffffu, piece, 0);
  double piece2 = 0.0;  // lane 0: p_d(t); lane 1: p_c(t) / p_d(t)
  if (lane == 0 && !d_st && tok_ok) piece2 = exp2_acc(argd);
  if (lane == 1 && !st) piece2 = exp2_acc(piece - argd);
  const double pdt = __shfl_sync(0xffffffffu, piece2, 0);
  const double Ar = __shfl_sync(0xffffffffu, piece2, 1);
  const double l2r = __shfl_sync(0xffffffffu, piece, 2);
  const double S = __shfl_sync(0xffffffffu, piece, 3);
  if (!d_st && tok_ok && pdt == 0.0) st |= 8; /*SV_ROW_DRAFT_ZERO*/
  double A = 0.0, KL = 0.0;
  if (!st) {
    A = fmin(1.0, Ar);
    KL = 0.6931471805599453 * (W / L_d - l2r);
    if (KL > 1e20) KL = __longlong_as_double(0x7ff0000000000000LL);  // p_c = 0 where p_d > 0
  }
  float phat = 0.f;
  if (!st && a.p_hat) {  // bin = number of interior edges strictly below the value (R9)
    const float Sf = (float)S, Af = (float)A;
    int si = (se[0] < Sf) + (se[1] < Sf), ai = (ae[0] < Af) + (ae[1] < Af);
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
  }
}

// Task t of the 2 * R * cs tasks (R = B * k rows; < 2^31): E = min(lag, R) * cs leading P1 tasks,
// then P1 and P2 tasks alternate, then the remaining P2 tasks.  Returns the chunk-task index q
// (row = q / cs) and whether it is a P2 task.
__device__ __forceinline__ void decode_task(uint32_t t, uint32_t RC, uint32_t E, uint32_t &q, bool &p2) {
  if (t < E) {
    q = t;
    p2 = false;
    return;
  }
  const uint32_t j = t - E, mid = 2 * (RC - E);
  if (j < mid) {
    p2 = (j & 1) != 0;
    q = p2 ? (j >> 1) : E + (j >> 1);
  } else {
    p2 = true;
    q = RC - E + (j - mid);
  }
}

// Where a chunk task sits: row, chunk rank, (b, i).
struct Task {
  uint32_t q, row, bb, ii;
  int rank;
  bool p2;
};

// Merge of a row's np P1 partials (vocabulary order) into sm.glob / sm.lam by one warp: lane l
// holds partials l, l + 32, ... (part(j) = partial j); global maxima first, then the sums in
// partial order (sequential over the lanes' shuffled values), so the bits depend on the
// partials only.  Shared by K1's P2, its epilogue and the vocab-sharded staging.
template <typename PartFn, bool kGlobal = true>
__device__ __forceinline__ void merge_partials_to(const ScoreArgs &a, int np, PartFn part_of, double (&glob)[5],
                                                  float (&lam)[2]) {
  auto ld = [](const double *p) { return kGlobal ? __ldcg(p) : *p; };  // global: through L2 (other CTAs')
  const int lane = threadIdx.x & 31;
  const float cd = a.cd, cc = a.cc;
  float GMd = kMFloor, GMc = kMFloor;
  for (int j0 = 0; j0 < np; j0 += 32) {
    float md = kMFloor, mc = kMFloor;
    if (j0 + lane < np) {
      const double *part = part_of(j0 + lane);
      md = (float)ld(part + 0);
      mc = (float)ld(part + 2);
    }
    GMd = fmaxf(GMd, warp_max(md));
    GMc = fmaxf(GMc, warp_max(mc));
  }
  double L_d = 0.0, L_c = 0.0, W = 0.0;
  for (int j0 = 0; j0 < np; j0 += 32) {
    double pr[5] = {kMFloor, 0.0, kMFloor, 0.0, 0.0};
    if (j0 + lane < np) {
      const double *part = part_of(j0 + lane);
#pragma unroll
      for (int j = 0; j < 5; ++j) pr[j] = ld(part + j);
    }
    const float rmd = (float)pr[0], rmc = (float)pr[2];
    const float sdf = ex2((rmd - GMd) * cd), scf = ex2((rmc - GMc) * cc);
    const float delta = (GMc - rmc) * cc - (GMd - rmd) * cd;
    double ww = pr[4];
    if (pr[1] > 0.0) ww += pr[1] * (double)delta;
    const double cl_d = pr[1] * sdf, cl_c = pr[3] * scf, cw = ww * sdf;
    const int nr = min(32, np - j0);
    for (int r = 0; r < nr; ++r) {  // partial order
      L_d += __shfl_sync(0xffffffffu, cl_d, r);
      L_c += __shfl_sync(0xffffffffu, cl_c, r);
      W += __shfl_sync(0xffffffffu, cw, r);
    }
  }
  if (lane == 0) {
    glob[0] = GMd;
    glob[1] = L_d;
    glob[2] = GMc;
    glob[3] = L_c;
    glob[4] = W;
    const bool ok = L_d > 0.0 && L_c > 0.0 && L_d < 1e300 && L_c < 1e300 && GMd < FLT_MAX && GMc < FLT_MAX;
    lam[0] = ok ? (float)((double)GMd * cd + log2_acc(L_d)) : __int_as_float(0x7fc00000);
    lam[1] = ok ? (float)((double)GMc * cc + log2_acc(L_c)) : __int_as_float(0x7fc00000);
  }
}
template <int NW, typename PartFn>
__device__ __forceinline__ void merge_partials(const ScoreArgs &a, int np, PartFn part_of, Smem<NW> &sm) {
  merge_partials_to(a, np, part_of, sm.glob, sm.lam);
}

// P1 tail: block merge of the threads' pass-1 states (fixed warp / lane order), the last warp
// publishes (M_d, L_d, M_c, L_c, W) and bumps the row counter (release).  All NW warps call it.
// P1 tail: block merge of the threads' pass-1 outputs (fixed warp / lane order), the last warp
// publishes (M_d, L_d, M_c, L_c, W) and bumps the row counter (release).  All NW warps call both
// halves; the first ends with a block barrier (the persistent K1 issues the next task's first
// loads between the two).
// The warp's pass-1 partial (M_d, L_d, M_c, L_c, W) against the warp's maxima of the lanes'
// references (fp64 butterfly sums); lane 0 writes it to dst.
__device__ __forceinline__ void warp_p1_partial(const P1Out &t, float cd, float cc, double *dst) {
  const int lane = threadIdx.x & 31;
  const float Mw = warp_max(t.rd), Mcw = warp_max(t.rc);
  const float sdf = ex2((t.rd - Mw) * cd), scf = ex2((t.rc - Mcw) * cc);
  const float delta = (Mcw - t.rc) * cc - (Mw - t.rd) * cd;
  double ww = t.w;
  if (t.ld > 0.f) ww += (double)t.ld * (double)delta;
  const double v0 = warp_sum_d((double)t.ld * sdf), v1 = warp_sum_d((double)t.lc * scf), v2 = warp_sum_d(ww * sdf);
  if (lane == 0) {
    dst[0] = Mw;
    dst[1] = v0;
    dst[2] = Mcw;
    dst[3] = v1;
    dst[4] = v2;
  }
}
template <int NW>
__device__ __forceinline__ void p1_publish_head(const P1Out &t, Smem<NW> &sm, float cd, float cc) {
  // warp partial against the warp's maxima of the references (fp64 butterfly sums), one barrier
  warp_p1_partial(t, cd, cc, sm.dscr + 5 * (threadIdx.x >> 5));
  __syncthreads();
}
template <int NW>
__device__ __forceinline__ void p1_publish_tail(const ScoreArgs &a, const Task &k, Smem<NW> &sm) {
  // the last warp merges the NW warp partials in warp order (the row merge's arithmetic) and
  // publishes the chunk's (M_d, L_d, M_c, L_c, W)
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (wid != NW - 1) return;
  auto warp_part = [&](int j) { return (const double *)(sm.dscr + 5 * j); };
  merge_partials_to<decltype(warp_part), false>(a, NW, warp_part, sm.glob, sm.lam);
  __syncwarp();
  if (lane == 0) {
    double *part = a.part + (size_t)k.q * 5;
#pragma unroll
    for (int j = 0; j < 5; ++j) part[j] = sm.glob[j];
    if (a.cnt) red_release_add(a.cnt + 2 * (size_t)k.row, 1u);
  }
}
template <int NW>
__device__ __forceinline__ void p1_publish(const ScoreArgs &a, const Task &k, const P1Out &t, Smem<NW> &sm) {
  p1_publish_head<NW>(t, sm, a.cd, a.cc);
  p1_publish_tail<NW>(a, k, sm);
}

template <int NW>
__device__ __forceinline__ void p2_merge(const ScoreArgs &a, const Task &k, Smem<NW> &sm) {
  wait_count(a.cnt + 2 * (size_t)k.row, (uint32_t)a.cs);  // every lane acquires
  merge_partials<NW>(a, a.cs, [&](int j) { return a.part + ((size_t)k.row * a.cs + j) * 5; }, sm);
}
// Every warp of a P2 task merges the row's P1 partials itself (identical bits: the same loads and
// operations), so no warp waits at a block barrier for another warp's merge; returns Lambda.
template <int NW>
__device__ __forceinline__ float2 p2_merge_warp(const ScoreArgs &a, const Task &k, Smem<NW> &sm) {
  const int wid = threadIdx.x >> 5;
  wait_count(a.cnt + 2 * (size_t)k.row, (uint32_t)a.cs);  // every lane acquires
  merge_partials_to(a, a.cs, [&](int j) { return a.part + ((size_t)k.row * a.cs + j) * 5; }, sm.wglob[wid],
                    sm.wlam[wid]);
  __syncwarp();
  return make_float2(sm.wlam[wid][0], sm.wlam[wid][1]);
}

// P2 tail: block sum of the S partials, publish; the row's LAST P2 task to finish (elected by an
// acq_rel counter) runs the epilogue -- S in chunk order, so the bits do not depend on which task
// that is -- and re-arms the row's counters.  All NW warps call it.
template <int NW>
__device__ __forceinline__ void p2_finish_head(float s_loc, Smem<NW> &sm) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  s_loc = warp_sum(s_loc);
  if (lane == 0) sm.fscr[wid] = s_loc;
  __syncthreads();
}
template <typename T, int NW>
__device__ __forceinline__ void p2_finish_tail(const ScoreArgs &a, const Task &k, Smem<NW> &sm) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, cs = a.cs;
  if (wid != NW - 1) return;
  uint32_t *cnt = a.cnt + 2 * (size_t)k.row;
  float *srow = a.spart + (size_t)k.row * cs;
  uint32_t old = 0;
  if (lane == 0) {
    float r = sm.fscr[0];
    for (int w = 1; w < NW; ++w) r += sm.fscr[w];
    srow[k.rank] = r;
    old = atom_add_acq_rel(cnt + 1, 1u);  // releases this S partial, acquires the others
  }
  old = __shfl_sync(0xffffffffu, old, 0);
  if (old != (uint32_t)(cs - 1)) return;
  __syncwarp();
  fence_acq_rel();  // every lane: the other tasks' S partials are visible
  epilogue<T>(a, k.bb, k.ii, sm.wglob[NW - 1], srow, cs, 1, 0, nullptr, 0);
  if (lane == 0) {
    cnt[0] = 0u;  // every P1 / P2 task of this row is past its use of the counters
    cnt[1] = 0u;
  }
}

// A task's place: decoded ticket, chunk pointers and its unit source with the pass's L2 policy.
template <typename T>
struct TaskView {
  Task k;
  Chunk<T> ch;
  GSrc<T> src;
};
template <typename T>
__device__ __forceinline__ TaskView<T> task_view(const ScoreArgs &a, uint32_t t) {
  TaskView<T> v;
  const uint32_t cs = (uint32_t)a.cs, RC = (uint32_t)a.B * (uint32_t)a.k * cs;
  decode_task(t, RC, (uint32_t)a.lead, v.k.q, v.k.p2);
  v.k.row = v.k.q / cs;
  v.k.rank = (int)(v.k.q - v.k.row * cs);
  v.k.bb = v.k.row / (uint32_t)a.k;
  v.k.ii = v.k.row - v.k.bb * a.k;
  v.ch = chunk_of<T>(a, v.k.bb, v.k.ii, v.k.rank);
  // P1 reads HBM and keeps the chunk for P2 (evict_last); P2 is the chunk's last use
  v.src = GSrc<T>{v.ch.d, v.ch.c, v.k.p2 ? l2_policy_evict_first() : l2_policy_evict_last()};
  return v;
}

}  // namespace
}  // namespace sv
