// sv_device.cuh -- device-side helpers of libsv (sm_100a): MUFU exp2, bf16 unpacking, warp/block reductions, Philox4x32-10.
// Product code only; shares nothing with oracle/.
#pragma once

#include <cooperative_groups.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace sv {

namespace cg = cooperative_groups;

constexpr float kLog2e = 1.4426950408889634f;
// Floor for running maxima.  Starting at -1e30 instead of -inf keeps every exponent
// argument finite: a -inf logit gives ex2(-inf) = 0 and an all -inf row ends with l = 0
// (flagged SV_ROW_ALL_NEG_INF) instead of producing (-inf) - (-inf) = NaN.
constexpr float kMFloor = -1.0e30f;

// ---------------------------------------------------------------- math
__device__ __forceinline__ float ex2(float x) {  // MUFU.EX2, rel. err ~2^-22
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Short-latency fp64 log2 / exp2 for the per-row epilogues: exact range reduction in fp64, the
// transcendental of the reduced argument in fp32 (|error| ~1.5e-7 absolute for log2, ~1.2e-7
// relative for exp2 -- far below the 1e-6 decision tie band), instead of the long dependent
// DFMA chains of the fp64 library routines.
__device__ __forceinline__ double log2_acc(double L) {  // L > 0, finite
  int e;
  const double m = frexp(L, &e);  // m in [0.5, 1)
  return (double)e + (double)log2f((float)m);
}
__device__ __forceinline__ double exp2_acc(double a) {  // 2^a; -inf -> 0, +inf / NaN pass through
  if (!(a > -1100.0) || !(a < 1100.0)) return (a > 0.0 || a != a) ? a + 2048.0 : 0.0;
  const double n = floor(a);
  return ldexp((double)exp2f((float)(a - n)), (int)n);
}

// ---- packed fp32x2 arithmetic (sm_100a FFMA2 / FADD2 / FMUL2: two lanes per instruction)
struct f2 {
  float x, y;
};
__device__ __forceinline__ uint64_t f2_bits(f2 a) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a.x), "f"(a.y));
  return r;
}
__device__ __forceinline__ f2 f2_from(uint64_t b) {
  f2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(b));
  return r;
}
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(f2_bits(a)), "l"(f2_bits(b)), "l"(f2_bits(c)));
  return f2_from(r);
}
__device__ __forceinline__ f2 add2(f2 a, f2 b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2_bits(a)), "l"(f2_bits(b)));
  return f2_from(r);
}
__device__ __forceinline__ f2 sub2(f2 a, f2 b) {
  uint64_t r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2_bits(a)), "l"(f2_bits(b)));
  return f2_from(r);
}
__device__ __forceinline__ f2 mul2(f2 a, f2 b) {
  uint64_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2_bits(a)), "l"(f2_bits(b)));
  return f2_from(r);
}
__device__ __forceinline__ f2 ex2x2(f2 a) { return f2{ex2(a.x), ex2(a.y)}; }

// 2^y for a packed pair on the FMA pipe (no MUFU): y clamped to >= -127, j = round(y) by the
// 1.5 * 2^23 magic (biased by 127, so the low mantissa bits of t ARE the exponent field of 2^j),
// f = y - j in [-0.5, 0.5], p(f) = degree-5 minimax polynomial of 2^f (max rel. error 7.5e-8 in
// exact arithmetic, 2.4e-7 with fp32 Horner), times 2^j built by a shift.  y <= -127 gives
// exactly 0 (2^j's bits are then 0), like MUFU.EX2.FTZ for such arguments.  Valid for y <= 127.
__device__ __forceinline__ f2 ex2_poly2(f2 y) {
  y.x = fmaxf(y.x, -127.f);
  y.y = fmaxf(y.y, -127.f);
  const f2 M{12583039.f, 12583039.f};  // 1.5 * 2^23 + 127
  const f2 t = add2(y, M);
  const f2 f = sub2(y, sub2(t, M));
  f2 p = fma2(f2{1.3276472e-3f, 1.3276472e-3f}, f, f2{9.6755410e-3f, 9.6755410e-3f});
  p = fma2(p, f, f2{5.5507131e-2f, 5.5507131e-2f});
  p = fma2(p, f, f2{2.4022120e-1f, 2.4022120e-1f});
  p = fma2(p, f, f2{6.9314694e-1f, 6.9314694e-1f});
  p = fma2(p, f, f2{1.0000001f, 1.0000001f});
  const f2 sc{__uint_as_float(__float_as_uint(t.x) << 23), __uint_as_float(__float_as_uint(t.y) << 23)};
  return mul2(p, sc);
}

// bf16 pair packed in a 32-bit word -> two floats (exact)
__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }

template <typename T> struct Elem;
template <> struct Elem<float> {
  static constexpr int kPerUnit = 4;  // elements per 16-byte unit
  __device__ static float load(const float *p) { return *p; }
  __device__ static void unit(const uint4 &u, float (&x)[4]) {
    x[0] = __uint_as_float(u.x); x[1] = __uint_as_float(u.y);
    x[2] = __uint_as_float(u.z); x[3] = __uint_as_float(u.w);
  }
};
template <> struct Elem<__nv_bfloat16> {
  static constexpr int kPerUnit = 8;
  __device__ static float load(const __nv_bfloat16 *p) {
    return __uint_as_float(((uint32_t) * reinterpret_cast<const uint16_t *>(p)) << 16);
  }
  __device__ static void unit(const uint4 &u, float (&x)[8]) {
    x[0] = bf_lo(u.x); x[1] = bf_hi(u.x); x[2] = bf_lo(u.y); x[3] = bf_hi(u.y);
    x[4] = bf_lo(u.z); x[5] = bf_hi(u.z); x[6] = bf_lo(u.w); x[7] = bf_hi(u.w);
  }
};

// one 16-byte unit -> packed element pairs (exact)
template <typename T>
__device__ __forceinline__ void unit_pairs(const uint4 &u, f2 (&x)[Elem<T>::kPerUnit / 2]) {
  if constexpr (sizeof(T) == 2) {
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int p = 0; p < 4; ++p) x[p] = f2{bf_lo(w[p]), bf_hi(w[p])};
  } else {
    x[0] = f2{__uint_as_float(u.x), __uint_as_float(u.y)};
    x[1] = f2{__uint_as_float(u.z), __uint_as_float(u.w)};
  }
}

// max of one 16-byte unit straight from the packed bits (bf16x2 HMNMX2 is exact)
__device__ __forceinline__ float unit_max_bf16(const uint4 &v) {
  const __nv_bfloat162 *p = reinterpret_cast<const __nv_bfloat162 *>(&v);
  const __nv_bfloat162 m = __hmax2(__hmax2(p[0], p[1]), __hmax2(p[2], p[3]));
  return fmaxf(__low2float(m), __high2float(m));
}
template <typename T>
__device__ __forceinline__ float unit_max(const uint4 &v) {
  if constexpr (sizeof(T) == 2) {
    return unit_max_bf16(v);
  } else {
    return fmaxf(fmaxf(__uint_as_float(v.x), __uint_as_float(v.y)), fmaxf(__uint_as_float(v.z), __uint_as_float(v.w)));
  }
}

// ---------------------------------------------------------------- L2 cache policies
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// ---------------------------------------------------------------- mbarrier + bulk copy (TMA engine)
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {  // release (CTA scope)
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Bounded wait: a broken invariant traps (a CUDA error the caller sees) instead of hanging.
__device__ __forceinline__ void mbar_wait_bounded(uint64_t *bar, uint32_t parity) {
  for (uint32_t n = 0; !mbar_try_wait(bar, parity); ++n)
    if (n > (1u << 24)) __trap();
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// 1-D bulk copy global -> this CTA's shared memory through the TMA engine, completion counted
// in bytes on `bar`, with an L2 cache policy.  dst, src 16-byte aligned; bytes a multiple of 16.
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], "
      "%4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

// orders this thread's (and, after a warp / CTA barrier, its peers') generic-proxy shared-memory
// accesses before subsequent async-proxy (bulk copy) accesses
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// the same without an L2 cache hint
__device__ __forceinline__ void bulk_g2s_plain(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// streaming 16-byte global load (read once: do not allocate in L1)
__device__ __forceinline__ uint4 ldg_stream(const void *p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// ---------------------------------------------------------------- programmatic dependent launch
// Every libsv kernel is launched with programmatic stream serialization (PDL): it may start
// while the previous kernel on the stream drains, so it first waits for that grid's completion
// and memory flush (a no-op when launched without the attribute), then lets its own dependent
// launch as early as possible.  Nothing is read from global memory before pdl_wait().
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ---------------------------------------------------------------- experiment-only kernel trace
// SV_EXP_TRACE builds (scripts/trace_step.py) record, per kernel slot k, the earliest start and
// the latest warp exit (%globaltimer, ns) in a per-translation-unit device array read back by
// sv_debug_trace_<tu>(); the product build compiles none of it.
#ifndef SV_EXP_TRACE
#define SV_EXP_TRACE 0
#endif
#if SV_EXP_TRACE
__device__ __forceinline__ unsigned long long sv_gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define SV_TRACE_DECL static __device__ unsigned long long g_sv_trace[32];
#define SV_TRACE_START(k) \
  do {                    \
    if (threadIdx.x == 0) atomicMin(&g_sv_trace[2 * (k)], sv_gtimer()); \
  } while (0)
#define SV_TRACE_END(k) \
  do {                  \
    if ((threadIdx.x & 31) == 0) atomicMax(&g_sv_trace[2 * (k) + 1], sv_gtimer()); \
  } while (0)
#define SV_TRACE_POINT(k) \
  do {                    \
    if (threadIdx.x == 0 && blockIdx.x == 0) g_sv_trace[2 * (k)] = g_sv_trace[2 * (k) + 1] = sv_gtimer(); \
  } while (0)
#define SV_TRACE_POINT_ANY(k) \
  do {                        \
    g_sv_trace[2 * (k)] = g_sv_trace[2 * (k) + 1] = sv_gtimer(); \
  } while (0)
#define SV_TRACE_READER(name)                                                              \
  extern "C" __attribute__((visibility("default"))) int sv_debug_trace_##name(unsigned long long *out) { \
    unsigned long long init[32];                                                           \
    for (int i = 0; i < 32; ++i) init[i] = (i & 1) ? 0ull : ~0ull;                         \
    if (out && cudaMemcpyFromSymbol(out, sv::g_sv_trace, sizeof(init)) != cudaSuccess) return 1; \
    return cudaMemcpyToSymbol(sv::g_sv_trace, init, sizeof(init)) != cudaSuccess;          \
  }
#else
#define SV_TRACE_DECL
#define SV_TRACE_START(k) \
  do {                    \
  } while (0)
#define SV_TRACE_END(k) \
  do {                  \
  } while (0)
#define SV_TRACE_POINT(k) \
  do {                    \
  } while (0)
#define SV_TRACE_POINT_ANY(k) \
  do {                        \
  } while (0)
#define SV_TRACE_READER(name)
#endif

// ---------------------------------------------------------------- reductions
// Fixed butterfly order: the result depends only on the lane -> value mapping.
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
// inclusive prefix sum over lanes (Kogge-Stone, fixed order)
__device__ __forceinline__ double warp_incl_scan_d(double v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    double t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

// Block-wide reductions; `scratch` holds >= NT/32 floats.  Warp partials are combined
// in warp order by every thread, so all threads return the same bits.
template <int NT>
__device__ __forceinline__ float block_max(float v, float *scratch) {
  constexpr int NW = NT / 32;
  v = warp_max(v);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) scratch[w] = v;
  __syncthreads();
  float r = scratch[0];
#pragma unroll
  for (int i = 1; i < NW; ++i) r = fmaxf(r, scratch[i]);
  return r;
}
// ---------------------------------------------------------------- Philox4x32-10
// Salmon et al., SC'11.  counter = (i, global seq, lo(offset), hi(offset)),
// key = (lo(seed), hi(seed)) (DESIGN R12).
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += 0x9E3779B9u;
    k.y += 0xBB67AE85u;
  }
  return c;
}
__device__ __forceinline__ uint4 sv_philox(uint64_t seed, uint64_t offset, int64_t gseq, int32_t i) {
  return philox4x32_10(make_uint4((uint32_t)i, (uint32_t)gseq, (uint32_t)offset, (uint32_t)(offset >> 32)),
                       make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
}
// U24(w) = (w >> 8) * 2^-24, exact in fp32 and fp64
__device__ __forceinline__ double u24(uint32_t w) { return (double)(w >> 8) * (1.0 / 16777216.0); }

}  // namespace sv
