// Microbenchmark: streaming-read ceilings on this B200 for the SV kernels' access patterns.
//   mode 0: plain read (sum of words)     mode 1: 1 ex2 per bf16 element (K4 / K5 math)
//   mode 2: 2 ex2 per element pair + w    mode 3: mode 2 + 1 ex2 per pair (K1's total MUFU load)
// Grid-stride LDG.128, U loads per tensor per thread in flight; T tensors read (1 or 2).
#include <cstdint>
#include <cstdio>
__device__ __forceinline__ float ex2(float x) { float y; asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ uint4 ldg(const void *p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
// exp2 on the FMA pipe: Cody-Waite split at the nearest integer (magic-number rounding), a
// degree-6 minimax-style Taylor polynomial of 2^f on [-0.5, 0.5], exponent by integer add.
__device__ __forceinline__ float ex2_poly(float x) {
  x = fmaxf(x, -126.f);
  const float t = x + 12582912.f;
  const float f = x - (t - 12582912.f);
  float p = 1.5403530e-4f;
  p = fmaf(p, f, 1.3333558e-3f);
  p = fmaf(p, f, 9.6181291e-3f);
  p = fmaf(p, f, 5.5504109e-2f);
  p = fmaf(p, f, 2.4022651e-1f);
  p = fmaf(p, f, 6.9314718e-1f);
  p = fmaf(p, f, 1.0f);
  return __int_as_float(__float_as_int(p) + ((__float_as_int(t) - 0x4B400000) << 23));
}
template <int MODE, int U, int NT>
__global__ void __launch_bounds__(256) k(const uint4 *__restrict__ d, const uint4 *__restrict__ c, size_t n, float *out) {
  float acc0 = 0.f, acc1 = 0.f, acc2 = 0.f;
  const size_t stride = (size_t)gridDim.x * blockDim.x * U;
  for (size_t i0 = (size_t)blockIdx.x * blockDim.x * U + threadIdx.x; i0 < n; i0 += stride) {
    uint4 a[U], b[U];
#pragma unroll
    for (int q = 0; q < U; ++q) {
      size_t i = i0 + (size_t)q * blockDim.x;
      if (i < n) { a[q] = ldg(d + i); if (NT == 2) b[q] = ldg(c + i); } else { a[q] = make_uint4(0, 0, 0, 0); b[q] = a[q]; }
    }
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const uint32_t wa[4] = {a[q].x, a[q].y, a[q].z, a[q].w};
      uint32_t wb[4] = {0, 0, 0, 0};
      if (NT == 2) { wb[0] = b[q].x; wb[1] = b[q].y; wb[2] = b[q].z; wb[3] = b[q].w; }
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        float x0 = __uint_as_float(wa[p] << 16), x1 = __uint_as_float(wa[p] & 0xffff0000u);
        float y0 = __uint_as_float(wb[p] << 16), y1 = __uint_as_float(wb[p] & 0xffff0000u);
        if (MODE == 0) { acc0 += x0 + x1; acc1 += y0 + y1; }
        if (MODE == 1) { acc0 += ex2(fmaf(x0, 1.44f, -3.f)) + ex2(fmaf(x1, 1.44f, -3.f)); if (NT == 2) acc1 += ex2(fmaf(y0, 1.44f, -3.f)) + ex2(fmaf(y1, 1.44f, -3.f)); }
        if (MODE >= 2) {
          float e0 = ex2(fmaf(x0, 1.44f, -3.f)), e1 = ex2(fmaf(x1, 1.44f, -3.f)), f0 = ex2(fmaf(y0, 1.44f, -3.f)), f1 = ex2(fmaf(y1, 1.44f, -3.f));
          acc0 += e0 + e1; acc1 += f0 + f1; acc2 = fmaf(e0, x0 - y0, fmaf(e1, x1 - y1, acc2));
        }
        if (MODE == 3) acc2 += ex2(fminf(fmaf(x0, 1.44f, -5.f), fmaf(y0, 1.44f, -5.f))) + ex2(fminf(fmaf(x1, 1.44f, -5.f), fmaf(y1, 1.44f, -5.f)));
        if (MODE == 4) acc2 += ex2_poly(fminf(fmaf(x0, 1.44f, -5.f), fmaf(y0, 1.44f, -5.f))) + ex2_poly(fminf(fmaf(x1, 1.44f, -5.f), fmaf(y1, 1.44f, -5.f)));
        if (MODE == 5) acc2 += ex2_poly(fminf(fmaf(x0, 1.44f, -5.f), fmaf(y0, 1.44f, -5.f))) + ex2(fminf(fmaf(x1, 1.44f, -5.f), fmaf(y1, 1.44f, -5.f)));
      }
    }
  }
  if (acc0 + acc1 + acc2 == 1234.5f) out[0] = acc0;
}
__global__ void acc_kernel(float *acc) {
  float e1 = 0.f, e2 = 0.f;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < 4000000; i += gridDim.x * blockDim.x) {
    const float x = -40.f * (float)i / 4000000.f;
    const double r = exp2((double)x);
    e1 = fmaxf(e1, (float)fabs((ex2_poly(x) - r) / r));
    e2 = fmaxf(e2, (float)fabs((ex2(x) - r) / r));
  }
  atomicMax((int *)&acc[0], __float_as_int(e1));
  atomicMax((int *)&acc[1], __float_as_int(e2));
}
// MUFU.EX2 throughput from registers (no memory): 8 independent chains per thread
__global__ void __launch_bounds__(256) mufu_kernel(float *out, int iters) {
  float v[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) v[j] = -0.001f * (threadIdx.x + j);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = ex2(v[j]) - 1.5f;
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += v[j];
  if (s == 1234.5f) out[0] = s;
}
#include <cstdlib>
int main() {
  const size_t big = (size_t)194584320;  // one of D / C at the headline (B=80, k=8, V=152064, bf16)
  uint4 *d, *c, *fl;
  float *out;
  cudaMalloc(&d, big); cudaMalloc(&c, big); cudaMalloc(&out, 64); cudaMalloc(&fl, 256 << 20);
  cudaMemset(d, 0x3f, big); cudaMemset(c, 0x3e, big);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](auto kern, const char *name, int blocks, size_t bytes, int nt) {
    size_t n = bytes / 16;
    float tot = 0;
    for (int r = 0; r < 6; ++r) {
      cudaMemsetAsync(fl, r, 256 << 20);  // flush L2
      cudaEventRecord(e0); kern<<<blocks, 256>>>(d, c, n, out); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (r) tot += ms;
    }
    float ms = tot / 5;
    printf("%-26s %6.1f MB x%d blocks %5d: %7.1f us  %6.0f GB/s\n", name, bytes / 1e6, nt, blocks, ms * 1e3, nt * bytes / ms / 1e6);
  };
  const size_t t86 = (size_t)86 << 20;  // ~ K4's target rows at mean gamma 2.5
  for (int bpsm : {4, 8}) {
    run(k<3, 4, 2>, "3 ex2/pair 2T U4", sms * bpsm, big, 2);
    run(k<4, 4, 2>, "2 ex2 + 1 poly /pair U4", sms * bpsm, big, 2);
    run(k<5, 4, 2>, "2.5 ex2 + .5 poly U4", sms * bpsm, big, 2);
  }
  {  // MUFU ex2 rate
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    const int iters = 4096, blocks = sms * 8;
    mufu_kernel<<<blocks, 256>>>(out, iters);
    cudaEventRecord(e0);
    mufu_kernel<<<blocks, 256>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = (double)blocks * 256 * iters * 8;
    printf("MUFU.EX2: %.3g ex2/s = %.2f per clk per SM at the %.0f MHz max clock (%.1f us)\n", ops / (ms * 1e-3),
           ops / (ms * 1e-3) / sms / (clk_khz * 1e3), clk_khz / 1e3, ms * 1e3);
  }
  // accuracy of ex2_poly vs exp2 over [-40, 0]
  {
    float *acc; cudaMallocManaged(&acc, 4 * sizeof(float));
    acc_kernel<<<256, 256>>>(acc);
    cudaDeviceSynchronize();
    printf("ex2_poly max rel err %.3g (vs exp2f), ex2.approx max rel err %.3g\n", acc[0], acc[1]);
  }
  if (getenv("CEIL_ONLY_POLY")) return 0;
  for (int bpsm : {2, 4, 8}) {
    run(k<0, 4, 1>, "read U4", sms * bpsm, t86, 1);
    run(k<0, 8, 1>, "read U8", sms * bpsm, t86, 1);
    run(k<1, 4, 1>, "1 ex2/elem U4", sms * bpsm, t86, 1);
    run(k<1, 8, 1>, "1 ex2/elem U8", sms * bpsm, t86, 1);
  }
  for (int bpsm : {2, 4, 8}) {
    run(k<0, 4, 2>, "read 2T U4", sms * bpsm, big, 2);
    run(k<2, 4, 2>, "2 ex2/pair 2T U4", sms * bpsm, big, 2);
    run(k<3, 4, 2>, "3 ex2/pair 2T U4", sms * bpsm, big, 2);
    run(k<3, 2, 2>, "3 ex2/pair 2T U2", sms * bpsm, big, 2);
  }
  for (int f : {1, 2, 4, 16, 64})
    run(k<0, 4, 1>, "read U4 grid/f", sms * 8 / f > 0 ? sms * 8 / f : 1, t86, 1);
}
