// microbenchmark: L2-resident read bandwidth vs HBM read bandwidth on this GPU
#include <cstdio>
#include <cstdint>
__global__ void rd(const uint4* __restrict__ p, size_t n, int reps, uint4* out) {
  uint4 acc = make_uint4(0,0,0,0);
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
      uint4 v = __ldcg(p + i);
      acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
    }
  if (acc.x == 0x12345 && acc.y == 7) out[0] = acc;
}
int main() {
  size_t sizes[] = {(size_t)16 << 20, (size_t)48 << 20, (size_t)96 << 20, (size_t)2048 << 20};
  uint4* buf; cudaMalloc(&buf, (size_t)2048 << 20); cudaMemset(buf, 1, (size_t)2048 << 20);
  uint4* out; cudaMalloc(&out, 64);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (size_t bytes : sizes) {
    size_t n = bytes / 16; int reps = bytes >= ((size_t)1 << 30) ? 2 : 20;
    rd<<<sms * 4, 512>>>(buf, n, 1, out);
    cudaEventRecord(a); rd<<<sms * 4, 512>>>(buf, n, reps, out); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("%6zu MB x%d: %.1f GB/s\n", bytes >> 20, reps, (double)bytes * reps / ms / 1e6);
  }
}
