// Microbenchmark: the latency floor of a chain of dependent kernels in one CUDA graph (the SV
// step is 6 PDL-chained kernels + one torch kernel).  Each kernel: griddepcontrol.wait, then R
// dependent global round trips by thread 0 of block 0 (load x[i] -> store x[i+1]), then
// griddepcontrol.launch_dependents.  Reports us per graph replay for N kernels, with and without
// programmatic stream serialization (PDL), L2 warm (no flush).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void kern(unsigned *x, int R) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned v = 0;
    for (int r = 0; r < R; ++r) {
      v = *((volatile unsigned *)x + (v & 7));
      *((volatile unsigned *)x + 8 + r) = v + 1;
    }
  }
}
int main() {
  unsigned *x;
  cudaMalloc(&x, 4096);
  cudaMemset(x, 0, 4096);
  cudaStream_t s;
  cudaStreamCreate(&s);
  for (int pdl = 0; pdl < 2; ++pdl)
    for (int grid : {1, 148})
      for (int R : {0, 4})
        for (int N : {1, 2, 4, 7}) {
          cudaGraph_t g;
          cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
          for (int i = 0; i < N; ++i) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(grid);
            cfg.blockDim = dim3(256);
            cfg.stream = s;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = at;
            cfg.numAttrs = pdl;
            cudaLaunchKernelEx(&cfg, kern, x, R);
          }
          cudaStreamEndCapture(s, &g);
          cudaGraphExec_t ge;
          cudaGraphInstantiate(&ge, g, 0);
          for (int w = 0; w < 10; ++w) cudaGraphLaunch(ge, s);
          cudaEvent_t e0, e1;
          cudaEventCreate(&e0);
          cudaEventCreate(&e1);
          float tot = 0.f;
          for (int it = 0; it < 50; ++it) {
            cudaEventRecord(e0, s);
            cudaGraphLaunch(ge, s);
            cudaEventRecord(e1, s);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            tot += ms;
          }
          printf("pdl=%d grid=%3d R=%d N=%d: %6.2f us per replay\n", pdl, grid, R, N, tot / 50 * 1e3);
          cudaGraphExecDestroy(ge);
          cudaGraphDestroy(g);
        }
  return 0;
}
