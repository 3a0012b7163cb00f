// FP64 pipe micro-benchmark: throughput of dependent DFMA chains as a
// function of independent chains per thread (ILP) and resident warps per
// SMSP, plus DADD-only and a shuffle-reduction mix.  Standalone:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_ilp fp64_ilp.cu && ./fp64_ilp
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP, int KIND>
__global__ void k(double* out, int iters, double a, double b) {
  double v[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) v[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int rep = 0; rep < 8; ++rep)
#pragma unroll
      for (int i = 0; i < ILP; ++i) {
        if (KIND == 0) v[i] = fma(v[i], a, b);
        else if (KIND == 1) v[i] = v[i] + b;
        else v[i] = v[i] * a;
      }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += v[i];
  if (s == 12345.0) out[0] = s;
}

template <int ILP, int KIND>
void run(int warps_per_smsp) {
  const int sms = 148, threads = 128;   // 4 warps per CTA = 1 per SMSP
  const int blocks = sms * warps_per_smsp;
  double* out;
  cudaMalloc(&out, 8);
  const int iters = 2048;
  k<ILP, KIND><<<blocks, threads>>>(out, 16, 1.0000001, 1e-9);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<ILP, KIND><<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double ops = (double)blocks * threads * iters * 8 * ILP;   // FP64 instructions (lane ops)
  const double flop = ops * (KIND == 0 ? 2 : 1);
  printf("kind %d ilp %2d warps/smsp %d: %.2f Tops/s (%.1f TFLOP/s)\n", KIND, ILP, warps_per_smsp,
         ops / (ms * 1e-3) / 1e12, flop / (ms * 1e-3) / 1e12);
  cudaFree(out);
}

int main() {
  for (int w : {1, 2, 3, 4, 8}) {
    run<1, 0>(w);
    run<2, 0>(w);
    run<4, 0>(w);
    run<8, 0>(w);
  }
  for (int w : {1, 2, 4}) {
    run<4, 1>(w);
    run<4, 2>(w);
  }
  return 0;
}
