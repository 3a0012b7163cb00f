// Where one iteration of the resident per-chain CG (k_cg_resblk, 16^2) spends
// its cycles: thread 0 of every CTA reads the SM clock at ten points of the
// iteration (RES_STAMP in csrc/resident_col.cuh) and the per-phase sums are
// averaged over CTAs and iterations, for one chain alone, one per SM, one
// wave (4 per SM) and 8192 chains.  Standalone (run on the GPU box):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1512_03812_b200/csrc \
//        -o /tmp/resblk_phases tools/micro/resblk_phases.cu && /tmp/resblk_phases
// The stamps cost a few registers and the compiler may move arithmetic across
// them: read the numbers as a profile, not as exact boundaries.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

__device__ unsigned long long g_phase[12];
__device__ unsigned long long g_iters;

#ifdef NOSTAMP   // -DNOSTAMP: timing only, the kernel as the library builds it
#define RES_STAMP_BEGIN()
#define RES_STAMP(i)
#define RES_STAMP_END(iters)
#else
#define RES_STAMP_BEGIN()                 \
  __shared__ unsigned int ph_acc[12];     \
  unsigned int ph_last = 0;               \
  if (threadIdx.x == 0) {                 \
    for (int i_ = 0; i_ < 12; ++i_) ph_acc[i_] = 0; \
    ph_last = (unsigned int)clock();      \
  }
#define RES_STAMP(i)                      \
  if (threadIdx.x == 0) {                 \
    const unsigned int c_ = (unsigned int)clock(); \
    ph_acc[i] += c_ - ph_last;            \
    ph_last = c_;                         \
  }
#define RES_STAMP_END(iters)              \
  if (threadIdx.x == 0) {                 \
    for (int i_ = 0; i_ < 12; ++i_) atomicAdd(&g_phase[i_], (unsigned long long)ph_acc[i_]); \
    atomicAdd(&g_iters, (unsigned long long)(iters)); \
  }

#endif

#include "resident_col.cuh"

int main() {
  const int L = 16, V = L * L, maxB = 8192, iters = 200;
  std::vector<double> hU((size_t)maxB * 2 * V * 2), hb((size_t)maxB * V * 4);
  srand(1);
  for (size_t i = 0; i < hU.size(); i += 2) {
    const double th = 6.283185307179586 * rand() / RAND_MAX;
    hU[i] = cos(th);
    hU[i + 1] = sin(th);
  }
  for (auto& v : hb) v = 2.0 * rand() / RAND_MAX - 1.0;
  double2 *U, *b, *x;
  int *it, *st;
  double* rr;
  cudaMalloc(&U, hU.size() * 8);
  cudaMalloc(&b, hb.size() * 8);
  cudaMalloc(&x, hb.size() * 8);
  cudaMalloc(&it, maxB * 4);
  cudaMalloc(&st, maxB * 4);
  cudaMalloc(&rr, maxB * 8);
  cudaMemcpy(U, hU.data(), hU.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(b, hb.data(), hb.size() * 8, cudaMemcpyHostToDevice);
  ResArgs a{};
  a.U = U;
  a.b = b;
  a.x0 = nullptr;
  a.x = x;
  a.iters = it;
  a.relres = rr;
  a.status = st;
  a.L = a.T = L;
  a.diag = 2.1;
  a.tol = 0.0;   // never converges: every chain runs `iters` iterations
  a.maxiter = iters;
  auto kern = k_cg_resblk<16, 16, 2, 2, 4, 1, true>;
  const size_t smem = sizeof(double2) * 2 * (2 * 2 + 2 * 2) * 64;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, kern);
  printf("registers %d, local bytes %zu\n", fa.numRegs, fa.localSizeBytes);
  const char* names[10] = {"loop back-edge", "stage_pre D", "barrier 1", "stage_post D + |Dp|^2 + stage_pre D^dag + put",
                           "barrier 2", "stage_post D^dag", "sum slots + alpha = rs/den", "x, r update + |r|^2",
                           "block sum of |r|^2 (barrier 3)", "stop test + beta + p update + rcp"};
  for (int B : {1, 148, 592, 8192}) {
    unsigned long long z[12] = {0}, zi = 0;
    cudaMemcpyToSymbol(g_phase, z, sizeof(z));
    cudaMemcpyToSymbol(g_iters, &zi, sizeof(zi));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    kern<<<B, 64, smem>>>(a);
    cudaMemcpyToSymbol(g_phase, z, sizeof(z));
    cudaMemcpyToSymbol(g_iters, &zi, sizeof(zi));
    cudaEventRecord(e0);
    kern<<<B, 64, smem>>>(a);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long ph[12], ni;
    cudaMemcpyFromSymbol(ph, g_phase, sizeof(ph));
    cudaMemcpyFromSymbol(&ni, g_iters, sizeof(ni));
    double tot = 0;
    for (int i = 0; i < 10; ++i) tot += (double)ph[i] / ni;
    printf("B = %d: %.3f ms, %.2f ns per chain-iteration (err %s)\n", B, ms, ms * 1e6 / ((double)B * iters),
           cudaGetErrorString(cudaGetLastError()));
    if (ni == 0) continue;   // -DNOSTAMP
    printf("   %.0f cycles per iteration of one chain (thread 0's clock):\n", tot);
    for (int i = 0; i < 10; ++i)
      printf("   %-50s %7.1f cycles (%4.1f %%)\n", names[i], (double)ph[i] / ni, 100.0 * ph[i] / ni / tot);
  }
  return 0;
}
