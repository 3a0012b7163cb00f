// Where one iteration of the cluster-resident per-chain CG (k_cg_cluster_tx,
// 64^2 on 4 CTAs) spends its cycles: thread 0 of every CTA reads its SM's
// clock at eleven points of the iteration (RES_STAMP in
// csrc/resident_cluster.cuh) and the per-phase sums are averaged over CTAs
// and iterations, for one chain alone, one wave (37 chains) and 1024 chains.
// Standalone (run on the GPU box):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1512_03812_b200/csrc \
//        -o /tmp/cluster_phases tools/micro/cluster_phases.cu && /tmp/cluster_phases
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

#include "resident_cluster.cuh"

int main() {
  const int L = 64, V = L * L, maxB = 1024, iters = 200;
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
  auto kern = k_cg_cluster_tx<64, 64, 4, 2, 2, 1, true>;
  constexpr int NT = 64 * 64 / (4 * 2 * 2), PL = (2 * 2 + 2 * 2) * NT, FACE = 2 * (64 / 2);
  const size_t smem = sizeof(double2) * (2 * PL + 8 * FACE);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, kern);
  printf("registers %d, local bytes %zu\n", fa.numRegs, fa.localSizeBytes);
  {   // how many 4-CTA clusters the GPU holds at once (cluster CTAs share a GPC)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(1024 * 4);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 4;
    at[0].val.clusterDim.y = at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int nc = 0;
    cudaOccupancyMaxActiveClusters(&nc, kern, &cfg);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    printf("resident 4-CTA clusters: %d (= %d of %d SMs)\n", nc, 4 * nc, sms);
  }
  const char* names[11] = {"loop back-edge", "produce D (exports, face pushes)", "barrier + interior D",
                           "face wait + faces D", "|Dp|^2 + produce D^dag + publish", "barrier + interior D^dag",
                           "face wait + faces D^dag", "cluster sum <p,Ap> (wait + butterfly)",
                           "alpha + r update + |r|^2 + publish + x update", "cluster sum |r|^2 (wait + butterfly)",
                           "stop test + beta + p update + rcp"};
  for (int B : {1, 37, 1024}) {
    unsigned long long z[12] = {0}, zi = 0;
    cudaMemcpyToSymbol(g_phase, z, sizeof(z));
    cudaMemcpyToSymbol(g_iters, &zi, sizeof(zi));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    kern<<<B * 4, NT, smem>>>(a);
    cudaMemcpyToSymbol(g_phase, z, sizeof(z));
    cudaMemcpyToSymbol(g_iters, &zi, sizeof(zi));
    cudaEventRecord(e0);
    kern<<<B * 4, NT, smem>>>(a);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long ph[12], ni;
    cudaMemcpyFromSymbol(ph, g_phase, sizeof(ph));
    cudaMemcpyFromSymbol(&ni, g_iters, sizeof(ni));
    double tot = 0;
    for (int i = 0; i < 11; ++i) tot += (double)ph[i] / ni;
    printf("B = %d: %.3f ms, %.2f ns per chain-iteration (err %s)\n", B, ms, ms * 1e6 / ((double)B * iters),
           cudaGetErrorString(cudaGetLastError()));
    if (ni == 0) continue;   // -DNOSTAMP
    printf("   %.0f cycles per iteration of one chain (thread 0's clock):\n", tot);
    for (int i = 0; i < 11; ++i)
      printf("   %-50s %7.1f cycles (%4.1f %%)\n", names[i], (double)ph[i] / ni, 100.0 * ph[i] / ni / tot);
  }
  return 0;
}
