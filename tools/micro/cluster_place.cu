// Where do the CTAs of a thread-block cluster land?  Launches B clusters of
// CS CTAs (128 threads, `smem` bytes of shared memory each, so that `per_sm`
// CTAs fit an SM) and records %smid per CTA; prints how many SMs hold two or
// more CTAs of the SAME cluster (which would serialize one chain's barrier
// phases on one SM) and the per-SM CTA count histogram.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o cluster_place cluster_place.cu
//   ./cluster_place CS per_sm
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <vector>

__global__ void k_place(int* smid, long long spin) {
  extern __shared__ char sm[];
  namespace cg = cooperative_groups;
  unsigned s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  if (threadIdx.x == 0) {
    smid[blockIdx.x] = (int)s;
    sm[0] = 1;
  }
  const long long t0 = clock64();
  while (clock64() - t0 < spin) {
  }
  cg::this_cluster().sync();
}

int main(int argc, char** argv) {
  const int CS = argc > 1 ? atoi(argv[1]) : 8;
  const int per_sm = argc > 2 ? atoi(argv[2]) : 2;
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const size_t smem = (size_t)(220 * 1024 / per_sm);
  cudaFuncSetAttribute(k_place, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int nclusters = nsm * per_sm / CS;   // one wave
  const int nblk = nclusters * CS;
  int* d;
  cudaMalloc(&d, sizeof(int) * nblk);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nblk);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k_place, d, 2000000LL);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(e));
    return 1;
  }
  std::vector<int> h(nblk);
  cudaMemcpy(h.data(), d, sizeof(int) * nblk, cudaMemcpyDeviceToHost);
  int shared_sm = 0, clusters_sharing = 0;
  std::map<int, int> per;
  for (int c = 0; c < nclusters; ++c) {
    std::map<int, int> m;
    for (int r = 0; r < CS; ++r) m[h[c * CS + r]]++;
    bool any = false;
    for (auto& kv : m)
      if (kv.second > 1) {
        ++shared_sm;
        any = true;
      }
    clusters_sharing += any;
  }
  for (int i = 0; i < nblk; ++i) per[h[i]]++;
  std::map<int, int> hist;
  for (auto& kv : per) hist[kv.second]++;
  printf("CS=%d per_sm=%d: %d clusters, %d with two or more CTAs on one SM (%d such SMs); "
         "SMs by CTA count:", CS, per_sm, nclusters, clusters_sharing, shared_sm);
  for (auto& kv : hist) printf(" %d:%d", kv.first, kv.second);
  printf("\n");
  return 0;
}
