// Counter-based device RNG for bench mode (momentum and pseudofermion
// heatbaths on the GPU).  Philox4x32-10 keyed by splitmix64(seed, stream),
// counter = (element pair, ctr); Box-Muller in FP64.  Parity mode does NOT
// use this: it draws with the reference's own NumPy Philox generator on the
// host (lattice.py:86-95, fermion.py:289) and uploads the draws.
#include "common.cuh"
#include "runtime.hpp"
#include "../../include/schwinger_sm100.h"

namespace {

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

struct U4 {
  uint32_t x, y, z, w;
};

__device__ __forceinline__ U4 philox4x32_10(U4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

__device__ __forceinline__ double u53(uint32_t hi, uint32_t lo) {
  uint64_t v = ((uint64_t)hi << 32) | lo;
  return (double)(v >> 11) * (1.0 / 9007199254740992.0);   // [0, 1)
}

template <bool NORMAL>
__global__ void k_rng(double* __restrict__ out, int B, long long per_chain, uint64_t seed,
                      uint64_t stream0, uint64_t ctr, double scale) {
  const long long pairs = (per_chain + 1) / 2;
  const long long n = (long long)B * pairs;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int b = (int)(i / pairs);
    const long long j = i - (long long)b * pairs;
    const uint64_t key = splitmix64(seed ^ splitmix64(stream0 + (uint64_t)b));
    U4 c{(uint32_t)j, (uint32_t)(j >> 32), (uint32_t)ctr, (uint32_t)(ctr >> 32)};
    U4 r = philox4x32_10(c, (uint32_t)key, (uint32_t)(key >> 32));
    double a = u53(r.x, r.y), bb = u53(r.z, r.w);
    double v0, v1;
    if (NORMAL) {
      double rad = sqrt(-2.0 * log(1.0 - a));   // 1-a in (0, 1]
      double sn, cs;
      sincospi(2.0 * bb, &sn, &cs);
      v0 = scale * (rad * cs);
      v1 = scale * (rad * sn);
    } else {
      v0 = a;
      v1 = bb;
    }
    double* o = out + (long long)b * per_chain + 2 * j;
    o[0] = v0;
    if (2 * j + 1 < per_chain) o[1] = v1;
  }
}

unsigned grid_for(long long n, int nt = 256) {
  long long b = (n + nt - 1) / nt;
  if (b > 148LL * 32) b = 148LL * 32;
  if (b < 1) b = 1;
  return (unsigned)b;
}

}  // namespace

extern "C" {

int sch_rng_normal(sch_ctx* ctx, double* out, int B, long long per_chain, uint64_t seed,
                   uint64_t stream0, uint64_t ctr, double scale) {
  SCH_CHECK_ARG(ctx, out && B >= 1 && per_chain >= 1, "rng_normal: bad args");
  k_rng<true><<<grid_for((long long)B * ((per_chain + 1) / 2)), 256, 0, ctx->stream>>>(
      out, B, per_chain, seed, stream0, ctr, scale);
  SCH_LAUNCHED(ctx);
  return SCH_OK;
}

int sch_rng_uniform(sch_ctx* ctx, double* out, int B, long long per_chain, uint64_t seed,
                    uint64_t stream0, uint64_t ctr) {
  SCH_CHECK_ARG(ctx, out && B >= 1 && per_chain >= 1, "rng_uniform: bad args");
  k_rng<false><<<grid_for((long long)B * ((per_chain + 1) / 2)), 256, 0, ctx->stream>>>(
      out, B, per_chain, seed, stream0, ctr, 1.0);
  SCH_LAUNCHED(ctx);
  return SCH_OK;
}

}  // extern "C"
