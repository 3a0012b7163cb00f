// Measurement probes used by bench.py to establish denominators that
// MEASURED_PEAKS.json does not carry: the FP64 FMA issue rate of this B200.
#include "common.cuh"
#include "runtime.hpp"
#include "../../include/schwinger_sm100.h"

namespace {

// 8 independent DFMA chains per thread; flops = grid*256*iters*8*2
__global__ void __launch_bounds__(256) k_fp64_fma(double* __restrict__ out, int iters, double a,
                                                  double b) {
  double v0 = threadIdx.x, v1 = v0 + 1, v2 = v0 + 2, v3 = v0 + 3;
  double v4 = v0 + 4, v5 = v0 + 5, v6 = v0 + 6, v7 = v0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      v0 = fma(v0, a, b); v1 = fma(v1, a, b); v2 = fma(v2, a, b); v3 = fma(v3, a, b);
      v4 = fma(v4, a, b); v5 = fma(v5, a, b); v6 = fma(v6, a, b); v7 = fma(v7, a, b);
    }
  }
  double s = ((v0 + v1) + (v2 + v3)) + ((v4 + v5) + (v6 + v7));
  if (s == 1.2345) out[blockIdx.x] = s;   // keep the chains alive
}

}  // namespace

extern "C" int sch_probe_fp64(sch_ctx* ctx, double* scratch, int blocks, int iters) {
  SCH_CHECK_ARG(ctx, scratch && blocks >= 1 && iters >= 1, "probe_fp64: bad args");
  k_fp64_fma<<<blocks, 256, 0, ctx->stream>>>(scratch, iters, 0.999999, 1e-7);
  SCH_LAUNCHED(ctx);
  return SCH_OK;
}
