// Bit-exact device replica of the reference's random streams
// (lattice.py:86-104, fermion.py:289, hmc.py:54-60):
//   np.random.Generator(np.random.Philox(key=[seed, stream]))
//     .standard_normal / .uniform / .random
//
// * bit generator: Philox4x64-10 (Random123 constants), 4-word output
//   buffer, 256-bit counter starting at 0 and incremented before each block,
//   as NumPy's philox bit generator does;
// * next_double = (next_uint64 >> 11) * 2^-53;
// * standard_normal: NumPy's 256-layer ziggurat (random_standard_normal) with
//   the layer tables read out of the installed NumPy at build time
//   (tools/extract_ziggurat.py -> _lib/gen/ziggurat_tables.h);
// * uniform(lo, hi) = lo + (hi - lo) * next_double.
//
// One thread owns one chain's stream (the draw sequence of a stream is
// inherently serial: the ziggurat consumes a data-dependent number of words).
// The generator state lives in device memory between calls, so a chain's
// stream advances exactly as the reference's Generator object would.
#include "common.cuh"
#include "runtime.hpp"
#include "../_lib/gen/ziggurat_tables.h"
#include "../../include/schwinger_sm100.h"

namespace {

struct NpPhilox {
  uint64_t ctr[4];
  uint64_t key[2];
  uint64_t buf[4];
  int pos;
  int pad;
};
static_assert(sizeof(NpPhilox) == 88, "state layout");

constexpr uint64_t kM0 = 0xD2E7470EE14C6C93ULL, kM1 = 0xCA5A826395121157ULL;
constexpr uint64_t kW0 = 0x9E3779B97F4A7C15ULL, kW1 = 0xBB67AE8584CAA73BULL;
constexpr double kZigR = 3.6541528853610088;       // ziggurat_nor_r
constexpr double kZigInvR = 0.27366123732975828;   // ziggurat_nor_inv_r

struct Gen {
  uint64_t c0, c1, c2, c3, k0, k1, b0, b1, b2, b3;
  int pos;

  __device__ void load(const NpPhilox& s) {
    c0 = s.ctr[0]; c1 = s.ctr[1]; c2 = s.ctr[2]; c3 = s.ctr[3];
    k0 = s.key[0]; k1 = s.key[1];
    b0 = s.buf[0]; b1 = s.buf[1]; b2 = s.buf[2]; b3 = s.buf[3];
    pos = s.pos;
  }
  __device__ void store(NpPhilox& s) const {
    s.ctr[0] = c0; s.ctr[1] = c1; s.ctr[2] = c2; s.ctr[3] = c3;
    s.key[0] = k0; s.key[1] = k1;
    s.buf[0] = b0; s.buf[1] = b1; s.buf[2] = b2; s.buf[3] = b3;
    s.pos = pos;
  }
  __device__ void block() {
    if (++c0 == 0 && ++c1 == 0 && ++c2 == 0) ++c3;   // 256-bit counter increment
    uint64_t x0 = c0, x1 = c1, x2 = c2, x3 = c3, ka = k0, kb = k1;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
      const uint64_t hi0 = __umul64hi(kM0, x0), lo0 = kM0 * x0;
      const uint64_t hi1 = __umul64hi(kM1, x2), lo1 = kM1 * x2;
      x0 = hi1 ^ x1 ^ ka;
      x1 = lo1;
      x2 = hi0 ^ x3 ^ kb;
      x3 = lo0;
      ka += kW0;
      kb += kW1;
    }
    b0 = x0; b1 = x1; b2 = x2; b3 = x3;
    pos = 0;
  }
  __device__ uint64_t next_u64() {
    if (pos >= 4) block();
    const uint64_t v = pos == 0 ? b0 : pos == 1 ? b1 : pos == 2 ? b2 : b3;
    ++pos;
    return v;
  }
  __device__ double next_double() { return (double)(next_u64() >> 11) * (1.0 / 9007199254740992.0); }

  // NumPy random_standard_normal (ziggurat, 256 layers).  Written as one
  // loop with an explicit result flag: the reference's nested early returns,
  // executed by divergent lanes, were mis-scheduled (a draw returned without
  // consuming its word).
  __device__ double normal() {
    double result = 0.0;
    bool done = false;
    while (!done) {
      uint64_t r = next_u64();
      const int idx = (int)(r & 0xff);
      r >>= 8;
      const int sign = (int)(r & 0x1);
      const uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
      double x = (double)rabs * np_wi_double[idx];
      if (sign & 0x1) x = -x;
      if (rabs < np_ki_double[idx]) {
        result = x;
        done = true;
      } else if (idx == 0) {
        bool tail = false;
        while (!tail) {
          const double xx = -kZigInvR * log1p(-next_double());
          const double yy = -log1p(-next_double());
          if (yy + yy > xx * xx) {
            result = ((rabs >> 8) & 0x1) ? -(kZigR + xx) : kZigR + xx;
            tail = true;
          }
        }
        done = true;
      } else {
        // two roundings, as NumPy's baseline-x86 build evaluates it (no FMA)
        const double u = next_double();
        if (__dadd_rn(__dmul_rn(np_fi_double[idx - 1] - np_fi_double[idx], u), np_fi_double[idx]) <
            exp(-0.5 * x * x)) {
          result = x;
          done = true;
        }
      }
    }
    return result;
  }
};

__global__ void k_np_init(NpPhilox* st, int B, uint64_t seed, uint64_t stream0) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= B) return;
  NpPhilox s;
  s.ctr[0] = s.ctr[1] = s.ctr[2] = s.ctr[3] = 0;
  s.key[0] = seed;
  s.key[1] = stream0 + (uint64_t)c;
  s.buf[0] = s.buf[1] = s.buf[2] = s.buf[3] = 0;
  s.pos = 4;
  s.pad = 0;
  st[c] = s;
}

// mode 0: normal, 1: uniform lo + (hi - lo) * u, 2: raw next_double
__global__ void k_np_fill(NpPhilox* st, double* __restrict__ out, int B, long long n, int mode,
                          double lo, double hi) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= B) return;
  Gen g;
  g.load(st[c]);
  double* o = out + (long long)c * n;
  const double range = hi - lo;
  for (long long i = 0; i < n; ++i)
    o[i] = mode == 0   ? g.normal()
           : mode == 1 ? __dadd_rn(lo, __dmul_rn(range, g.next_double()))
                       : g.next_double();
  g.store(st[c]);
}

// HMC heatbath draws of one chain in the reference's order (hmc.py:78-82,
// fermion.py:289): p = N(2V); re = N(2V); im = N(2V); phi = (re + i im) * s
// with s = 1/sqrt(2) as NumPy's complex division by sqrt(2) evaluates it.
__global__ void k_np_heatbath(NpPhilox* st, double* __restrict__ p, double2* __restrict__ phi,
                              int B, long long V, double s, int quenched) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= B) return;
  Gen g;
  g.load(st[c]);
  double* pc = p + (long long)c * 2 * V;
  for (long long i = 0; i < 2 * V; ++i) pc[i] = g.normal();
  if (!quenched) {
    double2* fc = phi + (long long)c * 2 * V;
    for (long long i = 0; i < 2 * V; ++i) fc[i].x = g.normal() * s;
    for (long long i = 0; i < 2 * V; ++i) fc[i].y = g.normal() * s;
  }
  g.store(st[c]);
}

// metropolis (hmc.py:54-60): draw only when dH > 0
__global__ void k_np_metropolis(NpPhilox* st, const double* __restrict__ dh, int* __restrict__ acc,
                                int B) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= B) return;
  const double d = dh[c];
  if (!isfinite(d)) {
    acc[c] = -1;
    return;
  }
  if (d <= 0.0) {
    acc[c] = 1;
    return;
  }
  Gen g;
  g.load(st[c]);
  acc[c] = g.next_double() < exp(-d) ? 1 : 0;
  g.store(st[c]);
}

unsigned chain_blocks(int B) { return (unsigned)((B + 63) / 64); }

}  // namespace

extern "C" {

int sch_np_rng_state_bytes(void) { return (int)sizeof(NpPhilox); }

int sch_np_rng_init(sch_ctx* ctx, void* state, int B, uint64_t seed, uint64_t stream0) {
  SCH_CHECK_ARG(ctx, state && B >= 1, "np_rng_init: bad args");
  k_np_init<<<chain_blocks(B), 64, 0, ctx->stream>>>((NpPhilox*)state, B, seed, stream0);
  SCH_LAUNCHED(ctx);
  return SCH_OK;
}

int sch_np_rng_fill(sch_ctx* ctx, void* state, double* out, int B, long long n_per_chain, int mode,
                    double lo, double hi) {
  SCH_CHECK_ARG(ctx, state && out && B >= 1 && n_per_chain >= 0 && mode >= 0 && mode <= 2,
                "np_rng_fill: bad args");
  k_np_fill<<<chain_blocks(B), 64, 0, ctx->stream>>>((NpPhilox*)state, out, B, n_per_chain, mode,
                                                     lo, hi);
  SCH_LAUNCHED(ctx);
  return SCH_OK;
}

int sch_np_heatbath(sch_ctx* ctx, void* state, double* p, double* phi, int B, long long V,
                    double phi_scale, int quenched) {
  SCH_CHECK_ARG(ctx, state && p && (phi || quenched) && B >= 1 && V >= 1, "np_heatbath: bad args");
  k_np_heatbath<<<chain_blocks(B), 64, 0, ctx->stream>>>((NpPhilox*)state, p, (double2*)phi, B, V,
                                                         phi_scale, quenched);
  SCH_LAUNCHED(ctx);
  return SCH_OK;
}

int sch_np_metropolis(sch_ctx* ctx, void* state, const double* dh, int* accept, int B) {
  SCH_CHECK_ARG(ctx, state && dh && accept && B >= 1, "np_metropolis: bad args");
  k_np_metropolis<<<chain_blocks(B), 64, 0, ctx->stream>>>((NpPhilox*)state, dh, accept, B);
  SCH_LAUNCHED(ctx);
  return SCH_OK;
}

}  // extern "C"
