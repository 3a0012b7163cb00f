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

// Philox4x64-10 of one 256-bit counter (Random123 constants, NumPy's walk)
__device__ __forceinline__ void philox_block(uint64_t x0, uint64_t x1, uint64_t x2, uint64_t x3,
                                             uint64_t ka, uint64_t kb, uint64_t& o0, uint64_t& o1,
                                             uint64_t& o2, uint64_t& o3) {
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
  o0 = x0; o1 = x1; o2 = x2; o3 = x3;
}

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
    philox_block(c0, c1, c2, c3, k0, k1, b0, b1, b2, b3);
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

// ---------------------------------------------------------------------------
// Warp-per-chain generation.  A stream is a sequence of 64-bit words; word a
// (absolute index, counted from the first word of the block in the state's
// buffer) is word a%4 of Philox block ctr0 + a/4, and block ctr0 is the
// state's buffer itself.  Blocks are counter-based, so the 32 lanes compute
// 32 blocks (128 words) at a time into a per-warp shared-memory ring.  The
// ziggurat's fast path (one word -> one normal, ~99 % of draws) is evaluated
// for 32 consecutive words at once: a ballot finds the first word that needs
// the slow path, the words before it are emitted in order, and that one draw
// is then run serially by the whole warp (tail / wedge, consuming further
// words exactly as NumPy's random_standard_normal does).  The state written
// back is NumPy's: the block holding the last consumed word, buffer_pos
// after it.  Values and stream position are identical to the scalar walk.
constexpr int kRing = 256;   // words per warp (two 128-word chunks)

struct WarpGen {
  uint64_t* ring;
  uint64_t c0, c1, c2, c3, k0, k1, b0, b1, b2, b3;   // ctr0, key, buffer of block 0
  long long a;        // next word to consume (warp-uniform)
  long long filled;   // words [0, filled) have been generated
  long long a0;       // a at load
  int lane;

  __device__ void load(const NpPhilox& s, uint64_t* ring_, int lane_) {
    ring = ring_;
    lane = lane_;
    c0 = s.ctr[0]; c1 = s.ctr[1]; c2 = s.ctr[2]; c3 = s.ctr[3];
    k0 = s.key[0]; k1 = s.key[1];
    b0 = s.buf[0]; b1 = s.buf[1]; b2 = s.buf[2]; b3 = s.buf[3];
    a = a0 = s.pos;
    filled = 0;
  }
  // block j >= 1 after ctr0 (256-bit add)
  __device__ void block_at(long long j, uint64_t& o0, uint64_t& o1, uint64_t& o2, uint64_t& o3) const {
    uint64_t x0 = c0 + (uint64_t)j, x1 = c1, x2 = c2, x3 = c3;
    if (x0 < c0 && ++x1 == 0 && ++x2 == 0) ++x3;
    philox_block(x0, x1, x2, x3, k0, k1, o0, o1, o2, o3);
  }
  __device__ void fill_next() {   // blocks [filled/4, filled/4 + 32)
    const long long j = filled / 4 + lane;
    uint64_t w0, w1, w2, w3;
    if (j == 0) { w0 = b0; w1 = b1; w2 = b2; w3 = b3; }
    else block_at(j, w0, w1, w2, w3);
    const int sl = (int)((4 * j) % kRing);
    __syncwarp();
    ring[sl] = w0; ring[sl + 1] = w1; ring[sl + 2] = w2; ring[sl + 3] = w3;
    __syncwarp();
    filled += 128;
  }
  __device__ void ensure(long long i) {   // warp-uniform: words up to i are in the ring
    while (i >= filled) fill_next();
  }
  __device__ uint64_t next_u64() {         // warp-uniform serial draw
    ensure(a);
    return ring[(a++) % kRing];
  }
  __device__ double next_double() { return (double)(next_u64() >> 11) * (1.0 / 9007199254740992.0); }

  // one complete NumPy standard_normal, run redundantly by every lane
  __device__ double normal_serial() {
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

  // n normals, out[i * stride] = scale * N_i (scale 1 leaves the value exact)
  __device__ void normals(double* out, long long n, long long stride, double scale, bool scaled) {
    long long done = 0;
    while (done < n) {
      ensure(a + 31);
      uint64_t r = ring[(a + lane) % kRing];
      const int idx = (int)(r & 0xff);
      r >>= 8;
      const uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
      double x = (double)rabs * np_wi_double[idx];
      if (r & 0x1) x = -x;
      const unsigned slow = __ballot_sync(0xffffffffu, !(rabs < np_ki_double[idx]));
      const int f = slow ? __ffs(slow) - 1 : 32;
      const long long k = min((long long)f, n - done);
      if (lane < k) out[(done + lane) * stride] = scaled ? x * scale : x;
      a += k;
      done += k;
      if (done < n && k == f) {   // word a starts a slow-path draw
        const double y = normal_serial();
        if (lane == 0) out[done * stride] = scaled ? y * scale : y;
        ++done;
      }
    }
  }
  // n doubles lo + (hi - lo) * u (mode 1) or u (mode 2), one word each
  __device__ void doubles(double* out, long long n, int mode, double lo, double hi) {
    const double range = hi - lo;
    for (long long done = 0; done < n; done += 32) {
      ensure(a + 31);
      const double u = (double)(ring[(a + lane) % kRing] >> 11) * (1.0 / 9007199254740992.0);
      const long long k = min(32LL, n - done);
      if (lane < k) out[done + lane] = mode == 1 ? __dadd_rn(lo, __dmul_rn(range, u)) : u;
      a += k;
    }
  }
  __device__ void store(NpPhilox& s) const {
    if (a == a0) return;   // nothing consumed
    const long long jl = (a - 1) / 4;
    uint64_t w[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) w[e] = ring[(4 * jl + e) % kRing];
    if (lane == 0) {
      uint64_t x0 = c0 + (uint64_t)jl, x1 = c1, x2 = c2, x3 = c3;
      if (x0 < c0 && ++x1 == 0 && ++x2 == 0) ++x3;
      s.ctr[0] = x0; s.ctr[1] = x1; s.ctr[2] = x2; s.ctr[3] = x3;
      s.buf[0] = w[0]; s.buf[1] = w[1]; s.buf[2] = w[2]; s.buf[3] = w[3];
      s.pos = (int)((a - 1) % 4) + 1;
    }
  }
};

constexpr int kWarpsPerBlock = 4;

__global__ void __launch_bounds__(32 * kWarpsPerBlock) k_np_heatbath_w(
    NpPhilox* st, double* __restrict__ p, double* __restrict__ phi, int B, long long V, double s,
    int quenched) {
  __shared__ uint64_t rings[kWarpsPerBlock][kRing];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x * kWarpsPerBlock + w;
  if (c >= B) return;
  WarpGen g;
  g.load(st[c], rings[w], lane);
  g.normals(p + (long long)c * 2 * V, 2 * V, 1, 1.0, false);
  if (!quenched) {
    double* fc = phi + (long long)c * 4 * V;   // complex128 (re, im) pairs
    g.normals(fc, 2 * V, 2, s, true);
    g.normals(fc + 1, 2 * V, 2, s, true);
  }
  __syncwarp();
  g.store(st[c]);
}

__global__ void __launch_bounds__(32 * kWarpsPerBlock) k_np_fill_w(
    NpPhilox* st, double* __restrict__ out, int B, long long n, int mode, double lo, double hi) {
  __shared__ uint64_t rings[kWarpsPerBlock][kRing];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x * kWarpsPerBlock + w;
  if (c >= B) return;
  WarpGen g;
  g.load(st[c], rings[w], lane);
  if (mode == 0) g.normals(out + (long long)c * n, n, 1, 1.0, false);
  else g.doubles(out + (long long)c * n, n, mode, lo, hi);
  __syncwarp();
  g.store(st[c]);
}

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
unsigned warp_blocks(int B) { return (unsigned)((B + kWarpsPerBlock - 1) / kWarpsPerBlock); }

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
  k_np_fill_w<<<warp_blocks(B), 32 * kWarpsPerBlock, 0, ctx->stream>>>((NpPhilox*)state, out, B,
                                                                        n_per_chain, mode, lo, hi);
  SCH_LAUNCHED(ctx);
  return SCH_OK;
}

int sch_np_heatbath(sch_ctx* ctx, void* state, double* p, double* phi, int B, long long V,
                    double phi_scale, int quenched) {
  SCH_CHECK_ARG(ctx, state && p && (phi || quenched) && B >= 1 && V >= 1, "np_heatbath: bad args");
  k_np_heatbath_w<<<warp_blocks(B), 32 * kWarpsPerBlock, 0, ctx->stream>>>((NpPhilox*)state, p, phi,
                                                                            B, V, phi_scale, quenched);
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
