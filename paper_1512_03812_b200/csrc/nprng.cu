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
#include <algorithm>
#include <cstdlib>

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

// log1p(x) for x in (-1, 0] (the ziggurat tail's log1p(-u)), operation by
// operation what the reference's libm evaluates: glibc's log1p (the fdlibm
// algorithm with its polynomial split in four, as glibc evaluates it), built
// with FMA contraction as the variant x86-64 hosts with FMA dispatch to —
// checked here against the host libm on 2e7 arguments (0 differences; CUDA's
// log1p differs from it in the last bit for ~0.4 % of arguments) and by the
// stream tests against NumPy itself.  Every operation is an explicit
// intrinsic, so nvcc contracts nothing else.
__device__ double np_log1p_neg(double x) {
  const double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10;
  const double Lp1 = 6.666666666666735130e-01, Lp2 = 3.999999999940941908e-01,
               Lp3 = 2.857142874366239149e-01, Lp4 = 2.222219843214978396e-01,
               Lp5 = 1.818357216161805012e-01, Lp6 = 1.531383769920937332e-01,
               Lp7 = 1.479819860511658591e-01;
  const int hx = __double2hiint(x), ax = hx & 0x7fffffff;
  if (hx > 0 || ax >= 0x3ff00000) return log1p(x);   // outside (-1, 0]: not the tail's argument
  int k = 1, hu = 0;
  double f = 0.0, c = 0.0;
  if (ax < 0x3e200000) {                               // |x| < 2^-29
    if (ax < 0x3c900000) return x;                     // |x| < 2^-54
    return __fma_rn(-0.5, __dmul_rn(x, x), x);
  }
  if (hx <= (int)0xbfd2bec3) {                         // -0.2929 < x
    k = 0;
    f = x;
    hu = 1;
  } else {
    double u = __dadd_rn(1.0, x);
    hu = __double2hiint(u);
    k = (hu >> 20) - 1023;
    c = k > 0 ? __dsub_rn(1.0, __dsub_rn(u, x)) : __dsub_rn(x, __dsub_rn(u, 1.0));
    c = __ddiv_rn(c, u);
    hu &= 0x000fffff;
    if (hu < 0x6a09e) {
      u = __hiloint2double(hu | 0x3ff00000, __double2loint(u));
    } else {
      k += 1;
      u = __hiloint2double(hu | 0x3fe00000, __double2loint(u));
      hu = (0x00100000 - hu) >> 2;
    }
    f = __dsub_rn(u, 1.0);
  }
  const double hfsq = __dmul_rn(__dmul_rn(0.5, f), f);
  const double dk = (double)k;
  if (hu == 0) {                                       // |f| < 2^-20
    if (f == 0.0) return k == 0 ? 0.0 : __fma_rn(dk, ln2_hi, __fma_rn(dk, ln2_lo, c));
    const double R = __dmul_rn(__fma_rn(-0.66666666666666666, f, 1.0), hfsq);
    if (k == 0) return __dsub_rn(f, R);
    return __fma_rn(dk, ln2_hi, -__dsub_rn(__dsub_rn(R, __fma_rn(dk, ln2_lo, c)), f));
  }
  const double s = __ddiv_rn(f, __dadd_rn(f, 2.0));
  const double z = __dmul_rn(s, s);
  const double R4 = __fma_rn(z, Lp7, Lp6), R3 = __fma_rn(z, Lp5, Lp4), R2 = __fma_rn(z, Lp3, Lp2);
  const double z2 = __dmul_rn(z, z), z4 = __dmul_rn(z2, z2), z6 = __dmul_rn(z2, z4);
  double R = __fma_rn(z, Lp1, __dmul_rn(z2, R2));
  R = __fma_rn(z4, R3, R);
  R = __fma_rn(z6, R4, R);
  const double t = __dmul_rn(__dadd_rn(R, hfsq), s);
  if (k == 0) return __dsub_rn(f, __dsub_rn(hfsq, t));
  return __fma_rn(dk, ln2_hi, -__dsub_rn(__dsub_rn(hfsq, __dadd_rn(t, __fma_rn(dk, ln2_lo, c))), f));
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
          const double xx = -kZigInvR * np_log1p_neg(-next_double());
          const double yy = -np_log1p_neg(-next_double());
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
  // start at absolute word `start` (the parallel walk's chunks); a0 = -1: the
  // state is always written back
  __device__ void load_at(const NpPhilox& s, uint64_t* ring_, int lane_, long long start) {
    load(s, ring_, lane_);
    a = start;
    a0 = -1;
    filled = (start / 4) * 4;
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

  // one pass of NumPy's random_standard_normal loop at word a, run redundantly
  // by every lane: consumes the words the reference consumes; true if the
  // pass returned a value
  __device__ bool attempt_serial(double& result) {
    uint64_t r = next_u64();
    const int idx = (int)(r & 0xff);
    r >>= 8;
    const int sign = (int)(r & 0x1);
    const uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
    double x = (double)rabs * np_wi_double[idx];
    if (sign & 0x1) x = -x;
    if (rabs < np_ki_double[idx]) {
      result = x;
      return true;
    }
    if (idx == 0) {
      for (;;) {
        const double xx = -kZigInvR * np_log1p_neg(-next_double());
        const double yy = -np_log1p_neg(-next_double());
        if (yy + yy > xx * xx) {
          result = ((rabs >> 8) & 0x1) ? -(kZigR + xx) : kZigR + xx;
          return true;
        }
      }
    }
    // two roundings, as NumPy's baseline-x86 build evaluates it (no FMA)
    const double u = next_double();
    if (__dadd_rn(__dmul_rn(np_fi_double[idx - 1] - np_fi_double[idx], u), np_fi_double[idx]) <
        exp(-0.5 * x * x)) {
      result = x;
      return true;
    }
    return false;
  }
  // one complete NumPy standard_normal
  __device__ double normal_serial() {
    double result = 0.0;
    while (!attempt_serial(result)) {
    }
    return result;
  }

  // The passes that START at words [a, end): emit(g, value) for the values
  // they return, numbered g0, g0 + 1, ... and stopping at N.  Returns the
  // number emitted; `a` is left behind the last pass's words (it may lie
  // beyond `end`: a pass that starts inside the chunk runs to its end).
  template <class Emit>
  __device__ long long walk(long long end, long long g0, long long N, Emit emit) {
    long long g = g0;
    while (a < end && g < N) {
      ensure(a + 31);
      uint64_t r = ring[(a + lane) % kRing];
      const int idx = (int)(r & 0xff);
      r >>= 8;
      const uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
      double x = (double)rabs * np_wi_double[idx];
      if (r & 0x1) x = -x;
      const unsigned slow = __ballot_sync(0xffffffffu, a + lane < end && !(rabs < np_ki_double[idx]));
      const int f = slow ? __ffs(slow) - 1 : 32;
      const long long k = min(min((long long)f, end - a), N - g);
      if (lane < k) emit(g + lane, x);
      a += k;
      g += k;
      if (k == f && a < end && g < N) {   // word a starts a slow pass
        double y;
        if (attempt_serial(y)) {
          if (lane == 0) emit(g, y);
          ++g;
        }
      }
    }
    return g - g0;
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

// ---------------------------------------------------------------------------
// One long stream walked by the whole GPU (the decomposed lattice's heatbath
// draws 6 * L * T normals from ONE reference stream: a single warp needs
// 0.5 s for cfg5's 25 M).  The words of a stream are random-access (Philox is
// counter based); only the ziggurat's passes are serial, because a pass that
// leaves the fast path consumes extra words.  The stream's words are cut into
// chunks of C = kChunk words (SCH_NP_CHUNK sets another size: the tests walk
// streams in chunks of a few words, where nearly every chunk is entered at an
// offset and slow passes straddle several chunks):
//   A  every warp walks its chunk as if a pass started at the chunk's first
//      word: how many values the passes starting in the chunk return (cnt)
//      and how many words the last one runs past the chunk's end (over);
//   B  one warp goes through the chunks in order: the entry offset of chunk
//      k is the overrun of chunk k-1, and the numbering of its first value
//      the running sum of the counts.  Where the entry offset is not 0 (1 %
//      of the chunks) the chunk's count is corrected by walking both entry
//      points until they meet (two neighbouring passes meet at once unless
//      one is a slow pass: a few words);
//   C  every warp walks its chunk again from its true entry and writes the
//      values to their places; the warp that writes value N-1 stores the
//      generator state (NumPy's: block of the last consumed word, position);
//   D  if the chunks did not hold N values (they are sized for 1.02 words per
//      value; 1.0127 expected), one warp continues serially.
// Values and final state are those of the serial walk, bit for bit.
constexpr int kChunk = 2048;

struct OutMap {   // where value g of the stream goes
  double *p, *phi;
  long long V2;   // heatbath: 2 V values to p, then 2 V to Re phi, 2 V to Im phi (both x s)
  double s;
  int heatbath;
  __device__ void put(long long g, double x) const {
    if (!heatbath || g < V2) p[g] = x;
    else if (g < 2 * V2) phi[2 * (g - V2)] = x * s;
    else phi[2 * (g - 2 * V2) + 1] = x * s;
  }
};

struct ParArgs {
  NpPhilox* st;
  long long N;
  int K, C;         // chunks, words per chunk
  int *cnt, *over, *entry;
  long long* pref;
  long long* tot;   // [0] values the chunks hold (capped at N), [1] first word after the chunks' passes
  NpPhilox* st_end; // the state after value N-1, written by the warp that emits it (the other
                    // warps of that launch still read *st); the last kernel moves it to *st
  OutMap om;
};

// scalar random access to the stream's words (phase B's corrections)
struct WordAt {
  uint64_t c0, c1, c2, c3, k0, k1, b[4];
  long long cached;
  uint64_t w[4];
  __device__ void load(const NpPhilox& s) {
    c0 = s.ctr[0]; c1 = s.ctr[1]; c2 = s.ctr[2]; c3 = s.ctr[3];
    k0 = s.key[0]; k1 = s.key[1];
    for (int e = 0; e < 4; ++e) b[e] = s.buf[e];
    cached = -1;
  }
  __device__ uint64_t at(long long i) {
    const long long j = i / 4;
    if (j != cached) {
      if (j == 0) {
        for (int e = 0; e < 4; ++e) w[e] = b[e];
      } else {
        uint64_t x0 = c0 + (uint64_t)j, x1 = c1, x2 = c2, x3 = c3;
        if (x0 < c0 && ++x1 == 0 && ++x2 == 0) ++x3;
        philox_block(x0, x1, x2, x3, k0, k1, w[0], w[1], w[2], w[3]);
      }
      cached = j;
    }
    return w[i % 4];
  }
  __device__ double dbl(long long i) { return (double)(at(i) >> 11) * (1.0 / 9007199254740992.0); }
  // the pass starting at word i: words consumed, and whether it returns a value
  __device__ int pass(long long i, bool& value) {
    uint64_t r = at(i);
    const int idx = (int)(r & 0xff);
    r >>= 8;
    const int sign = (int)(r & 0x1);
    const uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
    value = true;
    if (rabs < np_ki_double[idx]) return 1;
    if (idx == 0) {
      int n = 1;
      for (;;) {
        const double xx = -kZigInvR * np_log1p_neg(-dbl(i + n));
        const double yy = -np_log1p_neg(-dbl(i + n + 1));
        n += 2;
        if (yy + yy > xx * xx) return n;
      }
    }
    double x = (double)rabs * np_wi_double[idx];
    if (sign & 0x1) x = -x;
    value = __dadd_rn(__dmul_rn(np_fi_double[idx - 1] - np_fi_double[idx], dbl(i + 1)), np_fi_double[idx]) <
            exp(-0.5 * x * x);
    return 2;
  }
};

constexpr int kWarpsPerBlock = 4;

__global__ void __launch_bounds__(32 * kWarpsPerBlock) k_np_par_count(ParArgs a) {
  __shared__ uint64_t rings[kWarpsPerBlock][kRing];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int k = blockIdx.x * kWarpsPerBlock + w;
  if (k >= a.K) return;
  const long long start = a.st->pos + (long long)k * a.C, end = start + a.C;
  WarpGen g;
  g.load_at(*a.st, rings[w], lane, start);
  const long long n = g.walk(end, 0, 0x7fffffffffffffffLL, [](long long, double) {});
  if (lane == 0) {
    a.cnt[k] = (int)n;
    a.over[k] = (int)(g.a - end);
  }
}

__global__ void __launch_bounds__(32) k_np_par_scan(ParArgs a) {
  const int lane = threadIdx.x;
  WordAt wa;
  wa.load(*a.st);
  const long long a0 = a.st->pos;
  int e = 0;            // entry offset of the current chunk (warp-uniform)
  long long run = 0;    // values before the current chunk
  for (int k0 = 0; k0 < a.K; k0 += 32) {
    const int kk = k0 + lane;
    int n = kk < a.K ? a.cnt[kk] : 0, o = kk < a.K ? a.over[kk] : 0;
    int my_e = 0;
    long long my_pref = 0;
    for (int j = 0; j < 32 && k0 + j < a.K; ++j) {   // every lane runs the same sequence
      int nj = __shfl_sync(0xffffffffu, n, j), oj = __shfl_sync(0xffffffffu, o, j);
      if (e != 0) {
        // passes from the assumed entry (word 0 of the chunk) and from the true
        // one (word e) until they stand on the same word
        const long long s0 = a0 + (long long)(k0 + j) * a.C, end = s0 + a.C;
        long long pm = s0, pa = s0 + e;
        int cm = 0, ca = 0;
        while (pm != pa && (pm < end || pa < end)) {
          bool v;
          if (pm < pa) {
            const int c = wa.pass(pm, v);
            if (pm < end) cm += v;
            pm += c;
          } else {
            const int c = wa.pass(pa, v);
            if (pa < end) ca += v;
            pa += c;
          }
        }
        if (pm == pa && pm < end) {
          nj = nj - cm + ca;   // the same passes from the meeting word on
        } else {               // no common word inside the chunk: the true walk alone
          while (pa < end) {
            bool v;
            const int c = wa.pass(pa, v);
            ca += v;
            pa += c;
          }
          nj = ca;
          oj = (int)(pa - end);
        }
      }
      if (lane == j) {
        my_e = e;
        my_pref = run;
      }
      run += nj;
      e = oj;
    }
    if (kk < a.K) {
      a.entry[kk] = my_e;
      a.pref[kk] = my_pref;
    }
  }
  if (lane == 0) {
    a.tot[0] = run < a.N ? run : a.N;
    a.tot[1] = a0 + (long long)a.K * a.C + e;
  }
}

__global__ void __launch_bounds__(32 * kWarpsPerBlock) k_np_par_emit(ParArgs a) {
  __shared__ uint64_t rings[kWarpsPerBlock][kRing];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int k = blockIdx.x * kWarpsPerBlock + w;
  if (k >= a.K) return;
  const long long g0 = a.pref[k];
  if (g0 >= a.N) return;   // warp-uniform
  const long long start = a.st->pos + (long long)k * a.C, end = start + a.C;
  WarpGen g;
  g.load_at(*a.st, rings[w], lane, start + a.entry[k]);
  const OutMap om = a.om;
  const long long n = g.walk(end, g0, a.N, [&](long long i, double x) { om.put(i, x); });
  __syncwarp();
  if (g0 + n == a.N) {   // this warp wrote the last value
    if (lane == 0) {
      a.st_end->key[0] = a.st->key[0];
      a.st_end->key[1] = a.st->key[1];
      a.st_end->pad = 0;
    }
    g.store(*a.st_end);
  }
}

// uniforms of one long stream: one word each, so value i is word a0 + i —
// a thread per Philox block; the last thread's block becomes the state
__global__ void __launch_bounds__(256) k_np_par_doubles(NpPhilox* st, NpPhilox* st_end, double* __restrict__ out,
                                                        long long n, int mode, double lo, double hi) {
  const NpPhilox s = *st;
  const long long a0 = s.pos, jl = (a0 + n - 1) / 4;
  const double range = hi - lo;
  for (long long j = a0 / 4 + blockIdx.x * (long long)blockDim.x + threadIdx.x; j <= jl;
       j += (long long)gridDim.x * blockDim.x) {
    uint64_t w[4];
    uint64_t x0 = s.ctr[0] + (uint64_t)j, x1 = s.ctr[1], x2 = s.ctr[2], x3 = s.ctr[3];
    if (x0 < s.ctr[0] && ++x1 == 0 && ++x2 == 0) ++x3;
    if (j == 0) {
      for (int e = 0; e < 4; ++e) w[e] = s.buf[e];
    } else {
      philox_block(x0, x1, x2, x3, s.key[0], s.key[1], w[0], w[1], w[2], w[3]);
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const long long i = 4 * j + e - a0;
      if (i < 0 || i >= n) continue;
      const double u = (double)(w[e] >> 11) * (1.0 / 9007199254740992.0);
      out[i] = mode == 1 ? __dadd_rn(lo, __dmul_rn(range, u)) : u;
    }
    if (j == jl) {   // NumPy's state after the last word
      NpPhilox t = s;
      t.ctr[0] = x0; t.ctr[1] = x1; t.ctr[2] = x2; t.ctr[3] = x3;
      for (int e = 0; e < 4; ++e) t.buf[e] = w[e];
      t.pos = (int)((a0 + n - 1) % 4) + 1;
      *st_end = t;
    }
  }
}
__global__ void k_np_state_copy(NpPhilox* dst, const NpPhilox* src) { *dst = *src; }

// the chunks held fewer than N values: the rest serially, from where they ended
__global__ void __launch_bounds__(32) k_np_par_rest(ParArgs a) {
  __shared__ uint64_t ring[kRing];
  const long long have = a.tot[0];
  if (have >= a.N) {
    if (threadIdx.x == 0) *a.st = *a.st_end;
    return;
  }
  WarpGen g;
  g.load_at(*a.st, ring, threadIdx.x, a.tot[1]);
  const OutMap om = a.om;
  g.walk(0x7fffffffffffffffLL, have, a.N, [&](long long i, double x) { om.put(i, x); });
  __syncwarp();
  g.store(*a.st);
}

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

// A few long streams: the parallel walk, stream by stream (the state of
// stream c is rewritten by its own last kernel only)
// (SCH_NP_PAR=0 keeps the warp-per-stream walk: the tests compare the two)
bool par_stream(int B, long long n) {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("SCH_NP_PAR");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on && B <= 8 && n >= (1LL << 17);
}
int par_normals(sch_ctx* ctx, NpPhilox* st, long long N, const OutMap& om) {
  ParArgs a;
  a.st = st;
  a.N = N;
  static int chunk = 0;
  if (!chunk) {
    const char* e = getenv("SCH_NP_CHUNK");
    chunk = e ? atoi(e) : kChunk;
    if (chunk < 1) chunk = kChunk;
  }
  a.C = chunk;
  const long long words = N + N / 50 + 4 * kChunk;   // 1.02 words per value (1.0127 expected)
  a.K = (int)((words + a.C - 1) / a.C);
  void* ws;
  const size_t ints = ((size_t)a.K * sizeof(int) + 255) & ~size_t(255);
  const size_t lls = ((size_t)a.K * sizeof(long long) + 255) & ~size_t(255);
  int rc = sch_workspace(ctx, 3 * ints + lls + 512, &ws);
  if (rc) return rc;
  char* w = (char*)ws;
  a.cnt = (int*)w;
  a.over = (int*)(w + ints);
  a.entry = (int*)(w + 2 * ints);
  a.pref = (long long*)(w + 3 * ints);
  a.tot = (long long*)(w + 3 * ints + lls);
  a.st_end = (NpPhilox*)(w + 3 * ints + lls + 256);
  a.om = om;
  const unsigned grid = (unsigned)((a.K + kWarpsPerBlock - 1) / kWarpsPerBlock);
  k_np_par_count<<<grid, 32 * kWarpsPerBlock, 0, ctx->stream>>>(a);
  k_np_par_scan<<<1, 32, 0, ctx->stream>>>(a);
  k_np_par_emit<<<grid, 32 * kWarpsPerBlock, 0, ctx->stream>>>(a);
  k_np_par_rest<<<1, 32, 0, ctx->stream>>>(a);
  ctx->launches += 4;
  return SCH_OK;
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
  if (mode == 0 && par_stream(B, n_per_chain)) {
    for (int c = 0; c < B; ++c) {
      OutMap om{out + (long long)c * n_per_chain, nullptr, 0, 1.0, 0};
      const int rc = par_normals(ctx, (NpPhilox*)state + c, n_per_chain, om);
      if (rc) return rc;
    }
    return SCH_OK;
  }
  if (mode != 0 && par_stream(B, n_per_chain)) {   // the other warps of the launch read the old state
    void* ws;
    const int rc = sch_workspace(ctx, 256, &ws);
    if (rc) return rc;
    const unsigned grid = (unsigned)std::min<long long>((n_per_chain / 4 + 256) / 256, 148 * 8);
    for (int c = 0; c < B; ++c) {
      NpPhilox* sc = (NpPhilox*)state + c;
      k_np_par_doubles<<<grid, 256, 0, ctx->stream>>>(sc, (NpPhilox*)ws, out + (long long)c * n_per_chain,
                                                      n_per_chain, mode, lo, hi);
      k_np_state_copy<<<1, 1, 0, ctx->stream>>>(sc, (const NpPhilox*)ws);
      ctx->launches += 2;
    }
    return SCH_OK;
  }
  k_np_fill_w<<<warp_blocks(B), 32 * kWarpsPerBlock, 0, ctx->stream>>>((NpPhilox*)state, out, B,
                                                                        n_per_chain, mode, lo, hi);
  SCH_LAUNCHED(ctx);
  return SCH_OK;
}

int sch_np_heatbath(sch_ctx* ctx, void* state, double* p, double* phi, int B, long long V,
                    double phi_scale, int quenched) {
  SCH_CHECK_ARG(ctx, state && p && (phi || quenched) && B >= 1 && V >= 1, "np_heatbath: bad args");
  if (par_stream(B, 2 * V)) {
    for (int c = 0; c < B; ++c) {
      OutMap om{p + (long long)c * 2 * V, quenched ? nullptr : phi + (long long)c * 4 * V, 2 * V, phi_scale,
                quenched ? 0 : 1};
      const int rc = par_normals(ctx, (NpPhilox*)state + c, quenched ? 2 * V : 6 * V, om);
      if (rc) return rc;
    }
    return SCH_OK;
  }
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
