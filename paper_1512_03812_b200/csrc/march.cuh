// Warp-marching fused D^dag D for the decomposed lattice (BASELINE
// configs[4]: rows of T = 2048 sites; fermion.py:129-131, fermion.py:194).
//
// The tile kernels (tile.cuh; round 2's TMA-pipelined 2-D variant) stage a
// 2-D region in shared memory and run D, then D^dag, as barrier-separated
// phases of a CTA: at 2048^2 they reach 49-55 % of HBM, bound by those
// phases (ncu: barrier and short-scoreboard stalls) and not by the memory
// system.  Here there is no
// shared memory and no barrier: a WARP owns a band of kMarchW = 28 time
// columns (lane l holds column c0 - 2 + l, i.e. the band plus the two halo
// columns D^dag D needs on either side) and marches down the x rows of its
// segment.  Per arriving input row a it
//   * forms t = D v on row a-1 from the three rows it holds in registers
//     (x-hops from the rows above and below; t-hops from the neighbouring
//     lanes by warp shuffle: two double2 shuffles per stage), and
//   * forms out = D^dag t on row a-2 the same way from the last three t rows,
// so every input value is loaded once per warp (coalesced 1-KiB spinor rows
// and 512-B link rows), D v never leaves the register file and the output
// row is stored as one 896-B run.  Loads run PF rows ahead of the arithmetic
// in a register ring, which is what keeps HBM busy: a warp always has PF = 4
// rows (2-3 KiB each) in flight and an SM holds 8 such warps.  The redundant
// work is the 4 halo lanes (12.5 %, L1/L2 hits: the 4 warps of a CTA own
// adjacent bands) and the 4 pipeline-fill rows per segment.
//
// Arithmetic per site is res_produce / res_consume's (resident.cuh), in the
// same order and through the same helpers (cmul, cmulc, spinor_redot), so the
// compiler contracts the multiply-adds as it does in the tile kernels.  MODE
// as in tile.cuh:
//   MODE_PLAIN : out = A in
//   MODE_P     : v = in + beta in2 formed on the fly; out = A v; <v, A v>
//   MODE_X     : out = bvec - A in; ||out||^2
// Row partials (P, X): one per aligned group of kMarchCW = 4 columns,
// ((c0 + c1) + (c2 + c3)) — a complete subtree of the canonical tree over the
// T columns of a row (dd.cu: C_c(C_t(.)) is the same balanced tree for every
// power-of-two chunk width), written as [strip][own row][T / 4].
#pragma once

#include "tile.cuh"

constexpr int kMarchW = 28;    // output columns per warp (32 lanes - 2 x 2 halo)
constexpr int kMarchCW = 4;    // columns per row partial
constexpr int kMarchWarps = 4; // warps per CTA (adjacent column bands)

struct MarchArgs {
  TileArgs t;     // B = strips, L = Lext, T, own_lo/own_hi, diag, in/in2/bvec/out, beta, flag, rowpart
  int nbt;        // column bands per row: ceil(T / kMarchW)
  int nbx;        // row segments per strip
  int R;          // rows per segment
};

template <int MODE>
struct MarchRaw {   // one loaded row, as it arrived (no arithmetic: the loads stay in flight)
  Spinor v, p;
  double2 u0, u1;
};

template <int MODE>
SCH_DEV MarchRaw<MODE> march_load(const TileArgs& t, long long srow, long long urow, int col) {
  MarchRaw<MODE> r;
  r.v = ld256_spinor_nc(t.in, srow + col);
  if (MODE == MODE_P) r.p = ld256_spinor_nc(t.in2, srow + col);
  r.u0 = __ldg(t.U + urow + col);
  r.u1 = __ldg(t.U + urow + (long long)t.L * t.T + col);
  return r;
}

SCH_DEV double2 shfl_dn_d2(double2 v) {
  return make_double2(__shfl_down_sync(0xffffffffu, v.x, 1), __shfl_down_sync(0xffffffffu, v.y, 1));
}
SCH_DEV double2 shfl_up_d2(double2 v) {
  return make_double2(__shfl_up_sync(0xffffffffu, v.x, 1), __shfl_up_sync(0xffffffffu, v.y, 1));
}

// res_consume's expression (resident.cuh) on hops already in registers
template <bool DAG>
SCH_DEV Spinor march_consume(const Spinor& v, double2 hf0, double2 hb0, double2 hf1, double2 hb1,
                             double diag) {
  const double2 o0 = cadd(cadd(cadd(hf0, hb0), hf1), hb1);
  const double2 o1 = DAG ? cadd(csub(hf0, hb0), cmuli(csub(hf1, hb1)))
                         : cadd(csub(hb0, hf0), cmuli(csub(hb1, hf1)));
  Spinor r;
  r.s0 = make_double2(diag * v.s0.x - 0.5 * o0.x, diag * v.s0.y - 0.5 * o0.y);
  r.s1 = make_double2(diag * v.s1.x - 0.5 * o1.x, diag * v.s1.y - 0.5 * o1.y);
  return r;
}

template <int MODE, int PF, int MINB>
__global__ void __launch_bounds__(32 * kMarchWarps, MINB) k_dd_march(const MarchArgs a) {
  const TileArgs& t = a.t;
  // the true-residual pass has work only when the stop test asked for it
  if (MODE == MODE_X && t.flag != nullptr && t.flag[0] == 0) return;
  const int lane = threadIdx.x & 31;
  const long long w = (long long)blockIdx.x * kMarchWarps + (threadIdx.x >> 5);
  const long long per = (long long)a.nbt * a.nbx;
  if (w >= per * t.B) return;   // warp-uniform; no barriers in this kernel
  const int s = (int)(w / per);
  const int rr = (int)(w - s * per);
  const int bx = rr / a.nbt, bt = rr - bx * a.nbt;
  const int T = t.T;
  const int c0 = bt * kMarchW;
  int col = c0 - 2 + lane;            // periodic in t
  col = col < 0 ? col + T : col;
  col = col % T;
  const int x0 = t.own_lo + bx * a.R;
  const int x1 = min(x0 + a.R, t.own_hi);
  const int nown = t.own_hi - t.own_lo, nch = T / kMarchCW;
  const bool lane_out = lane >= 2 && lane < 2 + kMarchW && c0 + (lane - 2) < T;
  double beta = 0.0;
  if (MODE == MODE_P) beta = t.beta[s];
  const double diag = t.diag;
  const long long sbase = (long long)s * t.L * T;        // spinor rows of strip s
  const long long ubase = (long long)s * 2 * t.L * T;    // U_0 plane of strip s

  // register pipeline: rows a-1 (c: v, links, to be hit by D) and a-2 (p: t = D v, links)
  const double2 z = make_double2(0.0, 0.0);
  Spinor vc{z, z}, vp{z, z}, tp{z, z};
  double2 u0c = z, u1c = z, u0p = z, u1p = z;
  double2 Bp = z;    // conj(U_0) w+0(v) of row a-2: the backward x-hop into row a-1
  double2 Bdp = z;   // conj(U_0) w-0(t) of row a-3: the backward x-hop of D^dag into row a-2

  const int a0 = x0 - 2, a1 = x1 + 1;   // arriving rows (extended indices, inside the halo)
  MarchRaw<MODE> ring[PF];
#pragma unroll
  for (int k = 0; k < PF; ++k)
    if (a0 + k <= a1)
      ring[k] = march_load<MODE>(t, sbase + (long long)(a0 + k) * T, ubase + (long long)(a0 + k) * T, col);

  for (int ab = a0; ab <= a1; ab += PF) {
#pragma unroll
    for (int k = 0; k < PF; ++k) {
      const int ar = ab + k;
      if (ar > a1) break;   // warp-uniform
      const MarchRaw<MODE> raw = ring[k];
      if (ar + PF <= a1)
        ring[k] = march_load<MODE>(t, sbase + (long long)(ar + PF) * T, ubase + (long long)(ar + PF) * T, col);
      Spinor bvec;
      const int xo = ar - 2;   // the row whose output completes in this step
      const bool row_out = xo >= x0;
      if (MODE == MODE_X && row_out && lane_out) bvec = ld256_spinor_nc(t.bvec, sbase + (long long)xo * T + col);

      Spinor vn = raw.v;
      if (MODE == MODE_P) {
        vn.s0 = make_double2(__fma_rn(beta, raw.p.s0.x, vn.s0.x), __fma_rn(beta, raw.p.s0.y, vn.s0.y));
        vn.s1 = make_double2(__fma_rn(beta, raw.p.s1.x, vn.s1.x), __fma_rn(beta, raw.p.s1.y, vn.s1.y));
      }
      // ---- t = D v on row a-1
      Spinor tc;
      double2 Bc;
      {
        const double2 hf0 = cmul(u0c, wminus0(vn));
        const double2 hf1 = cmul(u1c, shfl_dn_d2(wminus1(vc)));
        const double2 hb1 = shfl_up_d2(cmulc(u1c, wplus1(vc)));
        tc = march_consume<false>(vc, hf0, Bp, hf1, hb1, diag);
        Bc = cmulc(u0c, wplus0(vc));
      }
      // ---- out = D^dag t on row a-2
      Spinor o;
      double2 Bd;
      {
        const double2 hf0 = cmul(u0p, wplus0(tc));
        const double2 hf1 = cmul(u1p, shfl_dn_d2(wplus1(tp)));
        const double2 hb1 = shfl_up_d2(cmulc(u1p, wminus1(tp)));
        o = march_consume<true>(tp, hf0, Bdp, hf1, hb1, diag);
        Bd = cmulc(u0p, wminus0(tp));
      }
      if (row_out) {   // warp-uniform
        double cv = 0.0;
        if (lane_out) {
          if (MODE == MODE_X) {
            o.s0 = csub(bvec.s0, o.s0);
            o.s1 = csub(bvec.s1, o.s1);
            cv = spinor_norm2(o);
          } else if (MODE == MODE_P) {
            cv = spinor_redot(vp, o);
          }
          st256_spinor(t.out, sbase + (long long)xo * T + col, o);
        }
        if (MODE != MODE_PLAIN) {
          cv += __shfl_down_sync(0xffffffffu, cv, 1);
          cv += __shfl_down_sync(0xffffffffu, cv, 2);
          if (lane_out && ((lane - 2) & 3) == 0)
            t.rowpart[((long long)s * nown + (xo - t.own_lo)) * nch + (c0 + lane - 2) / kMarchCW] = cv;
        }
      }
      // ---- rotate the pipeline
      Bdp = Bd;
      Bp = Bc;
      tp = tc;
      u0p = u0c;
      u1p = u1c;
      if (MODE == MODE_P) vp = vc;
      vc = vn;
      u0c = raw.u0;
      u1c = raw.u1;
    }
  }
}

// SCH_DD_MARCH=0 keeps the shared-memory tile kernels (A/B runs)
inline bool march_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SCH_DD_MARCH");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}
// (the row sums combine up to 2048 partials per row: dd.cu warp_canon)
inline bool march_shape_ok(int T) { return T % 8 == 0 && T / kMarchCW <= 2048; }
inline int march_nch(int T) { return T / kMarchCW; }

// Measured on cfg5 (2048^2, profiles/r02/README.md): a 4-row register ring at
// 2 CTAs/SM (8 warps per SM, ~96 KB of loads in flight per SM) is the best of
// PF 1-6 x 2-4 CTAs/SM for all three modes; deeper rings spill, more warps
// with shallower rings keep fewer bytes in flight.  Shared-memory rings fed by
// per-lane cp.async or by per-warp TMA bulk copies, and L2 prefetches ahead
// of the ring, all measured slower.
template <int MODE, int PF = 4, int MINB = 2>
inline bool launch_dd_march(const TileArgs& t, cudaStream_t st, int num_sms) {
  MarchArgs a;
  a.t = t;
  a.nbt = (t.T + kMarchW - 1) / kMarchW;
  const int nown = t.own_hi - t.own_lo;
  // row segments: as many warps as one wave holds, so no CTA waits for a slot
  // (a segment costs 4 pipeline-fill rows: not shorter than 16 rows)
  static int per_sm = 0;
  if (!per_sm) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_dd_march<MODE, PF, MINB>,
                                                      32 * kMarchWarps, 0) != cudaSuccess || per_sm < 1)
      per_sm = 1;
  }
  const long long slots = (long long)num_sms * per_sm * kMarchWarps;
  const int nbx = (int)std::max<long long>(1, slots / ((long long)t.B * a.nbt));
  a.R = std::max(16, (nown + nbx - 1) / nbx);
  a.nbx = (nown + a.R - 1) / a.R;
  const long long warps = (long long)t.B * a.nbt * a.nbx;
  const unsigned grid = (unsigned)((warps + kMarchWarps - 1) / kMarchWarps);
  k_dd_march<MODE, PF, MINB><<<grid, 32 * kMarchWarps, 0, st>>>(a);
  return true;
}
