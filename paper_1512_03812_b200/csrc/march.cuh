// Warp-marching fused D^dag D for the decomposed lattice (BASELINE
// configs[4]: rows of T = 2048 sites; fermion.py:129-131, fermion.py:194).
//
// The tile kernels (tile.cuh, tma2d.cuh) stage a 2-D region in shared memory
// and run D, then D^dag, as barrier-separated phases of a CTA: at 2048^2
// they reach 49-55 % of HBM, bound by those phases (ncu: barrier and
// short-scoreboard stalls) and not by the memory system.  Here there is no
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
// in a register ring, which is what keeps HBM busy: a warp always has PF
// rows (2-3 KiB) in flight and an SM holds 12-16 such warps.  The redundant
// work is the 4 halo lanes (12.5 %, L1/L2 hits: the 4 warps of a CTA own
// adjacent bands) and the 4 pipeline-fill rows per segment.
//
// Arithmetic per site is res_produce / res_consume's (resident.cuh), in the
// same order.  MODE as in tile.cuh:
//   MODE_PLAIN : out = A in
//   MODE_P     : v = in + beta in2 formed on the fly; out = A v; <v, A v>
//   MODE_X     : out = bvec - A in; ||out||^2
//   MODE_PU    : MODE_P that also stores v as the new search direction and
//                applies the PREVIOUS iteration's solution update
//                x += alpha_prev p_old on the rows it owns ("Deferred
//                solution update" in dd.cu): the CG iteration then moves
//                320 B/site instead of 352.
//
// NS > 0 replaces the register ring by a per-lane shared-memory ring: every
// lane copies its own 16-B words of a row with cp.async (LDGSTS) into its own
// slots and reads them back itself after cp.async.wait_group, so there is
// still no barrier; NS - 1 rows per warp are in flight without holding
// registers (MODE_PU's four streams need more bytes in flight than the
// register file can land).
// Row partials (P, X): one per aligned group of kMarchCW = 4 columns,
// ((c0 + c1) + (c2 + c3)) — a complete subtree of the canonical tree over the
// T columns of a row (dd.cu: C_c(C_t(.)) is the same balanced tree for every
// power-of-two chunk width), written as [strip][own row][T / 4].
#pragma once

#include "tile.cuh"
#include "tma_tile.cuh"

constexpr int kMarchW = 28;    // output columns per warp (32 lanes - 2 x 2 halo)
constexpr int kMarchCW = 4;    // columns per row partial
constexpr int kMarchWarps = 4; // warps per CTA (adjacent column bands)
constexpr int MODE_PU = 3;

struct MarchArgs {
  TileArgs t;     // B = strips, L = Lext, T, own_lo/own_hi, diag, in/in2/bvec/out, beta, flag, rowpart
  int nbt;        // column bands per row: ceil(T / kMarchW)
  int nbx;        // row segments per strip
  int R;          // rows per segment
  // MODE_PU: the two direction buffers (the iteration's parity, ctl[3] & 1,
  // says which one holds p_old; v goes to the other), the solution and the
  // pending alpha (0 when nothing is pending); t.in2 is unused
  double2* pbuf[2];
  double2* xq;
  const double* xalpha;
  const int* ctl;
};

template <int MODE>
struct MarchRaw {   // one loaded row, as it arrived (no arithmetic: the loads stay in flight)
  Spinor v, p, x;
  double2 u0, u1;
};

// 16-B words per lane and row
template <int MODE>
struct MarchWords {
  static constexpr int value = MODE == MODE_PU ? 8 : MODE == MODE_P ? 6 : 4;
};

// `pold`: the second input field (MODE_P: t.in2; MODE_PU: the p_old buffer);
// `xq`: the solution, loaded only for rows this warp will write (wr)
template <int MODE>
SCH_DEV MarchRaw<MODE> march_load(const TileArgs& t, const double2* pold, const double2* xq, bool wr,
                                  long long srow, long long urow, int col) {
  MarchRaw<MODE> r;
  r.v = ld256_spinor_nc(t.in, srow + col);
  if (MODE == MODE_P || MODE == MODE_PU) r.p = ld256_spinor_nc(pold, srow + col);
  if (MODE == MODE_PU && wr) r.x = ld256_spinor(xq, srow + col);
  r.u0 = __ldg(t.U + urow + col);
  r.u1 = __ldg(t.U + urow + (long long)t.L * t.T + col);
  return r;
}

SCH_DEV void cp_async16(uint32_t sdst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sdst), "l"(gsrc) : "memory");
}
SCH_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
SCH_DEV void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
SCH_DEV double2 lds_d2(uint32_t a) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
  return v;
}

// the same row into a shared-memory slot (word w of lane l at slot + 512 w + 16 l)
template <int MODE>
SCH_DEV void march_issue(const TileArgs& t, const double2* pold, const double2* xq, bool wr,
                         long long srow, long long urow, int col, uint32_t slot) {
  const double2* v = t.in + 2 * (srow + col);
  cp_async16(slot, v);
  cp_async16(slot + 512, v + 1);
  cp_async16(slot + 1024, t.U + urow + col);
  cp_async16(slot + 1536, t.U + urow + (long long)t.L * t.T + col);
  if (MODE == MODE_P || MODE == MODE_PU) {
    const double2* p = pold + 2 * (srow + col);
    cp_async16(slot + 2048, p);
    cp_async16(slot + 2560, p + 1);
  }
  if (MODE == MODE_PU && wr) {
    const double2* x = xq + 2 * (srow + col);
    cp_async16(slot + 3072, x);
    cp_async16(slot + 3584, x + 1);
  }
}
template <int MODE>
SCH_DEV MarchRaw<MODE> march_fetch(uint32_t slot, bool wr) {
  MarchRaw<MODE> r;
  r.v.s0 = lds_d2(slot);
  r.v.s1 = lds_d2(slot + 512);
  r.u0 = lds_d2(slot + 1024);
  r.u1 = lds_d2(slot + 1536);
  if (MODE == MODE_P || MODE == MODE_PU) {
    r.p.s0 = lds_d2(slot + 2048);
    r.p.s1 = lds_d2(slot + 2560);
  }
  if (MODE == MODE_PU && wr) {
    r.x.s0 = lds_d2(slot + 3072);
    r.x.s1 = lds_d2(slot + 3584);
  }
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
  double2 o0 = cadd(cadd(cadd(hf0, hb0), hf1), hb1);
  double2 o1 = DAG ? cadd(csub(hf0, hb0), cmuli(csub(hf1, hb1)))
                   : cadd(csub(hb0, hf0), cmuli(csub(hb1, hf1)));
  Spinor r;
  r.s0 = make_double2(diag * v.s0.x - 0.5 * o0.x, diag * v.s0.y - 0.5 * o0.y);
  r.s1 = make_double2(diag * v.s1.x - 0.5 * o1.x, diag * v.s1.y - 0.5 * o1.y);
  return r;
}

template <int MODE, int PF, int MINB, int NS>
__global__ void __launch_bounds__(32 * kMarchWarps, MINB) k_dd_march(const MarchArgs a) {
  const TileArgs& t = a.t;
  // the true-residual pass has work only when the stop test asked for it
  if (MODE == MODE_X && t.flag != nullptr && t.flag[0] == 0) return;
  if (MODE == MODE_PU && a.ctl[0]) return;   // solve finished: x and p stay as they are
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
  constexpr bool PM = MODE == MODE_P || MODE == MODE_PU;   // v = in + beta p_old, <v, A v>
  double beta = 0.0, xal = 0.0;
  if (PM) beta = t.beta[s];
  const double2* pold = t.in2;
  double2* pnew = nullptr;
  if (MODE == MODE_PU) {
    const int par = a.ctl[3] & 1;
    pold = a.pbuf[par];
    pnew = a.pbuf[par ^ 1];
    xal = *a.xalpha;
  }
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
  // MODE_PU: the rows whose v and x this warp stores — its own rows, and the
  // strip's halo rows in the first / last segment (so p and x stay current
  // on every extended row, as k_dd_update keeps them)
  const int w0 = bx == 0 ? a0 : x0, w1 = bx == a.nbx - 1 ? a1 + 1 : x1;
  auto wr_row = [&](int r) { return r >= w0 && r < w1; };

  // one step: row `ar` has arrived as `raw`
  auto step = [&](int ar, const MarchRaw<MODE>& raw) {
    Spinor bvec;
    const int xo = ar - 2;   // the row whose output completes in this step
    const bool row_out = xo >= x0;
    if (MODE == MODE_X && row_out && lane_out) bvec = ld256_spinor_nc(t.bvec, sbase + (long long)xo * T + col);

    Spinor vn = raw.v;
    if (PM) {
      vn.s0 = make_double2(__fma_rn(beta, raw.p.s0.x, vn.s0.x), __fma_rn(beta, raw.p.s0.y, vn.s0.y));
      vn.s1 = make_double2(__fma_rn(beta, raw.p.s1.x, vn.s1.x), __fma_rn(beta, raw.p.s1.y, vn.s1.y));
    }
    if (MODE == MODE_PU && wr_row(ar) && lane_out) {   // the new direction; the pending x update
      const long long i = sbase + (long long)ar * T + col;
      st256_spinor(pnew, i, vn);
      Spinor xv = raw.x;
      xv.s0 = make_double2(__fma_rn(xal, raw.p.s0.x, xv.s0.x), __fma_rn(xal, raw.p.s0.y, xv.s0.y));
      xv.s1 = make_double2(__fma_rn(xal, raw.p.s1.x, xv.s1.x), __fma_rn(xal, raw.p.s1.y, xv.s1.y));
      st256_spinor(a.xq, i, xv);
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
        } else if (PM) {
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
    if (PM) vp = vc;
    vc = vn;
    u0c = raw.u0;
    u1c = raw.u1;
  };

  if constexpr (NS == 0) {
    MarchRaw<MODE> ring[PF];
#pragma unroll
    for (int k = 0; k < PF; ++k)
      if (a0 + k <= a1)
        ring[k] = march_load<MODE>(t, pold, a.xq, wr_row(a0 + k), sbase + (long long)(a0 + k) * T,
                                   ubase + (long long)(a0 + k) * T, col);
    for (int ab = a0; ab <= a1; ab += PF) {
#pragma unroll
      for (int k = 0; k < PF; ++k) {
        const int ar = ab + k;
        if (ar > a1) break;   // warp-uniform
        const MarchRaw<MODE> raw = ring[k];
        if (ar + PF <= a1)
          ring[k] = march_load<MODE>(t, pold, a.xq, wr_row(ar + PF), sbase + (long long)(ar + PF) * T,
                                     ubase + (long long)(ar + PF) * T, col);
        step(ar, raw);
      }
    }
  } else {
    // shared-memory ring of NS slots per warp, NS - 1 rows in flight: the row
    // of step ar is fetched from its slot, then row ar + NS - 1 is issued into
    // the slot read one step earlier (whose values have long been consumed)
    extern __shared__ __align__(16) char march_smem[];
    constexpr uint32_t SLOT = 512u * MarchWords<MODE>::value;
    const uint32_t wbase = smem_u32(march_smem) + (threadIdx.x >> 5) * (NS * SLOT) + lane * 16;
#pragma unroll
    for (int k = 0; k < NS - 1; ++k) {
      if (a0 + k <= a1)
        march_issue<MODE>(t, pold, a.xq, wr_row(a0 + k), sbase + (long long)(a0 + k) * T,
                          ubase + (long long)(a0 + k) * T, col, wbase + k * SLOT);
      cp_async_commit();
    }
    int slot = 0;
    for (int ar = a0; ar <= a1; ++ar) {
      cp_async_wait<NS - 2>();
      const MarchRaw<MODE> raw = march_fetch<MODE>(wbase + slot * SLOT, wr_row(ar));
      const int prev = slot == 0 ? NS - 1 : slot - 1;
      if (ar + NS - 1 <= a1)
        march_issue<MODE>(t, pold, a.xq, wr_row(ar + NS - 1), sbase + (long long)(ar + NS - 1) * T,
                          ubase + (long long)(ar + NS - 1) * T, col, wbase + prev * SLOT);
      cp_async_commit();
      step(ar, raw);
      slot = slot + 1 == NS ? 0 : slot + 1;
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
// SCH_DD_DEFER=1: the deferred solution update (MODE_PU + k_dd_update_r; measured slower, off)
inline bool march_defer_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SCH_DD_DEFER");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}
// (the row sums combine up to 2048 partials per row: dd.cu warp_canon)
inline bool march_shape_ok(int T) { return T % 8 == 0 && T / kMarchCW <= 2048; }
inline int march_nch(int T) { return T / kMarchCW; }

template <int MODE, int PF, int MINB, int NS = 0>
inline bool launch_dd_march_inst(const TileArgs& t, cudaStream_t st, int num_sms,
                                 const MarchArgs* extra = nullptr) {
  MarchArgs a{};
  if (extra) a = *extra;
  a.t = t;
  a.nbt = (t.T + kMarchW - 1) / kMarchW;
  const int nown = t.own_hi - t.own_lo;
  constexpr int SMEM = NS * 512 * MarchWords<MODE>::value * kMarchWarps;
  // row segments: as many warps as one wave holds, so no CTA waits for a slot
  // (a segment costs 4 pipeline-fill rows: not shorter than 16 rows)
  static int per_sm = 0;
  if (!per_sm) {
    if (SMEM > 0)
      cudaFuncSetAttribute(k_dd_march<MODE, PF, MINB, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_dd_march<MODE, PF, MINB, NS>,
                                                      32 * kMarchWarps, SMEM) != cudaSuccess || per_sm < 1)
      per_sm = 1;
  }
  const long long slots = (long long)num_sms * per_sm * kMarchWarps;
  int nbx = (int)std::max<long long>(1, slots / ((long long)t.B * a.nbt));
  int R = std::max(16, (nown + nbx - 1) / nbx);
  if (const char* e = getenv("SCH_DD_MARCH_R")) R = std::max(1, atoi(e));
  a.R = R;
  a.nbx = (nown + R - 1) / R;
  const long long warps = (long long)t.B * a.nbt * a.nbx;
  const unsigned grid = (unsigned)((warps + kMarchWarps - 1) / kMarchWarps);
  k_dd_march<MODE, PF, MINB, NS><<<grid, 32 * kMarchWarps, SMEM, st>>>(a);
  return true;
}

template <int MODE>
inline bool launch_dd_march(const TileArgs& t, cudaStream_t st, int num_sms,
                            const MarchArgs* extra = nullptr) {
  static int v = -1;   // tuning: SCH_DD_MARCH_V = 10 * PF + MINB (register ring), 100 * NS + MINB (shared ring)
  if (v < 0) {
    const char* e = getenv(MODE == MODE_P || MODE == MODE_PU ? "SCH_DD_MARCH_V" : "SCH_DD_MARCH_V0");
    v = e ? atoi(e) : (MODE == MODE_PU ? 22 : 42);
  }
  switch (v) {
    case 22: return launch_dd_march_inst<MODE, 2, 2>(t, st, num_sms, extra);
    case 23: return launch_dd_march_inst<MODE, 2, 3>(t, st, num_sms, extra);
    case 32: return launch_dd_march_inst<MODE, 3, 2>(t, st, num_sms, extra);
    case 402: return launch_dd_march_inst<MODE, 1, 2, 4>(t, st, num_sms, extra);
    case 602: return launch_dd_march_inst<MODE, 1, 2, 6>(t, st, num_sms, extra);
    case 403: return launch_dd_march_inst<MODE, 1, 3, 4>(t, st, num_sms, extra);
    case 503: return launch_dd_march_inst<MODE, 1, 3, 5>(t, st, num_sms, extra);
    case 304: return launch_dd_march_inst<MODE, 1, 4, 3>(t, st, num_sms, extra);
    case 404: return launch_dd_march_inst<MODE, 1, 4, 4>(t, st, num_sms, extra);
    default: return launch_dd_march_inst<MODE, 4, 2>(t, st, num_sms, extra);
  }
}
