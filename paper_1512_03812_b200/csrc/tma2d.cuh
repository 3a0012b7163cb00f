// Persistent, TMA-pipelined fused D^dag D on 2-D tiles with a t-halo: the
// decomposed lattice's D^dag D and its CG stencil pass (BASELINE configs[4]:
// rows of T = 2048 sites; fermion.py:129-131, fermion.py:194).
//
// k_normal_tma (tma_tile.cuh) needs tiles of whole time rows; the
// decomposed lattice's rows are 2048 sites long, and the one-tile-per-CTA
// halo kernel (k_normal_tile) leaves HBM idle while its CTAs compute (ncu:
// 49 % of HBM, long-scoreboard stalls).  Here a fixed grid walks the tiles;
// one elected thread loads each tile's region — TX+4 rows x TT+4 columns of
// every input field — with ONE 3-D tensor copy per field
// (cp.async.bulk.tensor, SASS UTMALDG; box {components, columns, rows})
// into stage s of a 2-deep shared-memory ring, completing on that stage's
// mbarrier, while the CTA computes the previous tile out of the other stage.
// The periodic t-wrap of the first and last band: the main box reads zeros
// out of bounds, and a 2-column side box from the other end of the row
// supplies the wrapped halo columns.
//
// Per tile: phase A (owners read cells from the stage, export the rank-1
// projections of D), B (D on the tile + 1-site halo, export D^dag's), C
// (D^dag on the tile, own rows only; out and per MODE the row-chunk partials
// of the canonical tree, tile.cuh row_chunk_sum over the TT columns).  Same
// res_produce / res_consume arithmetic as k_normal_tile, so the values are
// the halo-tile kernel's bit for bit.
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>

#include "tile.cuh"
#include "tma_tile.cuh"

template <int TX, int TT, int MODE>
struct Tma2dGeom {
  static constexpr int RX = TX + 4, RT = TT + 4, NR = RX * RT;
  static constexpr int NSP = MODE == MODE_P ? 2 : 1;
  static constexpr int CELL_B = 32 * NSP + 32;            // spinor field(s) + U_0 + U_1
  static constexpr int SIDE = RX * 2;                     // cells of one side box
  // box destinations 128-B aligned for every field (8 cells of 16 B)
  static constexpr int NRP = (NR + 7) / 8 * 8, SIDEP = (SIDE + 7) / 8 * 8;
  static constexpr int NS = NRP + 2 * SIDEP;              // cells per field block
  static constexpr int STAGE_B = NS * CELL_B;
  static constexpr int E_B = 4 * NR * 16;
  static constexpr int SMEM = 2 * STAGE_B + E_B;
};

// tensor maps of one pass: [0] in, [1] in2 (P), [2] U; each with its main
// box and its 2-column side box
struct Tma2dMaps {
  CUtensorMap in, in2, u, in_side, in2_side, u_side;
};

struct Tma2dArgs {
  TileArgs t;          // B = strips, L = Lext, T, own_lo/own_hi, diag, out, bvec, beta, rowpart
  int tiles_x, tiles_t;
};

SCH_DEV void tma3d_g2s(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

// stage layout: per field a block of NS cells: the main box (row-major
// RX x RT), then the left side box (RX x 2), then the right one, each
// starting on a 128-B boundary (a TMA destination requirement)
template <int TX, int TT, int MODE>
SCH_DEV void tma2d_issue(const Tma2dArgs& a, const Tma2dMaps& m, int w, char* st, uint64_t* bar) {
  using G = Tma2dGeom<TX, TT, MODE>;
  const int per = a.tiles_x * a.tiles_t;
  const int s = w / per, r = w - s * per;
  const int tx = r / a.tiles_t, tt = r - tx * a.tiles_t;
  const int T = a.t.T;
  const int row0 = s * a.t.L + a.t.own_lo + tx * TX - 2;   // spinor rows: strip-major
  const int urow0 = s * 2 * a.t.L + a.t.own_lo + tx * TX - 2;
  const int t0 = tt * TT - 2;
  const bool left = t0 < 0, right = t0 + G::RT > T;
  const uint32_t cells = G::NR + (left ? G::SIDE : 0) + (right ? G::SIDE : 0);
  mbar_arrive_expect_tx(bar, cells * (uint32_t)G::CELL_B);
  char* f = st;
  constexpr int NS = G::NS, L0 = G::NRP, R0 = G::NRP + G::SIDEP;
  tma3d_g2s(f, &m.in, 0, t0, row0, bar);
  if (left) tma3d_g2s(f + L0 * 32, &m.in_side, 0, T - 2, row0, bar);
  if (right) tma3d_g2s(f + R0 * 32, &m.in_side, 0, 0, row0, bar);
  f += NS * 32;
  if (MODE == MODE_P) {
    tma3d_g2s(f, &m.in2, 0, t0, row0, bar);
    if (left) tma3d_g2s(f + L0 * 32, &m.in2_side, 0, T - 2, row0, bar);
    if (right) tma3d_g2s(f + R0 * 32, &m.in2_side, 0, 0, row0, bar);
    f += NS * 32;
  }
  for (int d = 0; d < 2; ++d) {   // U_0 then U_1: planes of Lext rows
    const int ur = urow0 + d * a.t.L;
    tma3d_g2s(f, &m.u, 0, t0, ur, bar);
    if (left) tma3d_g2s(f + L0 * 16, &m.u_side, 0, T - 2, ur, bar);
    if (right) tma3d_g2s(f + R0 * 16, &m.u_side, 0, 0, ur, bar);
    f += NS * 16;
  }
}

template <int TX, int TT, int MODE, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB)
    k_dd_tma2d(const __grid_constant__ Tma2dArgs a, const __grid_constant__ Tma2dMaps maps) {
  using G = Tma2dGeom<TX, TT, MODE>;
  constexpr int RX = G::RX, RT = G::RT, NR = G::NR, NS = G::NS;
  constexpr int CPT = (NR + NT - 1) / NT;
  extern __shared__ __align__(128) char smem[];
  char* ring = smem;
  double2* E = reinterpret_cast<double2*>(smem + 2 * G::STAGE_B);
  __shared__ __align__(8) uint64_t bars[2];
  const TileArgs& t = a.t;
  const int T = t.T;
  const int per = a.tiles_x * a.tiles_t;
  const int ntiles = t.B * per;
  const int nown = t.own_hi - t.own_lo, nch = T / TT;
  // the true-residual pass runs every CG iteration but has work only when the
  // (global) stop test asked for it: exit before any load
  if (MODE == MODE_X && t.flag != nullptr && t.flag[0] == 0) return;
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
    for (int s = 0; s < 2; ++s) {
      const int w = blockIdx.x + s * gridDim.x;
      if (w < ntiles) tma2d_issue<TX, TT, MODE>(a, maps, w, ring + s * G::STAGE_B, &bars[s]);
    }
  }
  __syncthreads();

  int it = 0;
  for (int w = blockIdx.x; w < ntiles; w += gridDim.x, ++it) {
    const int stage = it & 1;
    const uint32_t parity = (uint32_t)((it >> 1) & 1);
    const int s = w / per, r = w - s * per;
    const int tx = r / a.tiles_t, tt = r - tx * a.tiles_t;
    const int x0 = t.own_lo + tx * TX, t0 = tt * TT;
    const bool left = t0 - 2 < 0, right = t0 - 2 + RT > T;
    const char* st = ring + stage * G::STAGE_B;
    double beta = 0.0;
    if (MODE == MODE_P) beta = t.beta[s];
    // cell k of the region -> its index in a field block (side boxes for the wrap)
    auto slot = [&](int ri, int rj) {
      if (left && rj < 2) return G::NRP + ri * 2 + rj;
      if (right && rj >= RT - 2) return G::NRP + G::SIDEP + ri * 2 + (rj - (RT - 2));
      return ri * RT + rj;
    };
    mbar_wait(&bars[stage], parity);

    // ---- phase A: owners read their cells, export D's projections
    Spinor v[CPT], tv[CPT];
    double2 u0[CPT], u1[CPT];
#pragma unroll
    for (int j = 0; j < CPT; ++j) {
      const int k = threadIdx.x + j * NT;
      if (k >= NR) continue;
      const int ri = k / RT, rj = k - (k / RT) * RT;
      const int q = slot(ri, rj);
      v[j] = reinterpret_cast<const Spinor*>(st)[q];
      const char* fu = st + NS * 32 * G::NSP;
      if (MODE == MODE_P) {
        const Spinor p = reinterpret_cast<const Spinor*>(st + NS * 32)[q];
        v[j].s0 = make_double2(__fma_rn(beta, p.s0.x, v[j].s0.x), __fma_rn(beta, p.s0.y, v[j].s0.y));
        v[j].s1 = make_double2(__fma_rn(beta, p.s1.x, v[j].s1.x), __fma_rn(beta, p.s1.y, v[j].s1.y));
      }
      u0[j] = reinterpret_cast<const double2*>(fu)[q];
      u1[j] = reinterpret_cast<const double2*>(fu + NS * 16)[q];
      res_produce<false>(E, NR, k, v[j], u0[j], u1[j]);
    }
    __syncthreads();   // stage consumed; exports visible
    if (threadIdx.x == 0) {
      const int wn = w + 2 * gridDim.x;
      if (wn < ntiles) {
        fence_proxy_async();
        tma2d_issue<TX, TT, MODE>(a, maps, wn, ring + stage * G::STAGE_B, &bars[stage]);
      }
    }
    // ---- phase B: D on the tile + 1-site halo
#pragma unroll
    for (int j = 0; j < CPT; ++j) {
      const int k = threadIdx.x + j * NT;
      if (k >= NR) continue;
      const int ri = k / RT, rj = k - (k / RT) * RT;
      if (ri < 1 || ri >= RX - 1 || rj < 1 || rj >= RT - 1) continue;
      tv[j] = res_consume<false>(E, NR, v[j], u0[j], u1[j], k + RT, k - RT, k + 1, k - 1, t.diag);
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < CPT; ++j) {
      const int k = threadIdx.x + j * NT;
      if (k >= NR) continue;
      const int ri = k / RT, rj = k - (k / RT) * RT;
      if (ri < 1 || ri >= RX - 1 || rj < 1 || rj >= RT - 1) continue;
      res_produce<true>(E, NR, k, tv[j], u0[j], u1[j]);
    }
    __syncthreads();
    // ---- phase C: D^dag on the tile's own rows
    double cv[CPT];
#pragma unroll
    for (int j = 0; j < CPT; ++j) {
      cv[j] = 0.0;
      const int k = threadIdx.x + j * NT;
      if (k >= NR) continue;
      const int ri = k / RT, rj = k - (k / RT) * RT;
      const int li = ri - 2, lj = rj - 2;
      if (li < 0 || li >= TX || lj < 0 || lj >= TT) continue;
      if (x0 + li >= t.own_hi) continue;   // clipped last tile of the strip
      Spinor o = res_consume<true>(E, NR, tv[j], u0[j], u1[j], k + RT, k - RT, k + 1, k - 1, t.diag);
      const long long site = ((long long)s * t.L + x0 + li) * T + t0 + lj;
      if (MODE == MODE_X) {
        const Spinor bb = ld256_spinor_nc(t.bvec, site);
        o.s0 = csub(bb.s0, o.s0);
        o.s1 = csub(bb.s1, o.s1);
        cv[j] = spinor_norm2(o);
      } else if (MODE == MODE_P) {
        cv[j] = spinor_redot(v[j], o);
      }
      st256_spinor(t.out, site, o);
    }
    if (MODE != MODE_PLAIN) {
      __syncthreads();   // every read of the exports is done: E holds the cell values
      double* val = reinterpret_cast<double*>(E);   // [TX][TT]
#pragma unroll
      for (int j = 0; j < CPT; ++j) {
        const int k = threadIdx.x + j * NT;
        if (k >= NR) continue;
        const int ri = k / RT, rj = k - (k / RT) * RT;
        const int li = ri - 2, lj = rj - 2;
        if (li < 0 || li >= TX || lj < 0 || lj >= TT) continue;
        val[li * TT + lj] = cv[j];
      }
      __syncthreads();
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
      for (int li = warp; li < TX; li += NT / 32) {
        const int x = x0 + li;
        if (x >= t.own_hi) continue;   // warp-uniform
        const double vsum = row_chunk_sum<TT>(val + li * TT, lane);
        if (lane == 0) t.rowpart[((long long)s * nown + (x - t.own_lo)) * nch + tt] = vsum;
      }
    }
    __syncthreads();   // E is rewritten by the next tile's phase A
  }
}

// ---------------------------------------------------------------- host side
// cuTensorMapEncodeTiled through the runtime's driver entry point (the
// library links cudart statically and does not link libcuda)
inline PFN_cuTensorMapEncodeTiled_v12000 tma2d_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// rows x T sites of `comp` doubles, box {comp, cols, box_rows}
inline bool tma2d_map(CUtensorMap* m, const void* base, int comp, long long rows, int T, int cols,
                      int box_rows) {
  auto enc = tma2d_encoder();
  if (!enc) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)comp, (cuuint64_t)T, (cuuint64_t)rows};
  const cuuint64_t strides[2] = {(cuuint64_t)comp * 8, (cuuint64_t)comp * 8 * T};
  const cuuint32_t box[3] = {(cuuint32_t)comp, (cuuint32_t)cols, (cuuint32_t)box_rows};
  const cuuint32_t es[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

constexpr int kT2T = 32;   // tile columns (row partials per 32 columns: the same canonical tree)

inline bool tma2d_shape_ok(int Lloc, int T) {
  (void)Lloc;
  return T % kT2T == 0 && tma2d_encoder() != nullptr;
}

// Launch one pass over S strips of Lext x T (own rows [own_lo, own_hi)).
template <int TX, int TT, int MODE, int NT, int MINB>
inline bool launch_dd_tma2d_inst(const TileArgs& t, cudaStream_t st, int num_sms) {
  using G = Tma2dGeom<TX, TT, MODE>;
  Tma2dArgs a;
  a.t = t;
  a.tiles_x = (t.own_hi - t.own_lo + TX - 1) / TX;
  a.tiles_t = t.T / TT;
  Tma2dMaps m;
  const long long srows = (long long)t.B * t.L, urows = 2LL * t.B * t.L;
  if (!tma2d_map(&m.in, t.in, 4, srows, t.T, G::RT, G::RX)) return false;
  if (!tma2d_map(&m.in_side, t.in, 4, srows, t.T, 2, G::RX)) return false;
  if (MODE == MODE_P) {
    if (!tma2d_map(&m.in2, t.in2, 4, srows, t.T, G::RT, G::RX)) return false;
    if (!tma2d_map(&m.in2_side, t.in2, 4, srows, t.T, 2, G::RX)) return false;
  } else {
    m.in2 = m.in;
    m.in2_side = m.in_side;
  }
  if (!tma2d_map(&m.u, t.U, 2, urows, t.T, G::RT, G::RX)) return false;
  if (!tma2d_map(&m.u_side, t.U, 2, urows, t.T, 2, G::RX)) return false;
  static int per_sm = 0;   // resident CTAs per SM (shared memory bound for MODE_P)
  if (!per_sm) {
    cudaFuncSetAttribute(k_dd_tma2d<TX, TT, MODE, NT, MINB>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_dd_tma2d<TX, TT, MODE, NT, MINB>,
                                                      NT, G::SMEM) != cudaSuccess || per_sm < 1)
      per_sm = 1;
  }
  const int ntiles = t.B * a.tiles_x * a.tiles_t;
  const int grid = std::min(ntiles, num_sms * per_sm);
  k_dd_tma2d<TX, TT, MODE, NT, MINB><<<grid, NT, G::SMEM, st>>>(a, m);
  return true;
}

// SCH_DD_TMA2D=0 runs the one-tile-per-CTA halo kernel instead (A/B runs)
inline bool tma2d_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SCH_DD_TMA2D");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

// Shapes measured on cfg5 (2048^2, profiles/r02/README.md): the D^dag D with
// 8 x 32 tiles, 256 threads (2 CTAs/SM by shared memory: 3.64 TB/s with the
// halo exchange vs 3.37 for the halo-tile kernel); the CG's stencil pass
// (two input spinor fields: 2 x 80 KB stages) with 16 x 32 tiles, 512
// threads, 1 CTA/SM (0.334 vs 0.355 ms per CG iteration).  Smaller tiles at
// 2 CTAs/SM, 8 x 32 at 1 CTA/SM with 128/448 threads, 12 x 32 and 4 x 32:
// 0.337-0.425 ms.  The true-residual pass (MODE_X, one input field + b read
// at the output) takes the D^dag D's shape; when the stop test did not ask
// for it, its CTAs exit before loading anything.
template <int MODE>
inline bool launch_dd_tma2d(const TileArgs& t, cudaStream_t st, int num_sms) {
  if constexpr (MODE == MODE_P) return launch_dd_tma2d_inst<16, 32, MODE, 512, 1>(t, st, num_sms);
  else return launch_dd_tma2d_inst<8, 32, MODE, 256, 1>(t, st, num_sms);   // PLAIN, X: one field
}
