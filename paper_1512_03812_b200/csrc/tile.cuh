// Fused D^dag D shared-memory tile kernel (fermion.py:129-131).
//
// One CTA computes D^dag D on a TX x TT tile of one chain.  The input spinor
// is read once per cell of the tile plus a 2-site halo (HX/HT = 2); a
// direction whose tile spans the whole lattice extent (HX or HT = 0) wraps
// periodically inside shared memory instead.  Every cell is owned by one
// thread, which keeps the cell's spinor and its two links in registers and
// exports the four rank-1 projections its neighbours need (half-spinor
// exchange, see resident.cuh) — so links are read once, by their owner, and
// shared-memory traffic is 64 B stored + 64 B loaded per cell per D.
//
//   phase A : owner loads psi (256-bit), U_0, U_1; exports D-projections
//   phase B : D on the tile + 1-site halo (from the exports); re-exports the
//             D^dag-projections of t = D psi into the same buffer
//   phase C : D^dag on the tile, epilogue per MODE
//
// Compulsory HBM traffic per site: spinor in 32 B + U 32 B + out 32 B = 96 B
// (SURVEY §8(d)); halo re-reads hit L2.
//
// MODE selects the CG fusion (cg_normal, fermion.py:194-214):
//   MODE_PLAIN : out = A in
//   MODE_P     : p = r + beta_c * p_old formed on the fly;  out = A p;
//                partial[tile] = Re<p, A p>
//   MODE_X     : out(r) = b - A x;  partial[tile] = ||r||^2
// Chains whose flag is 0 are skipped (per-chain CG masking).
#pragma once

#include "common.cuh"
#include "resident.cuh"
#include "runtime.hpp"

enum { MODE_PLAIN = 0, MODE_P = 1, MODE_X = 2 };

struct TileArgs {
  const double2* __restrict__ U;    // [B][2][V]
  const double2* __restrict__ in;   // PLAIN: psi, P: r, X: x
  const double2* __restrict__ in2;  // P: p_old
  const double2* __restrict__ bvec; // X: b
  double2* __restrict__ out;        // PLAIN: A psi, P: A p, X: r
  const int* __restrict__ flag;     // per chain (P/X); null => all
  const double* __restrict__ beta;  // per chain (P)
  double* __restrict__ partial;     // [B][tiles_per_chain] (P/X)
  int B, L, T;
  int tiles_t, tiles_per_chain;
  double diag;                      // 2 + m0
  int own_lo, own_hi;               // x rows written / summed; own_hi == 0 => all rows
  // RP (decomposed lattice): instead of one partial per tile, one partial per
  // (own row, TT-wide t-chunk), [B][own_hi-own_lo][T/TT], each the canonical
  // tree sum (row_chunk_sum) of its TT site values — so the global sum
  // (dd.cu) does not depend on how the lattice is cut into strips
  double* __restrict__ rowpart;
};

// Canonical deterministic sum of TT consecutive values p[0..TT) by one warp:
// a balanced binary tree over the values in index order (zero padded to 32
// lanes), i.e. adjacent pairs first.  Every kernel that forms a row-chunk
// partial of the decomposed lattice uses this order, so the partial does
// not depend on which kernel, tile or strip produced it.
template <int TT>
SCH_DEV double row_chunk_sum(const double* p, int lane) {
  double v;
  if constexpr (TT >= 64) {
    constexpr int K = TT / 32;   // power of two
    double a[K];
#pragma unroll
    for (int k = 0; k < K; ++k) a[k] = p[lane * K + k];
#pragma unroll
    for (int w = K / 2; w >= 1; w >>= 1)
#pragma unroll
      for (int k = 0; k < w; ++k) a[k] = a[2 * k] + a[2 * k + 1];
    v = a[0];
  } else {
    v = lane < TT ? p[lane] : 0.0;
  }
  return warp_tree_sum(v);
}

template <int TX, int TT, int HX, int HT, int MODE, int NT, bool RP = false>
__device__ __forceinline__ void tile_body(const TileArgs& a, int c, int tile, double2* E, int* gx,
                                          int* gxm, int* gt, int* gtm, double* slot) {
  constexpr int RX = TX + 2 * HX, RT = TT + 2 * HT, NR = RX * RT;
  constexpr int CPT = (NR + NT - 1) / NT;   // region cells per thread
  const int tx = tile / a.tiles_t, tt = tile - tx * a.tiles_t;
  const int x0 = tx * TX, t0 = tt * TT;
  const int L = a.L, T = a.T;
  const long long V = (long long)L * T;
  const long long cbase = (long long)c * V;   // first site of this chain

  for (int i = threadIdx.x; i < RX; i += NT) {
    int v = ((x0 - HX + i) % L + L) % L;
    gx[i] = v;
    gxm[i] = v == 0 ? L - 1 : v - 1;
  }
  for (int j = threadIdx.x; j < RT; j += NT) {
    int v = ((t0 - HT + j) % T + T) % T;
    gt[j] = v;
    gtm[j] = v == 0 ? T - 1 : v - 1;
  }
  __syncthreads();

  const double2* __restrict__ Uc = a.U + 2 * cbase;   // [2][V] of this chain
  double beta_c = 0.0;
  if (MODE == MODE_P) beta_c = a.beta[c];

  // ---- phase A: owner loads; exports D projections
  Spinor v[CPT], t[CPT];
  double2 u0[CPT], u1[CPT];
#pragma unroll
  for (int j = 0; j < CPT; ++j) {
    const int k = threadIdx.x + j * NT;
    if (k >= NR) continue;
    const int ri = k / RT, rj = k - (k / RT) * RT;
    const long long s = (long long)gx[ri] * T + gt[rj];
    v[j] = ld256_spinor_nc(a.in, cbase + s);
    if (MODE == MODE_P) {
      Spinor p = ld256_spinor_nc(a.in2, cbase + s);
      v[j].s0 = make_double2(__fma_rn(beta_c, p.s0.x, v[j].s0.x), __fma_rn(beta_c, p.s0.y, v[j].s0.y));
      v[j].s1 = make_double2(__fma_rn(beta_c, p.s1.x, v[j].s1.x), __fma_rn(beta_c, p.s1.y, v[j].s1.y));
    }
    u0[j] = __ldg(Uc + s);
    u1[j] = __ldg(Uc + V + s);
    res_produce<false>(E, NR, k, v[j], u0[j], u1[j]);
  }
  __syncthreads();

  auto nb = [&](int ri, int rj, int& kxp, int& kxm, int& ktp, int& ktm) {
    const int ip = HX ? ri + 1 : (ri + 1 == RX ? 0 : ri + 1);
    const int im = HX ? ri - 1 : (ri == 0 ? RX - 1 : ri - 1);
    const int jp = HT ? rj + 1 : (rj + 1 == RT ? 0 : rj + 1);
    const int jm = HT ? rj - 1 : (rj == 0 ? RT - 1 : rj - 1);
    kxp = ip * RT + rj;
    kxm = im * RT + rj;
    ktp = ri * RT + jp;
    ktm = ri * RT + jm;
  };

  // ---- phase B: t = D v on the tile + 1-site halo
  constexpr int DX0 = HX / 2, DT0 = HT / 2;
#pragma unroll
  for (int j = 0; j < CPT; ++j) {
    const int k = threadIdx.x + j * NT;
    if (k >= NR) continue;
    const int ri = k / RT, rj = k - (k / RT) * RT;
    if (ri < DX0 || ri >= RX - DX0 || rj < DT0 || rj >= RT - DT0) continue;
    int kxp, kxm, ktp, ktm;
    nb(ri, rj, kxp, kxm, ktp, ktm);
    t[j] = res_consume<false>(E, NR, v[j], u0[j], u1[j], kxp, kxm, ktp, ktm, a.diag);
  }
  __syncthreads();   // every export of phase A consumed
#pragma unroll
  for (int j = 0; j < CPT; ++j) {
    const int k = threadIdx.x + j * NT;
    if (k >= NR) continue;
    const int ri = k / RT, rj = k - (k / RT) * RT;
    if (ri < DX0 || ri >= RX - DX0 || rj < DT0 || rj >= RT - DT0) continue;
    res_produce<true>(E, NR, k, t[j], u0[j], u1[j]);
  }
  __syncthreads();

  // ---- phase C: D^dag on the tile
  double part = 0.0;
  double cv[CPT];   // RP: per-cell values, reduced per row after the loop
#pragma unroll
  for (int j = 0; j < CPT; ++j) {
    cv[j] = 0.0;
    const int k = threadIdx.x + j * NT;
    if (k >= NR) continue;
    const int ri = k / RT, rj = k - (k / RT) * RT;
    const int li = ri - HX, lj = rj - HT;
    if (li < 0 || li >= TX || lj < 0 || lj >= TT) continue;
    if (x0 + li >= L || t0 + lj >= T) continue;     // clipped tile
    if (a.own_hi > 0 && (x0 + li < a.own_lo || x0 + li >= a.own_hi)) continue;   // DD halo row
    int kxp, kxm, ktp, ktm;
    nb(ri, rj, kxp, kxm, ktp, ktm);
    Spinor r = res_consume<true>(E, NR, t[j], u0[j], u1[j], kxp, kxm, ktp, ktm, a.diag);
    const long long site = cbase + (long long)gx[ri] * T + gt[rj];
    if (MODE == MODE_X) {
      Spinor bb = ld256_spinor_nc(a.bvec, site);
      r.s0 = csub(bb.s0, r.s0);
      r.s1 = csub(bb.s1, r.s1);
      cv[j] = spinor_norm2(r);
    } else if (MODE == MODE_P) {
      cv[j] = spinor_redot(v[j], r);
    }
    part += cv[j];
    st256_spinor(a.out, site, r);
  }
  if (MODE != MODE_PLAIN && RP) {
    __syncthreads();   // every read of the exports is done: reuse E for the cell values
    double* val = reinterpret_cast<double*>(E);   // [TX][TT]
#pragma unroll
    for (int j = 0; j < CPT; ++j) {
      const int k = threadIdx.x + j * NT;
      if (k >= NR) continue;
      const int ri = k / RT, rj = k - (k / RT) * RT;
      const int li = ri - HX, lj = rj - HT;
      if (li < 0 || li >= TX || lj < 0 || lj >= TT) continue;
      val[li * TT + lj] = cv[j];
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nown = a.own_hi - a.own_lo, nch = T / TT;
    for (int li = warp; li < TX; li += NT / 32) {
      const int x = x0 + li;
      if (x >= L || x < a.own_lo || x >= a.own_hi) continue;   // warp-uniform
      const double v = row_chunk_sum<TT>(val + li * TT, lane);
      if (lane == 0) a.rowpart[((long long)c * nown + (x - a.own_lo)) * nch + tt] = v;
    }
  } else if (MODE != MODE_PLAIN) {
    double s = block_sum<NT>(part, slot);
    if (threadIdx.x == 0) a.partial[(long long)c * a.tiles_per_chain + tile] = s;
  }
}

// One CTA per tile.
template <int TX, int TT, int HX, int HT, int MODE, int NT, int MINB, bool RP = false>
__global__ void __launch_bounds__(NT, MINB) k_normal_tile(TileArgs a) {
  constexpr int RX = TX + 2 * HX, RT = TT + 2 * HT;
  static_assert(!RP || 8 * RX * RT >= TX * TT, "row values must fit the export buffer");
  extern __shared__ double2 E[];            // [4][NR] exported projections (dynamic)
  __shared__ int gx[RX], gxm[RX], gt[RT], gtm[RT];
  __shared__ double slot[NT / 32];
  pdl_enter();
  const int c = blockIdx.x / a.tiles_per_chain;
  const int tile = blockIdx.x - c * a.tiles_per_chain;
  if (MODE != MODE_PLAIN && a.flag && a.flag[c] == 0) return;
  tile_body<TX, TT, HX, HT, MODE, NT, RP>(a, c, tile, E, gx, gxm, gt, gtm, slot);
}

// Persistent variant for sparse work (the CG true-residual pass, where only
// flagged chains have anything to do): a fixed grid strides over tiles.
template <int TX, int TT, int HX, int HT, int MODE, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) k_normal_tile_sparse(TileArgs a) {
  constexpr int RX = TX + 2 * HX, RT = TT + 2 * HT;
  extern __shared__ double2 E[];
  __shared__ int gx[RX], gxm[RX], gt[RT], gtm[RT];
  __shared__ double slot[NT / 32];
  __shared__ unsigned mask;
  pdl_enter();
  const int ntiles = a.B * a.tiles_per_chain;
  // chunks of 32 tiles: warp 0 reads the 32 flags in parallel, the CTA then
  // walks the set bits (an idle pass costs one flag read per chunk)
  for (int base = blockIdx.x * 32; base < ntiles; base += gridDim.x * 32) {
    if (threadIdx.x < 32) {
      const int w = base + threadIdx.x;
      const bool f = w < ntiles && a.flag[w / a.tiles_per_chain] != 0;
      const unsigned m = __ballot_sync(0xffffffffu, f);
      if (threadIdx.x == 0) mask = m;
    }
    __syncthreads();
    unsigned m = mask;
    while (m) {
      const int bit = __ffs(m) - 1;
      m &= m - 1;
      const int w = base + bit;
      const int c = w / a.tiles_per_chain;
      tile_body<TX, TT, HX, HT, MODE, NT>(a, c, w - c * a.tiles_per_chain, E, gx, gxm, gt, gtm, slot);
      __syncthreads();   // shared-memory readers of this tile are done
    }
    __syncthreads();     // everyone has read `mask`
  }
}

// Host-side choice of the tile shape for an L x T lattice.
struct TileShape {
  int kind;        // index into the instantiation table
  int TX, TT;
  int tiles_x, tiles_t;
};

inline TileShape pick_tile(int L, int T) {
  TileShape s;
  if (L == 16 && T == 16) s = {0, 16, 16, 1, 1};
  else if (T == 32 && L % 16 == 0) s = {10, 16, 32, L / 16, 1};   // 256 thr, 3 CTAs/SM
  else if (T == 64 && L % 8 == 0) s = {2, 8, 64, L / 8, 1};
  else if (T % 64 == 0 && T > 64) s = {3, 16, 64, (L + 15) / 16, T / 64};   // x-clipped
  else s = {4, 8, 16, (L + 7) / 8, (T + 15) / 16};
  return s;
}

template <int TX, int TT, int HX, int HT, int MODE, int NT, int MINB>
inline void launch_tile_inst(const TileArgs& a, cudaStream_t st, int sparse_grid, bool pdl) {
  constexpr int NR = (TX + 2 * HX) * (TT + 2 * HT);
  constexpr size_t smem = sizeof(double2) * 4 * NR;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_normal_tile<TX, TT, HX, HT, MODE, NT, MINB>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_normal_tile_sparse<TX, TT, HX, HT, MODE, NT, MINB>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  if (sparse_grid > 0)
    launch_k(pdl, k_normal_tile_sparse<TX, TT, HX, HT, MODE, NT, MINB>, dim3(sparse_grid), dim3(NT),
             smem, st, a);
  else
    launch_k(pdl, k_normal_tile<TX, TT, HX, HT, MODE, NT, MINB>, dim3((unsigned)a.B * a.tiles_per_chain),
             dim3(NT), smem, st, a);
}

// Decomposed lattice (dd.cu): tiles whose t-extent is the row-chunk width CW
// of the canonical row partials (CW = 64, 32, 16 or 8 by T), x-clipped, with
// RP row partials.  kind = CW.
inline bool dd_tile_shape(int Lext, int T, TileShape& s) {
  int tx, tt;
  if (T % 64 == 0) { tx = 16; tt = 64; }
  else if (T % 32 == 0) { tx = 16; tt = 32; }
  else if (T % 16 == 0) { tx = 8; tt = 16; }
  else if (T % 8 == 0) { tx = 8; tt = 8; }
  else return false;
  s = {tt, tx, tt, (Lext + tx - 1) / tx, T / tt};
  return true;
}

template <int TX, int TT, int MODE, int NT, int MINB>
inline void launch_dd_tile_inst(const TileArgs& a, cudaStream_t st) {
  constexpr int NR = (TX + 4) * (TT + 4);
  constexpr size_t smem = sizeof(double2) * 4 * NR;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_normal_tile<TX, TT, 2, 2, MODE, NT, MINB, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  k_normal_tile<TX, TT, 2, 2, MODE, NT, MINB, true>
      <<<dim3((unsigned)a.B * a.tiles_per_chain), dim3(NT), smem, st>>>(a);
}

template <int MODE>
inline void launch_dd_tile(const TileShape& sh, const TileArgs& a, cudaStream_t st) {
  switch (sh.kind) {
    case 64: launch_dd_tile_inst<16, 64, MODE, 512, 2>(a, st); break;
    case 32: launch_dd_tile_inst<16, 32, MODE, 512, 2>(a, st); break;
    case 16: launch_dd_tile_inst<8, 16, MODE, 128, 4>(a, st); break;
    default: launch_dd_tile_inst<8, 8, MODE, 128, 4>(a, st); break;
  }
}

// Launch the instantiation matching `sh`.  sparse_grid > 0 selects the
// persistent flag-skipping variant with that many CTAs.
template <int MODE>
inline void launch_normal_tile(const TileShape& sh, const TileArgs& a, cudaStream_t st,
                               int sparse_grid = 0, bool pdl = false) {
  switch (sh.kind) {
    case 0: launch_tile_inst<16, 16, 0, 0, MODE, 256, 3>(a, st, sparse_grid, pdl); break;
    case 2: launch_tile_inst<8, 64, 2, 0, MODE, 512, 2>(a, st, sparse_grid, pdl); break;
    case 3: launch_tile_inst<16, 64, 2, 2, MODE, 512, 2>(a, st, sparse_grid, pdl); break;
    case 10: launch_tile_inst<16, 32, 2, 0, MODE, 256, 3>(a, st, sparse_grid, pdl); break;
    default: launch_tile_inst<8, 16, 2, 2, MODE, 128, 4>(a, st, sparse_grid, pdl); break;
  }
}
