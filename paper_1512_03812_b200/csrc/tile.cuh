// Fused D^dag D shared-memory tile kernel (fermion.py:129-131).
//
// One CTA computes D^dag D on a TX x TT tile of one chain.  It stages the
// input spinor on the tile plus a 2-site halo (HX/HT = 2) in shared memory,
// computes D on the tile plus a 1-site halo into a second shared buffer, then
// D^dag on the tile.  A direction whose tile spans the whole lattice extent
// (HX or HT = 0) wraps periodically inside shared memory instead.
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
};

template <int TX, int TT, int HX, int HT, int MODE, int NT>
__global__ void __launch_bounds__(NT) k_normal_tile(TileArgs a) {
  constexpr int RX = TX + 2 * HX, RT = TT + 2 * HT, NR = RX * RT;
  __shared__ double2 sA[2][NR];
  __shared__ double2 sD[2][NR];
  __shared__ int gx[RX], gxm[RX], gt[RT], gtm[RT];
  __shared__ double slot[NT / 32];

  const int c = blockIdx.x / a.tiles_per_chain;
  const int tile = blockIdx.x - c * a.tiles_per_chain;
  if (MODE != MODE_PLAIN && a.flag && a.flag[c] == 0) return;
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

  double beta_c = 0.0;
  if (MODE == MODE_P) beta_c = a.beta[c];
  for (int k = threadIdx.x; k < NR; k += NT) {
    const int i = k / RT, j = k - (k / RT) * RT;
    const long long site = cbase + (long long)gx[i] * T + gt[j];
    Spinor v = ld256_spinor_nc(a.in, site);
    if (MODE == MODE_P) {
      Spinor p = ld256_spinor_nc(a.in2, site);
      v.s0 = make_double2(__fma_rn(beta_c, p.s0.x, v.s0.x), __fma_rn(beta_c, p.s0.y, v.s0.y));
      v.s1 = make_double2(__fma_rn(beta_c, p.s1.x, v.s1.x), __fma_rn(beta_c, p.s1.y, v.s1.y));
    }
    sA[0][k] = v.s0;
    sA[1][k] = v.s1;
  }
  __syncthreads();

  const double2* __restrict__ Uc = a.U + 2 * cbase;   // [2][V] of this chain
  // ---- stage 1: D on tile + 1-site halo
  constexpr int DX0 = HX / 2, DXN = RX - 2 * DX0;
  constexpr int DT0 = HT / 2, DTN = RT - 2 * DT0;
  for (int k = threadIdx.x; k < DXN * DTN; k += NT) {
    const int i = DX0 + k / DTN, j = DT0 + (k - (k / DTN) * DTN);
    const int ip = HX ? i + 1 : (i + 1 == RX ? 0 : i + 1);
    const int im = HX ? i - 1 : (i == 0 ? RX - 1 : i - 1);
    const int jp = HT ? j + 1 : (j + 1 == RT ? 0 : j + 1);
    const int jm = HT ? j - 1 : (j == 0 ? RT - 1 : j - 1);
    Spinor cc{sA[0][i * RT + j], sA[1][i * RT + j]};
    Spinor xp{sA[0][ip * RT + j], sA[1][ip * RT + j]};
    Spinor xm{sA[0][im * RT + j], sA[1][im * RT + j]};
    Spinor tp{sA[0][i * RT + jp], sA[1][i * RT + jp]};
    Spinor tm{sA[0][i * RT + jm], sA[1][i * RT + jm]};
    const int X = gx[i], Tt = gt[j];
    double2 u0 = __ldg(Uc + (long long)X * T + Tt);
    double2 u1 = __ldg(Uc + V + (long long)X * T + Tt);
    double2 u0m = __ldg(Uc + (long long)gxm[i] * T + Tt);
    double2 u1m = __ldg(Uc + V + (long long)X * T + gtm[j]);
    Spinor r = wilson_site<false>(cc, xp, xm, tp, tm, u0, u0m, u1, u1m, a.diag);
    sD[0][i * RT + j] = r.s0;
    sD[1][i * RT + j] = r.s1;
  }
  __syncthreads();

  // ---- stage 2: D^dag on the tile
  double part = 0.0;
  for (int k = threadIdx.x; k < TX * TT; k += NT) {
    const int li = k / TT, lj = k - (k / TT) * TT;
    if (x0 + li >= L || t0 + lj >= T) continue;     // clipped tile
    const int i = HX + li, j = HT + lj;
    const int ip = HX ? i + 1 : (i + 1 == RX ? 0 : i + 1);
    const int im = HX ? i - 1 : (i == 0 ? RX - 1 : i - 1);
    const int jp = HT ? j + 1 : (j + 1 == RT ? 0 : j + 1);
    const int jm = HT ? j - 1 : (j == 0 ? RT - 1 : j - 1);
    Spinor cc{sD[0][i * RT + j], sD[1][i * RT + j]};
    Spinor xp{sD[0][ip * RT + j], sD[1][ip * RT + j]};
    Spinor xm{sD[0][im * RT + j], sD[1][im * RT + j]};
    Spinor tp{sD[0][i * RT + jp], sD[1][i * RT + jp]};
    Spinor tm{sD[0][i * RT + jm], sD[1][i * RT + jm]};
    const int X = gx[i], Tt = gt[j];
    double2 u0 = __ldg(Uc + (long long)X * T + Tt);
    double2 u1 = __ldg(Uc + V + (long long)X * T + Tt);
    double2 u0m = __ldg(Uc + (long long)gxm[i] * T + Tt);
    double2 u1m = __ldg(Uc + V + (long long)X * T + gtm[j]);
    Spinor r = wilson_site<true>(cc, xp, xm, tp, tm, u0, u0m, u1, u1m, a.diag);
    const long long site = cbase + (long long)X * T + Tt;
    if (MODE == MODE_X) {
      Spinor bb = ld256_spinor_nc(a.bvec, site);
      r.s0 = csub(bb.s0, r.s0);
      r.s1 = csub(bb.s1, r.s1);
      part += spinor_norm2(r);
    } else if (MODE == MODE_P) {
      Spinor pp{sA[0][i * RT + j], sA[1][i * RT + j]};
      part += spinor_redot(pp, r);
    }
    st256_spinor(a.out, site, r);
  }
  if (MODE != MODE_PLAIN) {
    double s = block_sum<NT>(part, slot);
    if (threadIdx.x == 0) a.partial[(long long)c * a.tiles_per_chain + tile] = s;
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
  else if (T == 32 && L % 8 == 0) s = {1, 8, 32, L / 8, 1};
  else if (T == 64 && L % 4 == 0) s = {2, 4, 64, L / 4, 1};
  else if (T % 32 == 0 && L % 8 == 0 && T > 64) s = {3, 8, 32, L / 8, T / 32};
  else s = {4, 8, 16, (L + 7) / 8, (T + 15) / 16};
  return s;
}

// Launch k_normal_tile with the instantiation matching `sh`.
template <int MODE>
inline void launch_normal_tile(const TileShape& sh, const TileArgs& a, cudaStream_t st) {
  const unsigned grid = (unsigned)a.B * a.tiles_per_chain;
  switch (sh.kind) {
    case 0: k_normal_tile<16, 16, 0, 0, MODE, 256><<<grid, 256, 0, st>>>(a); break;
    case 1: k_normal_tile<8, 32, 2, 0, MODE, 256><<<grid, 256, 0, st>>>(a); break;
    case 2: k_normal_tile<4, 64, 2, 0, MODE, 256><<<grid, 256, 0, st>>>(a); break;
    case 3: k_normal_tile<8, 32, 2, 2, MODE, 256><<<grid, 256, 0, st>>>(a); break;
    default: k_normal_tile<8, 16, 2, 2, MODE, 128><<<grid, 128, 0, st>>>(a); break;
  }
}
