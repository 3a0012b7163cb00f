// Persistent, TMA-pipelined fused D^dag D (fermion.py:129-131) — the HBM
// stream version of k_normal_tile.
//
// A fixed grid of CTAs walks the tiles of all chains.  For every tile one
// elected thread issues 1-D bulk copies (cp.async.bulk, sm_90+/sm_100a TMA
// path: SASS UBLKCP) of the tile's input rows — spinor, U_0, U_1, and for the
// CG stencil pass also p_old — into stage s of an S-deep shared-memory ring,
// completing on that stage's mbarrier.  While stage s is in flight the CTA
// computes the previous tile out of its own stage: the owner of each cell
// loads the cell from shared memory, exports the four rank-1 projections
// (half-spinor exchange, resident.cuh), and phases B/C of k_normal_tile
// follow.  Tiles span whole time rows (HT = 0: T in {16, 32, 64}) and TX
// rows plus a 2-row halo in x, so each tile is at most 3 contiguous row
// ranges per field (wrap at the chain boundary).
//
// Bytes per site (PLAIN): psi 32 + U 32 in, 32 out = 96 (+ halo rows from L2).
#pragma once

#include "common.cuh"
#include "resident.cuh"
#include "tile.cuh"

SCH_DEV uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

SCH_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

SCH_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

SCH_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

SCH_DEV void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

SCH_DEV void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

SCH_DEV void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

// Shared-memory footprint of one pipeline stage and of the whole kernel.
template <int TX, int T_, int MODE>
struct TmaGeom {
  static constexpr int RX = TX + 4, NR = RX * T_;
  static constexpr int SPIN_B = NR * 32;                       // one spinor field
  static constexpr int LINK_B = NR * 16;                       // one link direction
  static constexpr int STAGE_B = SPIN_B * (MODE == MODE_P ? 2 : 1) + 2 * LINK_B;
  static constexpr int E_B = 4 * NR * 16;
};

// Issue the bulk copies of tile `w` into stage buffer `st` (one thread).
template <int TX, int T_, int MODE>
SCH_DEV void tma_issue_tile(const TileArgs& a, int w, char* st, uint64_t* bar) {
  using G = TmaGeom<TX, T_, MODE>;
  const int c = w / a.tiles_per_chain;
  const int x0 = (w - c * a.tiles_per_chain) * TX;
  const int L = a.L;
  const long long V = (long long)L * T_;
  const long long cb = (long long)c * V;
  if (a.flag != nullptr && a.flag[c] == 0) {   // converged chain: complete the phase, no data
    mbar_arrive_expect_tx(bar, 0u);
    return;
  }
  mbar_arrive_expect_tx(bar, (uint32_t)G::STAGE_B);
  // region rows x0-2 .. x0+TX+1 (mod L) as contiguous row ranges
  int i = 0;
  while (i < G::RX) {
    const int gx = ((x0 - 2 + i) % L + L) % L;
    int n = min(G::RX - i, L - gx);        // rows until the chain wraps
    const long long s0 = (long long)gx * T_;
    const uint32_t cells = (uint32_t)n * T_;
    const int k0 = i * T_;
    char* dst = st;
    bulk_g2s(dst + (size_t)k0 * 32, a.in + 2 * (cb + s0), cells * 32, bar);
    dst += G::SPIN_B;
    if (MODE == MODE_P) {
      bulk_g2s(dst + (size_t)k0 * 32, a.in2 + 2 * (cb + s0), cells * 32, bar);
      dst += G::SPIN_B;
    }
    bulk_g2s(dst + (size_t)k0 * 16, a.U + 2 * cb + s0, cells * 16, bar);
    dst += G::LINK_B;
    bulk_g2s(dst + (size_t)k0 * 16, a.U + 2 * cb + V + s0, cells * 16, bar);
    i += n;
  }
}

#ifndef SCH_TMA_TSH
#define SCH_TMA_TSH 1
#endif
constexpr bool tma_tsh_enabled = SCH_TMA_TSH != 0;   // build with -DSCH_TMA_TSH=0 for the SMEM t-faces

template <int TX, int T_, int MODE, int NT, int STAGES, int MINB = 1>
__global__ void __launch_bounds__(NT, MINB) k_normal_tma(TileArgs a) {
  using G = TmaGeom<TX, T_, MODE>;
  constexpr int RX = G::RX, RT = T_, NR = G::NR;
  constexpr int CPT = (NR + NT - 1) / NT;
  constexpr bool TSH = T_ <= 32 && 32 % T_ == 0 && NT % 32 == 0 && NR % 32 == 0 && tma_tsh_enabled;
  extern __shared__ __align__(128) char smem[];
  char* ring = smem;                                            // STAGES x STAGE_B
  double2* E = reinterpret_cast<double2*>(smem + STAGES * G::STAGE_B);
  __shared__ __align__(8) uint64_t bars[STAGES];
  __shared__ double slot[NT / 32];

  const int ntiles = a.B * a.tiles_per_chain;
  const int L = a.L;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      const int w = blockIdx.x + s * gridDim.x;
      if (w < ntiles) tma_issue_tile<TX, T_, MODE>(a, w, ring + s * G::STAGE_B, &bars[s]);
    }
  }

  int it = 0;
  for (int w = blockIdx.x; w < ntiles; w += gridDim.x, ++it) {
    const int stage = it % STAGES;
    const uint32_t parity = (uint32_t)((it / STAGES) & 1);
    const int c = w / a.tiles_per_chain;
    const int tile = w - c * a.tiles_per_chain;
    const int x0 = tile * TX;
    const long long V = (long long)L * T_;
    const long long cbase = (long long)c * V;
    const char* st = ring + stage * G::STAGE_B;
    const Spinor* sPsi = reinterpret_cast<const Spinor*>(st);
    const Spinor* sPold = reinterpret_cast<const Spinor*>(st + G::SPIN_B);
    const double2* sU0 = reinterpret_cast<const double2*>(st + G::SPIN_B * (MODE == MODE_P ? 2 : 1));
    const double2* sU1 = sU0 + NR;
    const bool active = MODE == MODE_PLAIN || a.flag == nullptr || a.flag[c] != 0;
    double beta_c = 0.0;
    if (MODE == MODE_P) beta_c = a.beta[c];

    mbar_wait(&bars[stage], parity);

    // ---- phase A: owner reads its cells from the stage, exports projections
    // TSH: a time row (T_ <= 32 cells) lies inside one warp, lane % T_ = t,
    // so the t-direction exports move by warp shuffle and only the x ones
    // go through shared memory (E planes 0/1).
    Spinor v[CPT], t[CPT];
    double2 u0[CPT], u1[CPT];
    double2 tf[CPT], tb[CPT];
    const int lane = threadIdx.x & 31;
    const int lrow = lane & ~(T_ - 1), lt = lane & (T_ - 1);
    const int lane_tp = lrow | ((lt + 1) & (T_ - 1)), lane_tm = lrow | ((lt + T_ - 1) & (T_ - 1));
#pragma unroll
    for (int j = 0; j < CPT; ++j) {
      const int k = threadIdx.x + j * NT;
      if (k >= NR) continue;
      v[j] = sPsi[k];
      if (MODE == MODE_P) {
        const Spinor p = sPold[k];
        v[j].s0 = make_double2(__fma_rn(beta_c, p.s0.x, v[j].s0.x), __fma_rn(beta_c, p.s0.y, v[j].s0.y));
        v[j].s1 = make_double2(__fma_rn(beta_c, p.s1.x, v[j].s1.x), __fma_rn(beta_c, p.s1.y, v[j].s1.y));
      }
      u0[j] = sU0[k];
      u1[j] = sU1[k];
      if (active) {
        if constexpr (TSH) res_produce_x<false>(E, NR, k, v[j], u0[j], u1[j], tf[j], tb[j]);
        else res_produce<false>(E, NR, k, v[j], u0[j], u1[j]);
      }
    }
    __syncthreads();   // stage fully consumed; exports visible
    if (threadIdx.x == 0) {
      const int wn = w + STAGES * gridDim.x;
      if (wn < ntiles) {
        fence_proxy_async();
        tma_issue_tile<TX, T_, MODE>(a, wn, ring + stage * G::STAGE_B, &bars[stage]);
      }
    }
    if (active) {
      // ---- phase B: t = D v on rows 1 .. RX-2 (tile + 1-row halo)
#pragma unroll
      for (int j = 0; j < CPT; ++j) {
        const int k = threadIdx.x + j * NT;
        if (k >= NR) continue;   // warp-uniform (NR % 32 == 0 under TSH)
        double2 f1n, b1n;
        if constexpr (TSH) {     // every lane of the warp takes part
          f1n = tile_shfl_d2(tf[j], lane_tp);
          b1n = tile_shfl_d2(tb[j], lane_tm);
        }
        const int ri = k / RT, rj = k - (k / RT) * RT;
        if (ri < 1 || ri >= RX - 1) continue;
        if constexpr (TSH) {
          t[j] = res_consume_tsh<false>(E, NR, v[j], u0[j], u1[j], k + RT, k - RT, f1n, b1n, a.diag);
        } else {
          const int jp = rj + 1 == RT ? 0 : rj + 1, jm = rj == 0 ? RT - 1 : rj - 1;
          t[j] = res_consume<false>(E, NR, v[j], u0[j], u1[j], k + RT, k - RT, ri * RT + jp,
                                    ri * RT + jm, a.diag);
        }
      }
    }
    __syncthreads();
    if (active) {
#pragma unroll
      for (int j = 0; j < CPT; ++j) {
        const int k = threadIdx.x + j * NT;
        if (k >= NR) continue;
        const int ri = k / RT;
        if (ri < 1 || ri >= RX - 1) {
          if constexpr (TSH) tf[j] = tb[j] = make_double2(0.0, 0.0);   // never consumed
          continue;
        }
        if constexpr (TSH) res_produce_x<true>(E, NR, k, t[j], u0[j], u1[j], tf[j], tb[j]);
        else res_produce<true>(E, NR, k, t[j], u0[j], u1[j]);
      }
    }
    __syncthreads();
    // ---- phase C: D^dag on the tile rows 2 .. RX-3
    double part = 0.0;
    if (active) {
#pragma unroll
      for (int j = 0; j < CPT; ++j) {
        const int k = threadIdx.x + j * NT;
        if (k >= NR) continue;
        double2 f1n, b1n;
        if constexpr (TSH) {
          f1n = tile_shfl_d2(tf[j], lane_tp);
          b1n = tile_shfl_d2(tb[j], lane_tm);
        }
        const int ri = k / RT, rj = k - (k / RT) * RT;
        if (ri < 2 || ri >= RX - 2 || x0 + ri - 2 >= L) continue;
        Spinor r;
        if constexpr (TSH) {
          r = res_consume_tsh<true>(E, NR, t[j], u0[j], u1[j], k + RT, k - RT, f1n, b1n, a.diag);
        } else {
          const int jp = rj + 1 == RT ? 0 : rj + 1, jm = rj == 0 ? RT - 1 : rj - 1;
          r = res_consume<true>(E, NR, t[j], u0[j], u1[j], k + RT, k - RT, ri * RT + jp,
                                ri * RT + jm, a.diag);
        }
        const long long site = cbase + (long long)(x0 + ri - 2) * RT + rj;
        if (MODE == MODE_X) {
          Spinor bb = ld256_spinor_nc(a.bvec, site);
          r.s0 = csub(bb.s0, r.s0);
          r.s1 = csub(bb.s1, r.s1);
          part += spinor_norm2(r);
        } else if (MODE == MODE_P) {
          part += spinor_redot(v[j], r);
        }
        st256_spinor(a.out, site, r);
      }
    }
    if (MODE != MODE_PLAIN) {
      const double s = block_sum<NT>(part, slot);   // includes a barrier
      if (active && threadIdx.x == 0) a.partial[(long long)c * a.tiles_per_chain + tile] = s;
    } else {
      __syncthreads();   // E is rewritten by the next tile's phase A
    }
  }
}

// Host: shapes handled by the TMA path (whole time rows, x tiles of TX rows).
// T = 32 (cfg2): 8 x 32 tiles, 128 threads, 2 stages, 3 CTAs/SM — measured
// best of 16x32/512/1, 8x32/256/3, 4x32/256/3, 8x32/384/2, 8x32/192/3
// (profiles/r01/README.md).
inline bool tma_tile_shape(int L, int T, int& TX) {
  if (T == 32 && L % 8 == 0) { TX = 8; return true; }
  if (T == 16 && L % 16 == 0) { TX = 16; return true; }
  if (T == 64 && L % 4 == 0) { TX = 4; return true; }
  return false;
}

template <int TX, int T_, int MODE, int NT, int STAGES, int MINB>
inline int launch_tma_inst(const TileArgs& a, cudaStream_t st, int num_sms) {
  using G = TmaGeom<TX, T_, MODE>;
  constexpr size_t smem = (size_t)STAGES * G::STAGE_B + G::E_B;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_normal_tma<TX, T_, MODE, NT, STAGES, MINB>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  const int ntiles = a.B * a.tiles_per_chain;
  const int want = num_sms * MINB;
  const int grid = ntiles < want ? ntiles : want;
  k_normal_tma<TX, T_, MODE, NT, STAGES, MINB><<<grid, NT, smem, st>>>(a);
  return 0;
}

// Launch the TMA-pipelined D^dag D for (L, T) if supported; returns false otherwise.
//   T=32: 8 x 32 tiles (RX = 12), 128 threads, 3 CTAs/SM
//   T=16: 16 x 16 tiles (RX = 20), 320 threads, 2 CTAs/SM
//   T=64: 4 x 64 tiles (RX = 8), 512 threads, 2 CTAs/SM
template <int MODE>
inline bool launch_normal_tma(const TileArgs& a, cudaStream_t st, int num_sms) {
  int TX = 0;
  if (!tma_tile_shape(a.L, a.T, TX)) return false;
  constexpr int S = MODE == MODE_P ? 2 : 3;
  if (a.T == 32) {
    launch_tma_inst<8, 32, MODE, 128, 2, 3>(a, st, num_sms);
  } else if (a.T == 16) {
    launch_tma_inst<16, 16, MODE, 320, S, 2>(a, st, num_sms);
  } else {
    launch_tma_inst<4, 64, MODE, 512, 2, 2>(a, st, num_sms);
  }
  return true;
}
