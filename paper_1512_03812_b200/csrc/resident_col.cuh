// Resident per-chain CG, block-owned (the 16^2 / 32^2 hot shapes).
//
// Same algorithm, stopping rule and data placement as k_cg_resident
// (resident.cuh), but each thread owns a BX x BT block of sites (BX rows in
// x, BT consecutive sites in t; block_stencil.cuh) instead of sites strided
// by the block size.  Per D application a block exports only its faces:
//   plane 0 (read by x-1): the BT sites of its first row
//   plane 1 (read by x+1): the BT sites of its last row
//   plane 2 (read by t-1): the BX sites of its first column
//   plane 3 (read by t+1): the BX sites of its last column
// i.e. 2(BX+BT) projected components per BX*BT sites instead of 4 per site
// (2x2: -50 % shared-memory traffic).  The register-only internal hops are
// summed while the exchange barrier is pending.  Planes are indexed by
// thread id: every warp-wide store and neighbour load is one contiguous (or
// lane-permuted within aligned 128-B groups) run — conflict-free.
//
// The per-iteration stopping test sqrt(rs') <= target (fermion.py:202) is
// decided without the square root unless rs' falls inside a +-4e-15 band
// around target^2, where the exact comparison is evaluated: the decision is
// the one the reference takes, at two compares per iteration.  beta = rs'/rs
// is finished from a reciprocal formed off the critical path (Markstein:
// q0 = rs'*y, rem = rs' - rs*q0 exact, q = q0 + rem*y is correctly rounded
// for y = RN(1/rs)), three dependent operations instead of a division.
#pragma once

#include <type_traits>

#include "block_stencil.cuh"

// Phase stamps of the iteration for tools/micro/resblk_phases.cu (which
// defines them as clock reads by thread 0); nothing in the library build.
#ifndef RES_STAMP
#define RES_STAMP(i)
#define RES_STAMP_BEGIN()
#define RES_STAMP_END(iters)
#endif

//
// TSH = 1 moves the t-direction faces from shared memory to warp shuffles:
// a block row of NBT = TC/BT threads is contiguous in the thread index, so
// both t-neighbours of a thread sit in its own warp (NBT divides 32).  The
// t-face hops are then added before the exchange barrier and only the
// x-faces go through shared memory (-50 % shared-memory exchange traffic).
//
// The solve is a device function (cg_resblk_run) so that the trajectory
// megakernel (mega.cu) runs the same code on its own per-chain buffers:
// chain `c` indexes the iters/relres/status outputs, `cb` is the site offset
// of the chain's fields, `sm` the dynamic shared memory (2 exchange stages).
// COH = true reads U and b with coherent loads (they were written earlier in
// the same kernel); the batched kernel uses the read-only path.
template <bool COH>
SCH_DEV double2 res_ld2(const double2* p) {
  if constexpr (COH)
    return *p;
  else
    return __ldg(p);
}
template <bool COH>
SCH_DEV Spinor res_ld_spinor(const double2* p, long long site) {
  if constexpr (COH)
    return ld256_spinor(p, site);
  else
    return ldg_spinor(p, site);
}

// Per-iteration CTA sums with a shorter dependent chain than block_sum: three
// xor-butterfly levels leave each lane holding the sum of its 8-lane residue
// class; lanes 0..3 of every warp publish those (4 per warp), and after the
// barrier every thread adds the 4*NW slots as a fixed pairwise tree (the same
// value in every thread).
template <int NW>
SCH_DEV void part4_put(double v, double* slot) {
  v += __shfl_xor_sync(0xffffffffu, v, 16);
  v += __shfl_xor_sync(0xffffffffu, v, 8);
  v += __shfl_xor_sync(0xffffffffu, v, 4);
  const int lane = threadIdx.x & 31;
  if (lane < 4) slot[(threadIdx.x >> 5) * 4 + lane] = v;
}
template <int NW>
SCH_DEV double part4_sum(const double* slot) {
  constexpr int N = 4 * NW;
  double a[N / 2];
#pragma unroll
  for (int i = 0; i < N / 2; ++i) {
    const double2 v = reinterpret_cast<const double2*>(slot)[i];
    a[i] = v.x + v.y;
  }
#pragma unroll
  for (int w = N / 4; w >= 1; w >>= 1) {
#pragma unroll
    for (int i = 0; i < w; ++i) a[i] = a[2 * i] + a[2 * i + 1];
  }
  return a[0];
}
template <int NW>
SCH_DEV double part4_block_sum(double v, double* slot) {
  part4_put<NW>(v, slot);
  __syncthreads();
  return part4_sum<NW>(slot);
}

template <int LC, int TC, int BX, int BT, int TSH, bool COH, bool ROT = false>
SCH_DEV void cg_resblk_run(const ResArgs& a, int c, long long cb, double2* sm) {
  using Blk = std::conditional_t<ROT, SiteBlockRot<BX, BT>, SiteBlock<BX, BT>>;
  // ROT: the solve runs in the sigma1-diagonal spin basis (block_stencil.cuh)
  auto ld_b = [&](long long s) {
    const Spinor v = res_ld_spinor<COH>(a.b, s);
    return ROT ? spin_rot(v) : v;
  };
  auto st_x = [&](long long s, const Spinor& v) { st_spinor(a.x, s, ROT ? spin_unrot(v) : v); };
  constexpr int SPT = Blk::SPT;
  constexpr int NT = LC * TC / SPT;
  constexpr int NBT = TC / BT, NBX = LC / BX;
  constexpr int V = LC * TC;
  constexpr int NW = NT / 32;
  constexpr int PL = (2 * BT + 2 * BX) * NT;   // double2 per exchange stage
  static_assert(TC % BT == 0 && LC % BX == 0 && NT % 32 == 0, "block shape");
  static_assert(!TSH || 32 % NBT == 0, "t-neighbours must share a warp");
  // plane offsets inside one stage
  constexpr int O0 = 0, O1 = BT * NT, O2 = 2 * BT * NT, O3 = (2 * BT + BX) * NT;
  __shared__ double red[3][NW];
  // per-iteration sums: part4_* for two-warp CTAs (16^2: 2.02 -> 1.98 ns per
  // chain-iteration); wider CTAs keep the full butterfly (32^2 with part4: 9.17 -> 10.19)
  constexpr bool P4 = NW <= 2;
  __shared__ __align__(16) double red4[2][4 * NW];
  double2* E0 = sm;
  double2* E1 = sm + PL;
  const int tid = threadIdx.x;
  const int bx = tid / NBT, bt = tid % NBT;
  auto site = [&](int k) { return (bx * BX + k / BT) * TC + bt * BT + k % BT; };
  // exchange partners (thread ids owning the neighbouring blocks)
  const int txp = ((bx + 1) % NBX) * NBT + bt;
  const int txm = ((bx + NBX - 1) % NBX) * NBT + bt;
  const int ttp = bx * NBT + (bt + 1) % NBT;
  const int ttm = bx * NBT + (bt + NBT - 1) % NBT;

  double2 u0[SPT], u1[SPT];
  Spinor x[SPT], r[SPT], p[SPT];
  double bb = 0.0;
#pragma unroll
  for (int k = 0; k < SPT; ++k) {
    u0[k] = cscale(ROT ? -1.0 : -0.5, res_ld2<COH>(a.U + 2 * cb + site(k)));   // exact: power-of-two scale
    u1[k] = cscale(-0.5, res_ld2<COH>(a.U + 2 * cb + V + site(k)));
    r[k] = ld_b(cb + site(k));
    x[k].s0 = x[k].s1 = make_double2(0, 0);
    bb += spinor_norm2(r[k]);
  }
  const double normb2 = block_sum<NT>(bb, red[0]);
  const double normb = sqrt(normb2);
  const double target = a.tol * normb;
  if (normb == 0.0) {   // fermion.py:181-182, per chain
#pragma unroll
    for (int k = 0; k < SPT; ++k) st_x(cb + site(k), x[k]);
    if (tid == 0) {
      a.iters[c] = 0;
      a.relres[c] = 0.0;
      a.status[c] = 0;
    }
    return;
  }
  const double t2 = target * target;
  const double t2lo = t2 * (1.0 - 4e-15), t2hi = t2 * (1.0 + 4e-15);

  // One exchange stage, split around its barrier: exports + interior hops
  // before, face loads + face hops after.
  const int lane_tp = ttp & 31, lane_tm = ttm & 31;
  auto stage_pre = [&](auto dag, double2* E, const Spinor* v, Spinor* out) {
    constexpr bool DAG = decltype(dag)::value;
    double2 tf[2][BX];
    Blk::template produce<DAG>(u0, u1, v, [&](int plane, int idx, double2 val) {
      constexpr int off[4] = {O0, O1, O2, O3};
      if (TSH && plane >= 2)
        tf[plane - 2][idx] = val;
      else
        E[off[plane] + idx * NT + tid] = val;
    });
    Blk::template interior<DAG>(u0, u1, v, out, a.diag);
    if constexpr (TSH) {
      double2 ft[SPT];
#pragma unroll
      for (int k = 0; k < SPT; ++k) {
        const int i = k / BT, j = k % BT;
        if (j == BT - 1) ft[k] = shfl_d2(tf[0][i], lane_tp);
        if (j == 0) ft[k] = shfl_d2(tf[1][i], lane_tm);
      }
      Blk::template faces_t<DAG>(u1, ft, out);
    }
  };
  auto stage_post = [&](auto dag, const double2* E, Spinor* out) {
    constexpr bool DAG = decltype(dag)::value;
    double2 fx[SPT], ft[SPT];
#pragma unroll
    for (int k = 0; k < SPT; ++k) {   // all face loads in flight before any math
      const int i = k / BT, j = k % BT;
      if (i == BX - 1) fx[k] = E[O0 + j * NT + txp];
      if (i == 0) fx[k] = E[O1 + j * NT + txm];
      if (!TSH && j == BT - 1) ft[k] = E[O2 + i * NT + ttp];
      if (!TSH && j == 0) ft[k] = E[O3 + i * NT + ttm];
    }
    if constexpr (TSH)
      Blk::template faces_x<DAG>(u0, fx, out);
    else
      Blk::template faces<DAG>(u0, u1, fx, ft, out);
  };
  using F = std::integral_constant<bool, false>;
  using T = std::integral_constant<bool, true>;

  // out = D^dag D v (two exchange rounds).  Precondition: every thread has
  // finished reading E0/E1 of the previous application.
  auto normal_op = [&](const Spinor* v, Spinor* out) {
    Spinor t[SPT];
    stage_pre(F{}, E0, v, t);
    __syncthreads();
    stage_post(F{}, E0, t);
    stage_pre(T{}, E1, t, out);
    __syncthreads();
    stage_post(T{}, E1, out);
  };

  Spinor w[SPT];
  double rs = normb2;   // r = b exactly: the same sum as ||b||^2 (fermion.py:186,191)
  if (a.x0) {
#pragma unroll
    for (int k = 0; k < SPT; ++k) {
      x[k] = res_ld_spinor<COH>(a.x0, cb + site(k));
      if constexpr (ROT) x[k] = spin_rot(x[k]);
    }
    normal_op(x, w);
    double rr = 0.0;
#pragma unroll
    for (int k = 0; k < SPT; ++k) {
      r[k] = sp_sub(r[k], w[k]);
      rr += spinor_norm2(r[k]);
    }
    rs = block_sum<NT>(rr, red[1]);
  }
#pragma unroll
  for (int k = 0; k < SPT; ++k) p[k] = r[k];

  double best = INFINITY;
  double inv_rs = __drcp_rn(rs);
  RES_STAMP_BEGIN();
  for (int it = 1; it <= a.maxiter; ++it) {
    RES_STAMP(0);
    // w = D^dag D p; <p, D^dag D p> formed as ||D p||^2 during the D stage
    // and published by the barrier between the stages (resident.cuh)
    {
      Spinor t[SPT];
      stage_pre(F{}, E0, p, t);
      RES_STAMP(1);
      __syncthreads();
      RES_STAMP(2);
      stage_post(F{}, E0, t);
      double dd = 0.0;
#pragma unroll
      for (int k = 0; k < SPT; ++k) dd += spinor_norm2(t[k]);
      stage_pre(T{}, E1, t, w);
      if constexpr (P4) {
        part4_put<NW>(dd, red4[0]);
      } else {
        dd = warp_sum(dd);
        if ((tid & 31) == 0) red[0][tid >> 5] = dd;
      }
      RES_STAMP(3);
      __syncthreads();
      RES_STAMP(4);
      stage_post(T{}, E1, w);
      RES_STAMP(5);
    }
    double den;
    if constexpr (P4) {
      den = part4_sum<NW>(red4[0]);
    } else {
      den = red[0][0];
#pragma unroll
      for (int q = 1; q < NW; ++q) den += red[0][q];
    }
    const double alpha = den > 0.0 ? rs / den : 0.0;
    RES_STAMP(6);
    const bool repl = (it % kResReplace) == 0;
    double nrm[SPT];
#pragma unroll
    for (int k = 0; k < SPT; ++k) {
      x[k] = sp_fma(alpha, p[k], x[k]);
      if (!repl) {
        r[k] = sp_fma(-alpha, w[k], r[k]);
        nrm[k] = spinor_norm2(r[k]);
      }
    }
    // the thread's sites summed pairwise (a shorter chain ahead of the
    // butterfly than a running sum)
#pragma unroll
    for (int h = 1; h < SPT; h *= 2) {
#pragma unroll
      for (int k = 0; k + h < SPT; k += 2 * h) nrm[k] += nrm[k + h];
    }
    const double rsn = repl ? 0.0 : nrm[0];
    double rs_new = 0.0;
    bool check = true;
    RES_STAMP(7);
    if (!repl) {
      rs_new = P4 ? part4_block_sum<NW>(rsn, red4[1]) : block_sum<NT>(rsn, red[1]);
      RES_STAMP(8);
      check = rs_new <= t2lo;
      if (!check && rs_new <= t2hi) {   // inside the band: the exact test (asm keeps
        double sq;                      // the compiler from hoisting the sqrt)
        asm volatile("sqrt.rn.f64 %0, %1;" : "=d"(sq) : "d"(rs_new));
        check = sq <= target;
      }
    }
    if (check) {   // true residual b - A x (shared with the residual replacement)
      normal_op(x, w);
      double tn2 = 0.0;
#pragma unroll
      for (int k = 0; k < SPT; ++k) {
        w[k] = sp_sub(ld_b(cb + site(k)), w[k]);
        tn2 += spinor_norm2(w[k]);
      }
      tn2 = block_sum<NT>(tn2, red[2]);
      const double tn = sqrt(tn2);
      if (!repl || tn <= target) best = tn / normb;
      if (tn <= target) {
#pragma unroll
        for (int k = 0; k < SPT; ++k) st_x(cb + site(k), x[k]);
        if (tid == 0) {
          a.iters[c] = it;
          a.relres[c] = tn / normb;
          a.status[c] = 0;
        }
        return;
      }
#pragma unroll
      for (int k = 0; k < SPT; ++k) r[k] = w[k];
      rs_new = tn2;
    }
    double beta = 0.0;   // Markstein-finished rs'/rs (header comment)
    if (rs > 0.0) {
      const double q0 = rs_new * inv_rs;
      beta = __fma_rn(__fma_rn(-rs, q0, rs_new), inv_rs, q0);
    }
#pragma unroll
    for (int k = 0; k < SPT; ++k) p[k] = sp_fma(beta, p[k], r[k]);
    rs = rs_new;
    inv_rs = __drcp_rn(rs);
    RES_STAMP(9);
  }
  RES_STAMP_END(a.maxiter);
#pragma unroll
  for (int k = 0; k < SPT; ++k) st_x(cb + site(k), x[k]);
  if (tid == 0) {
    a.iters[c] = a.maxiter;
    a.relres[c] = fmin(best, sqrt(rs) / normb);
    a.status[c] = 1;
  }
}

template <int LC, int TC, int BX, int BT, int MINB, int TSH = 0, bool ROT = false>
__global__ void __launch_bounds__(LC * TC / (BX * BT), MINB) k_cg_resblk(ResArgs a) {
  extern __shared__ double2 sm[];
  cg_resblk_run<LC, TC, BX, BT, TSH, false, ROT>(a, blockIdx.x, (long long)blockIdx.x * LC * TC, sm);
}
