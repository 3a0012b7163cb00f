// Resident per-chain CG, column-owned variant (the 16^2 / 32^2 hot shapes).
//
// Same algorithm, stopping rule and data placement as k_cg_resident
// (resident.cuh), but each thread owns SPT t-consecutive sites of one x row
// ("column segment") instead of SPT sites strided by the block size.  The
// t-hops between a thread's own sites then never leave its registers: per
// D application a segment exports
//   plane 0 / plane 1 (read by x-1 / x+1)  for all SPT sites
//   plane 2           (read by t-1)        for its first site only
//   plane 3           (read by t+1)        for its last site only
// i.e. 2*SPT+2 projected components instead of 4*SPT (SPT=2: -25 % shared
// memory traffic, SPT=4: -37.5 %).  Shared-memory planes are indexed by
// thread id, so every warp-wide store and neighbour load touches one
// contiguous (or 8-lane-permuted) 512-B run: conflict-free.
//
// The per-iteration stopping test sqrt(rs') <= target (fermion.py:202) is
// decided without the square root unless rs' falls inside a +-4e-15 band
// around target^2, where the exact comparison is evaluated: the decision is
// the one the reference takes, at two compares per iteration.
#pragma once

#include "resident.cuh"

template <int LC, int TC, int SPT, int MINB>
__global__ void __launch_bounds__(LC * TC / SPT, MINB) k_cg_rescol(ResArgs a) {
  constexpr int NT = LC * TC / SPT;
  constexpr int NSEG = TC / SPT;
  constexpr int V = LC * TC;
  constexpr int NW = NT / 32;
  constexpr int PL = (2 * SPT + 2) * NT;   // double2 per exchange stage
  static_assert(TC % SPT == 0 && NT % 32 == 0, "segment shape");
  extern __shared__ double2 sm[];
  __shared__ double red[3][NW];
  double2* E0 = sm;
  double2* E1 = sm + PL;
  const int tid = threadIdx.x;
  const int c = blockIdx.x;
  const long long cb = (long long)c * V;
  const int xx = tid / NSEG, seg = tid % NSEG;
  const int s0 = xx * TC + seg * SPT;
  // exchange partners (thread ids owning the neighbouring segments)
  const int txp = ((xx + 1) % LC) * NSEG + seg;
  const int txm = ((xx + LC - 1) % LC) * NSEG + seg;
  const int ttp = xx * NSEG + (seg + 1) % NSEG;
  const int ttm = xx * NSEG + (seg + NSEG - 1) % NSEG;
  constexpr int OX1 = SPT * NT, OT0 = 2 * SPT * NT, OT1 = (2 * SPT + 1) * NT;

  double2 u0[SPT], u1[SPT];
  Spinor x[SPT], r[SPT], p[SPT];
  double bb = 0.0;
#pragma unroll
  for (int k = 0; k < SPT; ++k) {
    u0[k] = cscale(-0.5, __ldg(a.U + 2 * cb + s0 + k));   // exact: power-of-two scale
    u1[k] = cscale(-0.5, __ldg(a.U + 2 * cb + V + s0 + k));
    r[k] = ldg_spinor(a.b, cb + s0 + k);
    x[k].s0 = x[k].s1 = make_double2(0, 0);
    bb += spinor_norm2(r[k]);
  }
  const double normb2 = block_sum<NT>(bb, red[0]);
  const double normb = sqrt(normb2);
  const double target = a.tol * normb;
  if (normb == 0.0) {   // fermion.py:181-182, per chain
#pragma unroll
    for (int k = 0; k < SPT; ++k) st_spinor(a.x, cb + s0 + k, x[k]);
    if (tid == 0) {
      a.iters[c] = 0;
      a.relres[c] = 0.0;
      a.status[c] = 0;
    }
    return;
  }
  const double t2 = target * target;
  const double t2lo = t2 * (1.0 - 4e-15), t2hi = t2 * (1.0 + 4e-15);

  // ---- one D (DAG=false) or D^dag (DAG=true) exchange stage
  // produce: write this segment's exports of v into E, keep the t-internal
  // ones in registers
  auto produce = [&](auto dag, double2* E, const Spinor* v, double2* f2, double2* f3) {
    constexpr bool DAG = decltype(dag)::value;
#pragma unroll
    for (int k = 0; k < SPT; ++k) {
      E[k * NT + tid] = DAG ? wplus0(v[k]) : wminus0(v[k]);
      E[OX1 + k * NT + tid] = cmulc(u0[k], DAG ? wminus0(v[k]) : wplus0(v[k]));
      const double2 a2 = DAG ? wplus1(v[k]) : wminus1(v[k]);
      const double2 a3 = cmulc(u1[k], DAG ? wminus1(v[k]) : wplus1(v[k]));
      if (k == 0) E[OT0 + tid] = a2;
      else f2[k] = a2;
      if (k == SPT - 1) E[OT1 + tid] = a3;
      else f3[k] = a3;
    }
  };
  auto gather = [&](const double2* E, const double2* f2, const double2* f3, Hops* h) {
#pragma unroll
    for (int k = 0; k < SPT; ++k) {
      h[k].f0 = E[k * NT + txp];
      h[k].b0 = E[OX1 + k * NT + txm];
      h[k].f1 = (k == SPT - 1) ? E[OT0 + ttp] : f2[k + 1];
      h[k].b1 = (k == 0) ? E[OT1 + ttm] : f3[k - 1];
    }
  };
  using F = std::integral_constant<bool, false>;
  using T = std::integral_constant<bool, true>;

  // out = D^dag D v (two exchange rounds).  Precondition: every thread has
  // finished reading E0/E1 of the previous application.
  auto normal_op = [&](const Spinor* v, Spinor* out) {
    double2 f2[SPT], f3[SPT];
    Hops h[SPT];
    produce(F{}, E0, v, f2, f3);
    __syncthreads();
    gather(E0, f2, f3, h);
#pragma unroll
    for (int k = 0; k < SPT; ++k) out[k] = res_combine<false>(h[k], v[k], u0[k], u1[k], a.diag);
    produce(T{}, E1, out, f2, f3);
    __syncthreads();
    gather(E1, f2, f3, h);
#pragma unroll
    for (int k = 0; k < SPT; ++k) out[k] = res_combine<true>(h[k], out[k], u0[k], u1[k], a.diag);
  };

  Spinor w[SPT];
  double rs = normb2;   // r = b exactly: the same sum as ||b||^2 (fermion.py:186,191)
  if (a.x0) {
#pragma unroll
    for (int k = 0; k < SPT; ++k) x[k] = ldg_spinor(a.x0, cb + s0 + k);
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
  for (int it = 1; it <= a.maxiter; ++it) {
    // w = D^dag D p; <p, D^dag D p> formed as ||D p||^2 during the D stage
    // and published by the barrier between the stages (resident.cuh)
    double2 f2[SPT], f3[SPT];
    Hops h[SPT];
    produce(F{}, E0, p, f2, f3);
    __syncthreads();
    gather(E0, f2, f3, h);
    double dd = 0.0;
#pragma unroll
    for (int k = 0; k < SPT; ++k) {
      w[k] = res_combine<false>(h[k], p[k], u0[k], u1[k], a.diag);
      dd += spinor_norm2(w[k]);
    }
    produce(T{}, E1, w, f2, f3);
    dd = warp_sum(dd);
    if ((tid & 31) == 0) red[0][tid >> 5] = dd;
    __syncthreads();
    gather(E1, f2, f3, h);
#pragma unroll
    for (int k = 0; k < SPT; ++k) w[k] = res_combine<true>(h[k], w[k], u0[k], u1[k], a.diag);
    double den = 0.0;
#pragma unroll
    for (int q = 0; q < NW; ++q) den += red[0][q];
    const double alpha = den > 0.0 ? rs / den : 0.0;
    const bool repl = (it % kResReplace) == 0;
    double rsn = 0.0;
#pragma unroll
    for (int k = 0; k < SPT; ++k) {
      x[k] = sp_fma(alpha, p[k], x[k]);
      if (!repl) {
        r[k] = sp_fma(-alpha, w[k], r[k]);
        rsn += spinor_norm2(r[k]);
      }
    }
    double rs_new = 0.0;
    bool check = true;
    if (!repl) {
      rs_new = block_sum<NT>(rsn, red[1]);
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
        w[k] = sp_sub(ldg_spinor(a.b, cb + s0 + k), w[k]);
        tn2 += spinor_norm2(w[k]);
      }
      tn2 = block_sum<NT>(tn2, red[2]);
      const double tn = sqrt(tn2);
      if (!repl || tn <= target) best = tn / normb;
      if (tn <= target) {
#pragma unroll
        for (int k = 0; k < SPT; ++k) st_spinor(a.x, cb + s0 + k, x[k]);
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
    const double beta = rs > 0.0 ? rs_new / rs : 0.0;
#pragma unroll
    for (int k = 0; k < SPT; ++k) p[k] = sp_fma(beta, p[k], r[k]);
    rs = rs_new;
  }
#pragma unroll
  for (int k = 0; k < SPT; ++k) st_spinor(a.x, cb + s0 + k, x[k]);
  if (tid == 0) {
    a.iters[c] = a.maxiter;
    a.relres[c] = fmin(best, sqrt(rs) / normb);
    a.status[c] = 1;
  }
}
