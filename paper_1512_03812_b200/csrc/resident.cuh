// Resident per-chain CG (one CTA owns one chain for the whole solve).
//
// Data placement (B200 SM: 64K regs, 228 KB SMEM, 128 B/clk SMEM port):
//   registers : the thread's own sites' U_0, U_1, x, r, p (and t = D p)
//   SMEM      : only the rank-1 projections each site exports to its four
//               neighbours ("half-spinor exchange"), double-buffered
//   global    : b (read at start and on the rare true-residual path), x out
//
// For D the four hops of site n are (fermion.py:101-117, Appendix A2)
//   hf0 = U0(n)             w-0(v(n+x))     hb0 = [conj(U0) w+0(v)](n-x)
//   hf1 = U1(n)             w-1(v(n+t))     hb1 = [conj(U1) w+1(v)](n-t)
// and D^dag swaps w-/w+.  Each site m therefore PRODUCES
//   plane 0: w_f0(v(m))            (read by m-x)
//   plane 1: conj(U0(m)) w_b0(v(m)) (read by m+x)
//   plane 2: w_f1(v(m))            (read by m-t)
//   plane 3: conj(U1(m)) w_b1(v(m)) (read by m+t)
// so every link is read only by its owner (from registers) and the SMEM
// traffic per site per D application is 64 B stored + 64 B loaded, against
// 224 B of full-spinor neighbour loads in a direct stencil.
#pragma once

#include "common.cuh"

struct ResArgs {
  const double2* __restrict__ U;   // [B][2][V]
  const double2* __restrict__ b;   // [B][V][2]
  const double2* __restrict__ x0;  // may be null
  double2* __restrict__ x;         // out
  int* __restrict__ iters;
  double* __restrict__ relres;
  int* __restrict__ status;
  int L, T;
  double diag, tol;
  int maxiter;
};

constexpr int kResReplace = 50;   // residual replacement period (fermion.py:199)

// producer: the four exported projections of v at one site
template <bool DAG>
SCH_DEV void res_produce(double2* __restrict__ E, int V, int s, const Spinor& v, double2 u0,
                         double2 u1) {
  if (!DAG) {
    E[s] = wminus0(v);
    E[V + s] = cmulc(u0, wplus0(v));
    E[2 * V + s] = wminus1(v);
    E[3 * V + s] = cmulc(u1, wplus1(v));
  } else {
    E[s] = wplus0(v);
    E[V + s] = cmulc(u0, wminus0(v));
    E[2 * V + s] = wplus1(v);
    E[3 * V + s] = cmulc(u1, wminus1(v));
  }
}

// consumer: (D v)(n) or (D^dag v)(n) from the neighbours' exports.
// PRESCALED: the links were multiplied by -1/2 once (exact in binary), so the
// four hops arrive already scaled and the site term is one FMA per component.
template <bool DAG, bool PRESCALED = false>
SCH_DEV Spinor res_consume(const double2* __restrict__ E, int V, const Spinor& v, double2 u0,
                           double2 u1, int nxp, int nxm, int ntp, int ntm, double diag) {
  const double2 hf0 = cmul(u0, E[nxp]);
  const double2 hb0 = E[V + nxm];
  const double2 hf1 = cmul(u1, E[2 * V + ntp]);
  const double2 hb1 = E[3 * V + ntm];
  double2 o0 = cadd(cadd(cadd(hf0, hb0), hf1), hb1);
  double2 o1 = DAG ? cadd(csub(hf0, hb0), cmuli(csub(hf1, hb1)))
                   : cadd(csub(hb0, hf0), cmuli(csub(hb1, hf1)));
  Spinor r;
  if (PRESCALED) {
    r.s0 = make_double2(__fma_rn(diag, v.s0.x, o0.x), __fma_rn(diag, v.s0.y, o0.y));
    r.s1 = make_double2(__fma_rn(diag, v.s1.x, o1.x), __fma_rn(diag, v.s1.y, o1.y));
  } else {
    r.s0 = make_double2(diag * v.s0.x - 0.5 * o0.x, diag * v.s0.y - 0.5 * o0.y);
    r.s1 = make_double2(diag * v.s1.x - 0.5 * o1.x, diag * v.s1.y - 0.5 * o1.y);
  }
  return r;
}

// res_consume with the t-direction exports passed in (warp shuffles) instead
// of read from the E planes 2/3; same arithmetic, same order.
template <bool DAG>
SCH_DEV Spinor res_consume_tsh(const double2* __restrict__ E, int V, const Spinor& v, double2 u0,
                               double2 u1, int nxp, int nxm, double2 f1n, double2 b1n,
                               double diag) {
  const double2 hf0 = cmul(u0, E[nxp]);
  const double2 hb0 = E[V + nxm];
  const double2 hf1 = cmul(u1, f1n);
  const double2 hb1 = b1n;
  double2 o0 = cadd(cadd(cadd(hf0, hb0), hf1), hb1);
  double2 o1 = DAG ? cadd(csub(hf0, hb0), cmuli(csub(hf1, hb1)))
                   : cadd(csub(hb0, hf0), cmuli(csub(hb1, hf1)));
  Spinor r;
  r.s0 = make_double2(diag * v.s0.x - 0.5 * o0.x, diag * v.s0.y - 0.5 * o0.y);
  r.s1 = make_double2(diag * v.s1.x - 0.5 * o1.x, diag * v.s1.y - 0.5 * o1.y);
  return r;
}

// x-direction exports to E (planes 0/1); the t-direction ones returned
template <bool DAG>
SCH_DEV void res_produce_x(double2* __restrict__ E, int V, int s, const Spinor& v, double2 u0,
                           double2 u1, double2& f1, double2& b1) {
  if (!DAG) {
    E[s] = wminus0(v);
    E[V + s] = cmulc(u0, wplus0(v));
    f1 = wminus1(v);
    b1 = cmulc(u1, wplus1(v));
  } else {
    E[s] = wplus0(v);
    E[V + s] = cmulc(u0, wminus0(v));
    f1 = wplus1(v);
    b1 = cmulc(u1, wminus1(v));
  }
}

SCH_DEV double2 tile_shfl_d2(double2 v, int src) {
  return make_double2(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}

// consumer split in two: gather the four neighbour exports (issue all
// shared-memory loads first), then combine
struct Hops {
  double2 f0, b0, f1, b1;
};
SCH_DEV Hops res_gather(const double2* __restrict__ E, int V, int nxp, int nxm, int ntp, int ntm) {
  Hops h;
  h.f0 = E[nxp];
  h.b0 = E[V + nxm];
  h.f1 = E[2 * V + ntp];
  h.b1 = E[3 * V + ntm];
  return h;
}
template <bool DAG>
SCH_DEV Spinor res_combine(const Hops& h, const Spinor& v, double2 u0, double2 u1, double diag) {
  const double2 hf0 = cmul(u0, h.f0);
  const double2 hf1 = cmul(u1, h.f1);
  double2 o0 = cadd(cadd(cadd(hf0, h.b0), hf1), h.b1);
  double2 o1 = DAG ? cadd(csub(hf0, h.b0), cmuli(csub(hf1, h.b1)))
                   : cadd(csub(h.b0, hf0), cmuli(csub(h.b1, hf1)));
  Spinor r;   // links pre-scaled by -1/2
  r.s0 = make_double2(__fma_rn(diag, v.s0.x, o0.x), __fma_rn(diag, v.s0.y, o0.y));
  r.s1 = make_double2(__fma_rn(diag, v.s1.x, o1.x), __fma_rn(diag, v.s1.y, o1.y));
  return r;
}

// Incremental form of res_combine: o accumulates one site's hops one at a
// time, diag*v fused into the first, so the hops a thread already holds (its
// internal ones) can be summed while an exchange barrier is pending.
// KIND 0: forward x (h = U0(n) * export), 1: backward x, 2: forward t,
// 3: backward t.  Spin-1 coefficients: D f0 -1, b0 +1, f1 -i, b1 +i; D^dag
// the negatives (fermion.py:101-117).
template <bool DAG, int KIND>
SCH_DEV void hop_acc(Spinor& o, double2 h, bool first, const Spinor& v, double diag) {
  constexpr bool neg = (KIND == 0 || KIND == 2) != DAG;
  double2 g = KIND >= 2 ? cmuli(h) : h;
  if (neg) g = make_double2(-g.x, -g.y);
  if (first) {
    o.s0 = make_double2(__fma_rn(diag, v.s0.x, h.x), __fma_rn(diag, v.s0.y, h.y));
    o.s1 = make_double2(__fma_rn(diag, v.s1.x, g.x), __fma_rn(diag, v.s1.y, g.y));
  } else {
    o.s0 = cadd(o.s0, h);
    o.s1 = cadd(o.s1, g);
  }
}

SCH_DEV Spinor sp_fma(double a, const Spinor& p, const Spinor& x) {   // a*p + x
  Spinor r;
  r.s0 = make_double2(__fma_rn(a, p.s0.x, x.s0.x), __fma_rn(a, p.s0.y, x.s0.y));
  r.s1 = make_double2(__fma_rn(a, p.s1.x, x.s1.x), __fma_rn(a, p.s1.y, x.s1.y));
  return r;
}

SCH_DEV Spinor sp_sub(const Spinor& a, const Spinor& b) {
  Spinor r;
  r.s0 = csub(a.s0, b.s0);
  r.s1 = csub(a.s1, b.s1);
  return r;
}

template <int NT, int SPT, int MINB, int LC = 0, int TC = 0>
__global__ void __launch_bounds__(NT, MINB) k_cg_resident(ResArgs a) {
  extern __shared__ double2 sm[];
  __shared__ double red[3][NT / 32];
  // LC/TC > 0: compile-time lattice (the hot 16^2 / 32^2 shapes): no guards,
  // neighbour indices computed with shifts instead of held in registers
  const int L = LC > 0 ? LC : a.L, T = TC > 0 ? TC : a.T, V = L * T;
  static_assert(LC == 0 || LC * TC == NT * SPT, "specialised shape must fill the CTA");
  double2* E0 = sm;            // D-stage exports   [4][V]
  double2* E1 = sm + 4 * V;    // Ddag-stage exports [4][V]
  const int c = blockIdx.x;
  const long long cb = (long long)c * V;
  const int tid = threadIdx.x;

  int site[SPT], nxp_[SPT], nxm_[SPT], ntp_[SPT], ntm_[SPT];
  auto nbr = [&](int k, int which) -> int {
    if constexpr (LC > 0) {
      const int s = tid + k * NT;
      const int xx = s / TC, tt = s % TC;
      switch (which) {
        case 0: return ((xx + 1) % LC) * TC + tt;
        case 1: return ((xx + LC - 1) % LC) * TC + tt;
        case 2: return xx * TC + (tt + 1) % TC;
        default: return xx * TC + (tt + TC - 1) % TC;
      }
    } else {
      return which == 0 ? nxp_[k] : which == 1 ? nxm_[k] : which == 2 ? ntp_[k] : ntm_[k];
    }
  };
  auto valid = [&](int k) -> bool {
    if constexpr (LC > 0) return true;
    else return site[k] >= 0;
  };
  double2 u0[SPT], u1[SPT];
  Spinor x[SPT], r[SPT], p[SPT];
  double bb = 0.0;
#pragma unroll
  for (int k = 0; k < SPT; ++k) {
    const int s = tid + k * NT;
    site[k] = s < V ? s : -1;
    x[k].s0 = x[k].s1 = make_double2(0, 0);
    if (LC > 0 || s < V) {
      if constexpr (LC == 0) {
        const int xx = s / T, tt = s - xx * T;
        nxp_[k] = (xx + 1 == L ? 0 : xx + 1) * T + tt;
        nxm_[k] = (xx == 0 ? L - 1 : xx - 1) * T + tt;
        ntp_[k] = xx * T + (tt + 1 == T ? 0 : tt + 1);
        ntm_[k] = xx * T + (tt == 0 ? T - 1 : tt - 1);
      }
      u0[k] = cscale(-0.5, __ldg(a.U + 2 * cb + s));        // exact: power-of-two scale
      u1[k] = cscale(-0.5, __ldg(a.U + 2 * cb + V + s));
      r[k] = ldg_spinor(a.b, cb + s);
      bb += spinor_norm2(r[k]);
    } else {
      nxp_[k] = nxm_[k] = ntp_[k] = ntm_[k] = 0;
      u0[k] = u1[k] = make_double2(0, 0);
      r[k].s0 = r[k].s1 = make_double2(0, 0);
    }
  }
  const double normb2 = block_sum<NT>(bb, red[0]);
  const double normb = sqrt(normb2);
  const double target = a.tol * normb;
  if (normb == 0.0) {   // fermion.py:181-182, per chain
#pragma unroll
    for (int k = 0; k < SPT; ++k)
      if (valid(k)) st_spinor(a.x, cb + site[k], x[k]);
    if (tid == 0) {
      a.iters[c] = 0;
      a.relres[c] = 0.0;
      a.status[c] = 0;
    }
    return;
  }

  // out[k] = D^dag D v[k] for the thread's sites; two exchange rounds.
  // Precondition: every thread has finished reading E0 and E1 from any
  // previous application (guaranteed by the block_sum barriers in between).
  auto normal_op = [&](const Spinor* v, Spinor* out) {
#pragma unroll
    for (int k = 0; k < SPT; ++k)
      if (valid(k)) res_produce<false>(E0, V, site[k], v[k], u0[k], u1[k]);
    __syncthreads();
#pragma unroll
    for (int k = 0; k < SPT; ++k)
      if (valid(k)) {
        Spinor t = res_consume<false, true>(E0, V, v[k], u0[k], u1[k], nbr(k, 0), nbr(k, 1),
                                            nbr(k, 2), nbr(k, 3), a.diag);
        out[k] = t;
        res_produce<true>(E1, V, site[k], t, u0[k], u1[k]);
      }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < SPT; ++k)
      if (valid(k))
        out[k] = res_consume<true, true>(E1, V, out[k], u0[k], u1[k], nbr(k, 0), nbr(k, 1),
                                         nbr(k, 2), nbr(k, 3), a.diag);
  };

  Spinor w[SPT];   // A applied to something
  double rs = normb2;   // r = b exactly: the same sum as ||b||^2 (fermion.py:186,191)
  if (a.x0) {
#pragma unroll
    for (int k = 0; k < SPT; ++k)
      if (valid(k)) x[k] = ldg_spinor(a.x0, cb + site[k]);
    normal_op(x, w);
    double rr = 0.0;
#pragma unroll
    for (int k = 0; k < SPT; ++k)
      if (valid(k)) {
        r[k] = sp_sub(r[k], w[k]);
        rr += spinor_norm2(r[k]);
      }
    rs = block_sum<NT>(rr, red[1]);
  }
#pragma unroll
  for (int k = 0; k < SPT; ++k) p[k] = r[k];

  double best = INFINITY;
  constexpr int NW = NT / 32;
  for (int it = 1; it <= a.maxiter; ++it) {
    // w = D^dag D p with <p, D^dag D p> formed as ||D p||^2 during the D stage:
    // its warp partials are published by the barrier that already separates
    // the D and D^dag stages, so the reduction costs no extra barrier and
    // overlaps the D^dag stage.
#pragma unroll
    for (int k = 0; k < SPT; ++k)
      if (valid(k)) res_produce<false>(E0, V, site[k], p[k], u0[k], u1[k]);
    __syncthreads();
    double dd = 0.0;
    Hops hp[SPT];
#pragma unroll
    for (int k = 0; k < SPT; ++k)   // all neighbour loads in flight before any math
      if (valid(k)) hp[k] = res_gather(E0, V, nbr(k, 0), nbr(k, 1), nbr(k, 2), nbr(k, 3));
#pragma unroll
    for (int k = 0; k < SPT; ++k)
      if (valid(k)) {
        Spinor t = res_combine<false>(hp[k], p[k], u0[k], u1[k], a.diag);
        dd += spinor_norm2(t);
        w[k] = t;
        res_produce<true>(E1, V, site[k], t, u0[k], u1[k]);
      }
    dd = warp_sum(dd);
    if ((tid & 31) == 0) red[0][tid >> 5] = dd;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < SPT; ++k)
      if (valid(k)) hp[k] = res_gather(E1, V, nbr(k, 0), nbr(k, 1), nbr(k, 2), nbr(k, 3));
#pragma unroll
    for (int k = 0; k < SPT; ++k)
      if (valid(k)) w[k] = res_combine<true>(hp[k], w[k], u0[k], u1[k], a.diag);
    double den = 0.0;
#pragma unroll
    for (int q = 0; q < NW; ++q) den += red[0][q];
    const double alpha = den > 0.0 ? rs / den : 0.0;
    const bool repl = (it % kResReplace) == 0;
    double rsn = 0.0;
#pragma unroll
    for (int k = 0; k < SPT; ++k) {
      if (!valid(k)) continue;
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
      check = sqrt(rs_new) <= target;
    }
    if (check) {   // true residual b - A x (shared with the residual replacement)
      normal_op(x, w);
      double tn2 = 0.0;
#pragma unroll
      for (int k = 0; k < SPT; ++k)
        if (valid(k)) {
          w[k] = sp_sub(ldg_spinor(a.b, cb + site[k]), w[k]);
          tn2 += spinor_norm2(w[k]);
        }
      tn2 = block_sum<NT>(tn2, red[2]);
      const double tn = sqrt(tn2);
      if (!repl || tn <= target) best = tn / normb;
      if (tn <= target) {
#pragma unroll
        for (int k = 0; k < SPT; ++k)
          if (valid(k)) st_spinor(a.x, cb + site[k], x[k]);
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
  for (int k = 0; k < SPT; ++k)
    if (valid(k)) st_spinor(a.x, cb + site[k], x[k]);
  if (tid == 0) {
    a.iters[c] = a.maxiter;
    a.relres[c] = fmin(best, sqrt(rs) / normb);
    a.status[c] = 1;
  }
}
