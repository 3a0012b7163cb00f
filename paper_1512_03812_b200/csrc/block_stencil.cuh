// Block-owned Wilson stencil pieces shared by the resident CG engines
// (resident_col.cuh: one CTA per chain; resident_cluster.cuh: one cluster
// per chain).
//
// A thread owns a BX x BT block of sites (BX rows in x, BT consecutive sites
// in t; site k = i*BT + j).  For one D (DAG=false) or D^dag (DAG=true)
// application every site exports four rank-1 projections (fermion.py:101-117,
// resident.cuh):
//   f0 = w_f0(v)               read by the site at x-1
//   b0 = conj(U0) w_b0(v)      read by the site at x+1
//   f1 = w_f1(v)               read by the site at t-1
//   b1 = conj(U1) w_b1(v)      read by the site at t+1
// Only the block's faces leave the thread: f0 of its first row, b0 of its
// last row, f1 of its first column, b1 of its last column.  The hops between
// its own sites are formed from the neighbour site's registers.  Each site's
// result is accumulated hop by hop (hop_acc, diag*v fused into the first):
// `interior` sums the register-only hops — it needs no exchange, so the
// kernels run it while the exchange barrier is pending — and `faces` adds
// the hops that arrived through shared memory.  Links are prescaled by -1/2.
#pragma once

#include <type_traits>

#include "resident.cuh"

template <bool DAG> SCH_DEV double2 export_f0(const Spinor& v) { return DAG ? wplus0(v) : wminus0(v); }
template <bool DAG> SCH_DEV double2 export_b0(const Spinor& v, double2 u0) {
  return cmulc(u0, DAG ? wminus0(v) : wplus0(v));
}
template <bool DAG> SCH_DEV double2 export_f1(const Spinor& v) { return DAG ? wplus1(v) : wminus1(v); }
template <bool DAG> SCH_DEV double2 export_b1(const Spinor& v, double2 u1) {
  return cmulc(u1, DAG ? wminus1(v) : wplus1(v));
}

template <int BX, int BT>
struct SiteBlock {
  static constexpr int SPT = BX * BT;
  static_assert(BX >= 2 && BT >= 2, "every site needs an internal hop in x and in t");

  // The block's face exports of v: put(plane, index, value) with plane 0/1
  // the first/last row (index j = t offset) and plane 2/3 the first/last
  // column (index i = x offset).
  template <bool DAG, class Put>
  static SCH_DEV void produce(const double2* u0, const double2* u1, const Spinor* v, Put&& put) {
#pragma unroll
    for (int k = 0; k < SPT; ++k) {
      const int i = k / BT, j = k % BT;
      if (i == 0) put(0, j, export_f0<DAG>(v[k]));
      if (i == BX - 1) put(1, j, export_b0<DAG>(v[k], u0[k]));
      if (j == 0) put(2, i, export_f1<DAG>(v[k]));
      if (j == BT - 1) put(3, i, export_b1<DAG>(v[k], u1[k]));
    }
  }

  // out = diag*v + the hops between the block's own sites
  template <bool DAG>
  static SCH_DEV void interior(const double2* u0, const double2* u1, const Spinor* v, Spinor* out,
                               double diag) {
#pragma unroll
    for (int k = 0; k < SPT; ++k) {
      const int i = k / BT, j = k % BT;
      bool first = true;
      if (i < BX - 1) {
        hop_acc<DAG, 0>(out[k], cmul(u0[k], export_f0<DAG>(v[k + BT])), first, v[k], diag);
        first = false;
      }
      if (i > 0) {
        hop_acc<DAG, 1>(out[k], export_b0<DAG>(v[k - BT], u0[k - BT]), first, v[k], diag);
        first = false;
      }
      if (j < BT - 1) {
        hop_acc<DAG, 2>(out[k], cmul(u1[k], export_f1<DAG>(v[k + 1])), first, v[k], diag);
        first = false;
      }
      if (j > 0) hop_acc<DAG, 3>(out[k], export_b1<DAG>(v[k - 1], u1[k - 1]), first, v[k], diag);
    }
  }

  // Add the face hops: fx[k] is the x-neighbour block's export for a site on
  // the first or last row, ft[k] the t-neighbour's for the first or last column.
  template <bool DAG>
  static SCH_DEV void faces(const double2* u0, const double2* u1, const double2* fx,
                            const double2* ft, Spinor* out) {
#pragma unroll
    for (int k = 0; k < SPT; ++k) {
      const int i = k / BT, j = k % BT;
      if (i == BX - 1) hop_acc<DAG, 0>(out[k], cmul(u0[k], fx[k]), false, out[k], 0.0);
      if (i == 0) hop_acc<DAG, 1>(out[k], fx[k], false, out[k], 0.0);
      if (j == BT - 1) hop_acc<DAG, 2>(out[k], cmul(u1[k], ft[k]), false, out[k], 0.0);
      if (j == 0) hop_acc<DAG, 3>(out[k], ft[k], false, out[k], 0.0);
    }
  }

  // The same face hops split by direction (the shuffle-exchange kernels add
  // the t-faces before the exchange barrier, the x-faces after it).
  template <bool DAG>
  static SCH_DEV void faces_t(const double2* u1, const double2* ft, Spinor* out) {
#pragma unroll
    for (int k = 0; k < SPT; ++k) {
      const int j = k % BT;
      if (j == BT - 1) hop_acc<DAG, 2>(out[k], cmul(u1[k], ft[k]), false, out[k], 0.0);
      if (j == 0) hop_acc<DAG, 3>(out[k], ft[k], false, out[k], 0.0);
    }
  }
  template <bool DAG>
  static SCH_DEV void faces_x(const double2* u0, const double2* fx, Spinor* out) {
#pragma unroll
    for (int k = 0; k < SPT; ++k) {
      const int i = k / BT;
      if (i == BX - 1) hop_acc<DAG, 0>(out[k], cmul(u0[k], fx[k]), false, out[k], 0.0);
      if (i == 0) hop_acc<DAG, 1>(out[k], fx[k], false, out[k], 0.0);
    }
  }
};

// The same operator in the sigma1-diagonal spin basis v' = T v, T = [[1,1],
// [1,-1]] (T^2 = 2, T/sqrt2 = H unitary, H s1 H = s3, H s2 H = -s2).  There
// the x projectors (1 -+ s1) become (1 -+ s3) = 2 diag(0,1) / 2 diag(1,0): an
// x hop reads one spin component of its neighbour and lands in one spin
// component of the result, so its projection and half of its accumulation
// disappear; the t projectors become (1 +- s2), i.e. D's t hops are the old
// D^dag's and vice versa.  D' = H D H has the same spectrum and CG on
// D'^dag D' with b' = T b takes the same steps as on D^dag D with b (x =
// T x' / 2), up to rounding.  FP64 work per site per D: 32 instead of 40.
// Links: u0 prescaled by -1 (the x projector's 2 times -1/2), u1 by -1/2.
//   D:     x fwd  o1 += u0 v1(n+x)        x bwd  o0 += conj(u0) v0(n-x)
//   D^dag: x fwd  o0 += u0 v0(n+x)        x bwd  o1 += conj(u0) v1(n-x)
template <bool DAG> SCH_DEV double2 rexport_f0(const Spinor& v) { return DAG ? v.s0 : v.s1; }
template <bool DAG> SCH_DEV double2 rexport_b0(const Spinor& v, double2 u0) {
  return cmulc(u0, DAG ? v.s1 : v.s0);
}

// x hop into one spin component (KIND 0 forward, 1 backward), diag*v fused
// into the first hop of the site
template <bool DAG, int KIND>
SCH_DEV void rhop_x(Spinor& o, double2 h, bool first, const Spinor& v, double diag) {
  constexpr bool to1 = (KIND == 0) != DAG;
  if (first) {
    if (to1) {
      o.s0 = make_double2(diag * v.s0.x, diag * v.s0.y);
      o.s1 = make_double2(__fma_rn(diag, v.s1.x, h.x), __fma_rn(diag, v.s1.y, h.y));
    } else {
      o.s0 = make_double2(__fma_rn(diag, v.s0.x, h.x), __fma_rn(diag, v.s0.y, h.y));
      o.s1 = make_double2(diag * v.s1.x, diag * v.s1.y);
    }
  } else if (to1) {
    o.s1 = cadd(o.s1, h);
  } else {
    o.s0 = cadd(o.s0, h);
  }
}

// o + u*f and o + conj(u)*f as four FMAs each
SCH_DEV double2 cmul_acc(double2 o, double2 u, double2 f) {
  o.x = __fma_rn(u.x, f.x, o.x);
  o.x = __fma_rn(-u.y, f.y, o.x);
  o.y = __fma_rn(u.x, f.y, o.y);
  o.y = __fma_rn(u.y, f.x, o.y);
  return o;
}
SCH_DEV double2 cmulc_acc(double2 o, double2 u, double2 f) {
  o.x = __fma_rn(u.x, f.x, o.x);
  o.x = __fma_rn(u.y, f.y, o.x);
  o.y = __fma_rn(u.x, f.y, o.y);
  o.y = __fma_rn(-u.y, f.x, o.y);
  return o;
}

template <int BX, int BT>
struct SiteBlockRot {
  static constexpr int SPT = BX * BT;
  static_assert(BX >= 2 && BT >= 2, "every site needs an internal hop in x and in t");

  template <bool DAG, class Put>
  static SCH_DEV void produce(const double2* u0, const double2* u1, const Spinor* v, Put&& put) {
#pragma unroll
    for (int k = 0; k < SPT; ++k) {
      const int i = k / BT, j = k % BT;
      if (i == 0) put(0, j, rexport_f0<DAG>(v[k]));
      if (i == BX - 1) put(1, j, rexport_b0<DAG>(v[k], u0[k]));
      if (j == 0) put(2, i, export_f1<!DAG>(v[k]));
      if (j == BT - 1) put(3, i, export_b1<!DAG>(v[k], u1[k]));
    }
  }

  // diag*v is fused per spin component into the first hop that reaches it:
  // the internal t hop (BT >= 2), which reaches both
  template <bool DAG>
  static SCH_DEV void interior(const double2* u0, const double2* u1, const Spinor* v, Spinor* out,
                               double diag) {
#pragma unroll
    for (int k = 0; k < SPT; ++k) {
      const int i = k / BT, j = k % BT;
      bool f0 = true, f1 = true;
      auto acc = [&](double2& o, double2 val, double2 vc, bool& first) {
        if (first) o = make_double2(__fma_rn(diag, vc.x, val.x), __fma_rn(diag, vc.y, val.y));
        else o = cadd(o, val);
        first = false;
      };
      auto thop = [&](auto kind, double2 h) {   // hop_acc<!DAG, kind> with per-component fusion
        constexpr int KIND = decltype(kind)::value;
        constexpr bool neg = (KIND == 2) != !DAG;
        double2 g = cmuli(h);
        if (neg) g = make_double2(-g.x, -g.y);
        acc(out[k].s0, h, v[k].s0, f0);
        acc(out[k].s1, g, v[k].s1, f1);
      };
      using K2 = std::integral_constant<int, 2>;
      using K3 = std::integral_constant<int, 3>;
      // t hops first (they reach both components, so diag*v fuses into them);
      // the x hops then land on one component each as a fused complex
      // multiply-accumulate (4 DFMA instead of 2 DMUL + 2 DFMA + 2 DADD)
      if (j < BT - 1) thop(K2{}, cmul(u1[k], export_f1<!DAG>(v[k + 1])));
      if (j > 0) thop(K3{}, export_b1<!DAG>(v[k - 1], u1[k - 1]));
      constexpr bool fwd_to1 = !DAG, bwd_to1 = DAG;
      if (i < BX - 1) {
        double2& o = fwd_to1 ? out[k].s1 : out[k].s0;
        o = cmul_acc(o, u0[k], rexport_f0<DAG>(v[k + BT]));
      }
      if (i > 0) {
        double2& o = bwd_to1 ? out[k].s1 : out[k].s0;
        o = cmulc_acc(o, u0[k - BT], DAG ? v[k - BT].s1 : v[k - BT].s0);
      }
    }
  }

  template <bool DAG>
  static SCH_DEV void faces(const double2* u0, const double2* u1, const double2* fx,
                            const double2* ft, Spinor* out) {
    faces_x<DAG>(u0, fx, out);
    faces_t<DAG>(u1, ft, out);
  }
  template <bool DAG>
  static SCH_DEV void faces_t(const double2* u1, const double2* ft, Spinor* out) {
#pragma unroll
    for (int k = 0; k < SPT; ++k) {
      const int j = k % BT;
      if (j == BT - 1) hop_acc<!DAG, 2>(out[k], cmul(u1[k], ft[k]), false, out[k], 0.0);
      if (j == 0) hop_acc<!DAG, 3>(out[k], ft[k], false, out[k], 0.0);
    }
  }
  template <bool DAG>
  static SCH_DEV void faces_x(const double2* u0, const double2* fx, Spinor* out) {
#pragma unroll
    for (int k = 0; k < SPT; ++k) {
      const int i = k / BT;
      if (i == BX - 1) {
        double2& o = DAG ? out[k].s0 : out[k].s1;
        o = cmul_acc(o, u0[k], fx[k]);
      }
      if (i == 0) rhop_x<DAG, 1>(out[k], fx[k], false, out[k], 0.0);
    }
  }
};

// v' = T v and its inverse x = T x' / 2 (the /2 is exact)
SCH_DEV Spinor spin_rot(const Spinor& v) {
  Spinor r;
  r.s0 = cadd(v.s0, v.s1);
  r.s1 = csub(v.s0, v.s1);
  return r;
}
SCH_DEV Spinor spin_unrot(const Spinor& v) {
  Spinor r;
  r.s0 = cscale(0.5, cadd(v.s0, v.s1));
  r.s1 = cscale(0.5, csub(v.s0, v.s1));
  return r;
}

template <bool ROT> SCH_DEV Spinor rot_in(const Spinor& v) { return ROT ? spin_rot(v) : v; }
template <bool ROT> SCH_DEV Spinor rot_out(const Spinor& v) { return ROT ? spin_unrot(v) : v; }

SCH_DEV double2 shfl_d2(double2 v, int src) {
  return make_double2(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}
