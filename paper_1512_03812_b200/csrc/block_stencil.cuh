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

SCH_DEV double2 shfl_d2(double2 v, int src) {
  return make_double2(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}
