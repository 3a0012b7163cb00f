// Per-site arithmetic of the fermion force, the force-gradient pieces and
// the real-arithmetic link updates, shared by the batched kernels
// (wilson.cu, fields.cu) and the trajectory megakernel (mega.cu) so both
// evaluate identical expressions.  Field reads go through loader functors
// (the batched kernels use the read-only path; the megakernel reads fields it
// wrote itself, with coherent loads).
//
// Real-arithmetic updates (kicks, drift, gauge force, wrap) use explicit
// round-to-nearest intrinsics: no FMA contraction in any translation unit,
// NumPy's operation order (lattice.py, gauge.py, integrators.py).
#pragma once

#include "common.cuh"

// A(n) = conj(w-(a)(n)) U_mu(n) w-(b)(n+mu);  B(n) = conj(w+(a)(n+mu)) conj(U_mu(n)) w+(b)(n)
// (fermion.py:317-327), NumPy order: (conj(wa) * u) * wb.
struct Bil {
  double2 A, B;
};
template <int MU>
SCH_DEV Bil bilinear(const Spinor& a_n, const Spinor& a_f, const Spinor& b_n, const Spinor& b_f,
                     double2 u) {
  Bil r;
  if (MU == 0) {
    r.A = cmul(cmulc(wminus0(a_n), u), wminus0(b_f));
    r.B = cmul(cmulc(wplus0(a_f), cconj(u)), wplus0(b_n));
  } else {
    r.A = cmul(cmulc(wminus1(a_n), u), wminus1(b_f));
    r.B = cmul(cmulc(wplus1(a_f), cconj(u)), wplus1(b_n));
  }
  return r;
}

// Neighbour sites of s = x*T + t (periodic).
struct Nbr {
  int x, t, xp, xm, tp, tm;
};
SCH_DEV Nbr nbr(int s, int L, int T) {
  Nbr n;
  n.x = s / T;
  n.t = s - n.x * T;
  n.xp = n.x + 1 == L ? 0 : n.x + 1;
  n.xm = n.x == 0 ? L - 1 : n.x - 1;
  n.tp = n.t + 1 == T ? 0 : n.t + 1;
  n.tm = n.t == 0 ? T - 1 : n.t - 1;
  return n;
}

// Fermion force f(n, mu) = -Im(A - B) with a = chi, b = xi (fermion.py:330-336).
// chi(site), xi(site) -> Spinor; u(mu, site) -> double2.
template <class LC, class LX, class LU>
SCH_DEV void force_site(int s, int L, int T, LC chi, LX xi, LU u, double& f0, double& f1) {
  const Nbr n = nbr(s, L, T);
  const int sx = n.xp * T + n.t, st = n.x * T + n.tp;
  const Spinor cn = chi(s), xn = xi(s);
  const Spinor cx = chi(sx), xx = xi(sx);
  const Spinor ct = chi(st), xt = xi(st);
  const Bil b0 = bilinear<0>(cn, cx, xn, xx, u(0, s));
  const Bil b1 = bilinear<1>(cn, ct, xn, xt, u(1, s));
  f0 = -(b0.A.y - b0.B.y);
  f1 = -(b1.A.y - b1.B.y);
}

// Weighted w-sums at site s (fermion.py:362-383, gather form): b1 from chi,
// b2 from xi, weight w(mu, site) -> double.
template <class LC, class LX, class LU, class LW>
SCH_DEV void wsums_site(int s, int L, int T, LC chi, LX xi, LU u, LW w, Spinor& b1, Spinor& b2) {
  const Nbr n = nbr(s, L, T);
  double2 o10 = make_double2(0, 0), o11 = o10, o20 = o10, o21 = o10;
#pragma unroll
  for (int nu = 0; nu < 2; ++nu) {
    const int sf = nu == 0 ? n.xp * T + n.t : n.x * T + n.tp;   // n + nu
    const int sb = nu == 0 ? n.xm * T + n.t : n.x * T + n.tm;   // n - nu
    const Spinor cb_ = chi(sb), cf = chi(sf);
    const Spinor xb = xi(sb), xf = xi(sf);
    const double2 un = u(nu, s), ub = u(nu, sb);
    const double wn = w(nu, s), wb = w(nu, sb);
    const double2 wm_cb = nu == 0 ? wminus0(cb_) : wminus1(cb_);
    const double2 wp_cf = nu == 0 ? wplus0(cf) : wplus1(cf);
    const double2 wm_xf = nu == 0 ? wminus0(xf) : wminus1(xf);
    const double2 wp_xb = nu == 0 ? wplus0(xb) : wplus1(xb);
    // t1 = (0.5i * w*conj(U)*w-(chi))(n - nu)
    const double2 t1 = cscale(0.5, cmuli(cmul(cscale(wb, cconj(ub)), wm_cb)));
    // t2 = -0.5i * w(n) U(n) w+(chi)(n + nu)
    const double2 t2 = cscale(-0.5, cmuli(cmul(cscale(wn, un), wp_cf)));
    // t3 = -0.5i * w(n) U(n) w-(xi)(n + nu)
    const double2 t3 = cscale(-0.5, cmuli(cmul(cscale(wn, un), wm_xf)));
    // t4 = (0.5i * w*conj(U)*w+(xi))(n - nu)
    const double2 t4 = cscale(0.5, cmuli(cmul(cscale(wb, cconj(ub)), wp_xb)));
    o10 = cadd(o10, cadd(t1, t2));
    o20 = cadd(o20, cadd(t3, t4));
    if (nu == 0) {   // e- = -1, e+ = +1
      o11 = cadd(o11, csub(t2, t1));
      o21 = cadd(o21, csub(t4, t3));
    } else {         // e- = -i, e+ = +i
      o11 = cadd(o11, cmuli(csub(t2, t1)));
      o21 = cadd(o21, cmuli(csub(t4, t3)));
    }
  }
  b1.s0 = o10;
  b1.s1 = o11;
  b2.s0 = o20;
  b2.s1 = o21;
}

// C(n, mu) = 2Im(A[z1,xi]-B[z1,xi]) + 2Im(A[chi,z2]-B[chi,z2]) - 2Re(A[chi,xi]+B[chi,xi])*w
// (fermion.py:409-417)
template <int MU, class L1, class L2, class LC, class LX, class LU, class LW>
SCH_DEV double fg_combine_site(int s, int L, int T, L1 z1, L2 z2, LC chi, LX xi, LU u, LW w) {
  const Nbr n = nbr(s, L, T);
  const int sf = MU == 0 ? n.xp * T + n.t : n.x * T + n.tp;
  const Spinor z1n = z1(s), z1f = z1(sf);
  const Spinor z2n = z2(s), z2f = z2(sf);
  const Spinor cn = chi(s), cf = chi(sf);
  const Spinor xn = xi(s), xf = xi(sf);
  const double2 uu = u(MU, s);
  const Bil a1 = bilinear<MU>(z1n, z1f, xn, xf, uu);
  const Bil a2 = bilinear<MU>(cn, cf, z2n, z2f, uu);
  const Bil a3 = bilinear<MU>(cn, cf, xn, xf, uu);
  return 2.0 * (a1.A.y - a1.B.y) + 2.0 * (a2.A.y - a2.B.y) - 2.0 * (a3.A.x + a3.B.x) * w(MU, s);
}

// ------------------------------------------------------ real arithmetic
constexpr double kPi = 3.141592653589793;      // np.pi
constexpr double kTwoPi = 6.283185307179586;   // 2.0 * np.pi (lattice.py:21)

// fmod(a, 2pi) without the library's bit-serial loop: n = trunc(a / 2pi)
// from a rounded quotient, corrected by one if the rounding crossed an
// integer; then a - n*2pi in one FMA.  The remainder of a division of two
// doubles is exactly representable, so the single rounding of the FMA
// returns it exactly: the result equals fmod's bit for bit.
SCH_DEV double fmod_2pi(double a) {
  if (!(fabs(a) < 1e15)) return fmod(a, kTwoPi);   // inf / nan / huge: the library path
  double n = trunc(__dmul_rn(a, 1.0 / kTwoPi));
  double r = __fma_rn(-n, kTwoPi, a);
  if (r != 0.0 && (r < 0.0) != (a < 0.0)) {         // quotient rounded away from zero
    n -= a < 0.0 ? -1.0 : 1.0;
    r = __fma_rn(-n, kTwoPi, a);
  } else if (fabs(r) >= kTwoPi) {                   // rounded toward zero past an integer
    n += a < 0.0 ? -1.0 : 1.0;
    r = __fma_rn(-n, kTwoPi, a);
  }
  return r;
}

// NumPy's floored remainder (npy_divmod) followed by -pi: lattice.py:28-30
SCH_DEV double wrap_angle(double v) {
  const double a = __dadd_rn(v, kPi);
  double m = fmod_2pi(a);
  if (m != 0.0) {
    if (m < 0.0) m = __dadd_rn(m, kTwoPi);
  } else {
    m = 0.0;   // copysign(0, +2pi)
  }
  return __dsub_rn(m, kPi);
}

// drift: wrap(q + h p) (lattice.py:111-118)
SCH_DEV double rotate_elem(double q, double p, double h) { return wrap_angle(__dadd_rn(q, __dmul_rn(h, p))); }
// kick: p - a f  and  p - (a f + c g)  (integrators.py:161-246)
SCH_DEV double kick_elem(double p, double a, double f) { return __dsub_rn(p, __dmul_rn(a, f)); }
SCH_DEV double kick2_elem(double p, double a, double f, double c, double g) {
  return __dsub_rn(p, __dadd_rn(__dmul_rn(a, f), __dmul_rn(c, g)));
}
// gauge force at site s from the plaquette sines (gauge.py:43-59):
// g0 = beta (s - s(n - t)), g1 = beta (s(n - x) - s)
SCH_DEV void gauge_force_from_sines(double beta, double s0, double s_tm, double s_xm, double& f0,
                                    double& f1) {
  f0 = __dmul_rn(beta, __dsub_rn(s0, s_tm));
  f1 = __dmul_rn(beta, __dsub_rn(s_xm, s0));
}
