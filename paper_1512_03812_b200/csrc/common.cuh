// Shared device helpers for the sm_100a Schwinger-model HMC kernels.
//
// Layouts are the reference's (lattice.py:3-12), so no conversion pass is
// needed at the C-ABI boundary:
//   link fields  double  [chain][mu][x][t]          (mu=0: x, mu=1: t)
//   link cache U double2 [chain][mu][x][t]          U = exp(i q) (fermion.py:94)
//   spinors      double2 [chain][x][t][spin]        complex128 (..., L, T, 2)
// Site index s = x*T + t (t fastest).  All arithmetic is FP64; tensor cores
// are not used (sparse stencil, ~1.2 flop/B).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#define SCH_DEV __device__ __forceinline__

// ---------------------------------------------------------------- complex
SCH_DEV double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
SCH_DEV double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
SCH_DEV double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// conj(a) * b
SCH_DEV double2 cmulc(double2 a, double2 b) {
  return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
// i * a
SCH_DEV double2 cmuli(double2 a) { return make_double2(-a.y, a.x); }
SCH_DEV double2 cscale(double s, double2 a) { return make_double2(s * a.x, s * a.y); }
SCH_DEV double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
// Re(conj(a) b)
SCH_DEV double redot(double2 a, double2 b) { return a.x * b.x + a.y * b.y; }

struct Spinor {
  double2 s0, s1;
};

// ------------------------------------------------------- rank-1 projectors
// (1 -/+ sigma_mu) v = (w, e*w)   (fermion.py:36-51)
//   w-(v,0) = v0 - v1   e- = -1      w+(v,0) = v0 + v1   e+ = +1
//   w-(v,1) = v0 + i v1 e- = -i      w+(v,1) = v0 - i v1 e+ = +i
SCH_DEV double2 wminus0(const Spinor& v) { return csub(v.s0, v.s1); }
SCH_DEV double2 wplus0(const Spinor& v) { return cadd(v.s0, v.s1); }
SCH_DEV double2 wminus1(const Spinor& v) { return cadd(v.s0, cmuli(v.s1)); }
SCH_DEV double2 wplus1(const Spinor& v) { return csub(v.s0, cmuli(v.s1)); }

// Wilson-Dirac site kernel (fermion.py:101-127, Appendix A2).
//   c      psi(n)
//   xp/xm  psi(n +- x)      tp/tm  psi(n +- t)
//   u0     U_0(n)  u0m U_0(n-x)  u1 U_1(n)  u1m U_1(n-t)
// Accumulation order follows the reference: mu=0 then mu=1, forward then
// backward, so the result differs from NumPy only by FMA contraction.
template <bool DAG>
SCH_DEV Spinor wilson_site(const Spinor& c, const Spinor& xp, const Spinor& xm,
                           const Spinor& tp, const Spinor& tm, double2 u0, double2 u0m,
                           double2 u1, double2 u1m, double diag) {
  double2 o0, o1;
  if (!DAG) {
    double2 hf = cmul(u0, wminus0(xp));
    double2 hb = cmulc(u0m, wplus0(xm));
    o0 = cadd(hf, hb);
    o1 = csub(hb, hf);                       // (-1) hf + (+1) hb
    hf = cmul(u1, wminus1(tp));
    hb = cmulc(u1m, wplus1(tm));
    o0 = cadd(cadd(o0, hf), hb);
    o1 = cadd(o1, cmuli(csub(hb, hf)));      // (-i) hf + (+i) hb
  } else {
    double2 hf = cmul(u0, wplus0(xp));
    double2 hb = cmulc(u0m, wminus0(xm));
    o0 = cadd(hf, hb);
    o1 = csub(hf, hb);                       // (+1) hf + (-1) hb
    hf = cmul(u1, wplus1(tp));
    hb = cmulc(u1m, wminus1(tm));
    o0 = cadd(cadd(o0, hf), hb);
    o1 = cadd(o1, cmuli(csub(hf, hb)));      // (+i) hf + (-i) hb
  }
  Spinor r;
  r.s0 = make_double2(diag * c.s0.x - 0.5 * o0.x, diag * c.s0.y - 0.5 * o0.y);
  r.s1 = make_double2(diag * c.s1.x - 0.5 * o1.x, diag * c.s1.y - 0.5 * o1.y);
  return r;
}

SCH_DEV Spinor ld_spinor(const double2* __restrict__ p, long site) {
  Spinor v;
  v.s0 = p[2 * site];
  v.s1 = p[2 * site + 1];
  return v;
}
SCH_DEV Spinor ldg_spinor(const double2* __restrict__ p, long site) {
  Spinor v;
  v.s0 = __ldg(p + 2 * site);
  v.s1 = __ldg(p + 2 * site + 1);
  return v;
}
SCH_DEV void st_spinor(double2* __restrict__ p, long site, const Spinor& v) {
  p[2 * site] = v.s0;
  p[2 * site + 1] = v.s1;
}
// One 256-bit access per site (sm_100a LDG/STG.E.ENL2.256): a warp moves
// 1 KiB of spinors per instruction, fully coalesced, no half-used sectors.
// `p` must be 32-B aligned at the site (true for every [..][V][2] c128 field).
SCH_DEV Spinor ld256_spinor_nc(const double2* __restrict__ p, long long site) {
  Spinor v;
  asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(v.s0.x), "=d"(v.s0.y), "=d"(v.s1.x), "=d"(v.s1.y)
               : "l"(p + 2 * site));
  return v;
}
SCH_DEV Spinor ld256_spinor(const double2* p, long long site) {
  Spinor v;
  asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(v.s0.x), "=d"(v.s0.y), "=d"(v.s1.x), "=d"(v.s1.y)
               : "l"(p + 2 * site));
  return v;
}
SCH_DEV void st256_spinor(double2* p, long long site, const Spinor& v) {
  asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p + 2 * site), "d"(v.s0.x),
               "d"(v.s0.y), "d"(v.s1.x), "d"(v.s1.y)
               : "memory");
}

SCH_DEV double spinor_norm2(const Spinor& v) {
  return v.s0.x * v.s0.x + v.s0.y * v.s0.y + v.s1.x * v.s1.x + v.s1.y * v.s1.y;
}
SCH_DEV double spinor_redot(const Spinor& a, const Spinor& b) {
  return a.s0.x * b.s0.x + a.s0.y * b.s0.y + a.s1.x * b.s1.x + a.s1.y * b.s1.y;
}

// -------------------------------------------------------------- reductions
// Deterministic block sum: xor-butterfly inside a warp (IEEE addition is
// commutative, so every lane holds the identical value), then a fixed-order
// sum over the per-warp slots.  `slot` must hold blockDim.x/32 doubles and
// must not be reused until after the next __syncthreads().
SCH_DEV double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Canonical tree sum over the 32 lanes (lane l holds value l): a balanced
// binary tree in index order, adjacent pairs first (xor 1, 2, ..., 16);
// every lane ends with the same value.  Zero padding a shorter sequence to
// 32 lanes leaves this tree's value unchanged.
SCH_DEV double warp_tree_sum(double v) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int NT>
SCH_DEV double block_sum(double v, double* slot) {
  constexpr int NW = NT / 32;
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) slot[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = slot[0];
#pragma unroll
  for (int w = 1; w < NW; ++w) s += slot[w];
  return s;
}

// Runtime-width variant for generic kernels (blockDim.x multiple of 32, <= 1024).
SCH_DEV double block_sum_rt(double v, double* slot) {
  const int nw = blockDim.x >> 5;
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) slot[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < nw; ++w) s += slot[w];
  return s;
}

SCH_DEV int wrapi(int i, int n) { return i < 0 ? i + n : (i >= n ? i - n : i); }

// Programmatic dependent launch (sm_90+).  A kernel launched with the
// programmatic-stream-serialization attribute may be scheduled while its
// predecessor drains: kernels that take part call pdl_enter() first — it
// lets their own successor launch early and then waits until the
// predecessor has completed and its writes are visible.  Under a normal
// launch both instructions are no-ops.
SCH_DEV void pdl_enter() {
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

// theta(n) = q0(n) + q1(n+x) - q0(n+t) - q1(n)   (gauge.py:21-24), NumPy order.
// qc points at one chain's [2][L][T] angles.
SCH_DEV double plaq(const double* __restrict__ qc, int L, int T, int x, int t) {
  const long long V = (long long)L * T;
  int xp = x + 1 == L ? 0 : x + 1;
  int tp = t + 1 == T ? 0 : t + 1;
  double q0 = qc[x * T + t];
  double q1 = qc[V + x * T + t];
  double q1x = qc[V + xp * T + t];
  double q0t = qc[x * T + tp];
  return __dsub_rn(__dsub_rn(__dadd_rn(q0, q1x), q0t), q1);
}
