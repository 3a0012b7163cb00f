// Wilson-fermion kernels: link cache, D / D^dag, fused D^dag D, spinor dots,
// fermion force (+ fused kicks), weighted w-sums and the fermion
// force-gradient contraction.  Reference: fermion.py.
#include "common.cuh"
#include "site_ops.cuh"
#include "runtime.hpp"
#include "tile.cuh"
#include "tma_tile.cuh"
#include "../../include/schwinger_sm100.h"

namespace {

struct Geo {
  int B, L, T;
  long long V;
};

unsigned grid_for(long long n, int nt = 256) {
  long long b = (n + nt - 1) / nt;
  if (b > 148LL * 64) b = 148LL * 64;
  if (b < 1) b = 1;
  return (unsigned)b;
}

// U = exp(i q) = (cos q, sin q)  (fermion.py:94).  bc = 1 flips U_t on the
// last time slice (fermions antiperiodic in time, BASELINE configs).
__global__ void k_links_to_u(const double* __restrict__ q, double2* __restrict__ U, Geo g, int bc) {
  long long n = (long long)g.B * 2 * g.V;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    double s, c;
    sincos(q[i], &s, &c);
    if (bc) {
      long long r = i % (2 * g.V);
      if (r >= g.V && (r - g.V) % g.T == g.T - 1) {
        s = -s;
        c = -c;
      }
    }
    U[i] = make_double2(c, s);
  }
}

// One thread per site; neighbours through L1.  Used for the single-D
// applications (chi = D xi, eta = D^dag phi, D^dag b for solve_dirac).
template <bool DAG>
__global__ void k_dslash(const double2* __restrict__ U, long long ustride,
                         const double2* __restrict__ psi, double2* __restrict__ out, Geo g,
                         double diag) {
  long long n = (long long)g.B * g.V;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    long long b = i / g.V;
    int s = (int)(i - b * g.V);
    int x = s / g.T, t = s - x * g.T;
    int xp = x + 1 == g.L ? 0 : x + 1, xm = x == 0 ? g.L - 1 : x - 1;
    int tp = t + 1 == g.T ? 0 : t + 1, tm = t == 0 ? g.T - 1 : t - 1;
    long long cb = b * g.V;
    const double2* Uc = U + b * ustride;
    Spinor c = ld256_spinor_nc(psi, cb + s);
    Spinor vxp = ld256_spinor_nc(psi, cb + xp * g.T + t);
    Spinor vxm = ld256_spinor_nc(psi, cb + xm * g.T + t);
    Spinor vtp = ld256_spinor_nc(psi, cb + x * g.T + tp);
    Spinor vtm = ld256_spinor_nc(psi, cb + x * g.T + tm);
    double2 u0 = __ldg(Uc + s), u1 = __ldg(Uc + g.V + s);
    double2 u0m = __ldg(Uc + xm * g.T + t), u1m = __ldg(Uc + g.V + x * g.T + tm);
    st256_spinor(out, cb + s, wilson_site<DAG>(c, vxp, vxm, vtp, vtm, u0, u0m, u1, u1m, diag));
  }
}

// Per-chain complex dot sum conj(a) b (fermion.py:54-56); one CTA per (chain, slab).
__global__ void k_spinor_dot(const double2* __restrict__ a, const double2* __restrict__ b,
                             long long per_chain, int slabs, double* __restrict__ part) {
  __shared__ double slot[2][32];
  int c = blockIdx.y;
  long long lo = per_chain * blockIdx.x / slabs, hi = per_chain * (blockIdx.x + 1) / slabs;
  const double2* ac = a + (long long)c * per_chain;
  const double2* bc = b + (long long)c * per_chain;
  double re = 0.0, im = 0.0;
  for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    double2 x = __ldg(ac + i), y = __ldg(bc + i);
    re += x.x * y.x + x.y * y.y;
    im += x.x * y.y - x.y * y.x;
  }
  double sr = block_sum_rt(re, slot[0]);
  double si = block_sum_rt(im, slot[1]);
  if (threadIdx.x == 0) {
    part[2 * ((long long)c * slabs + blockIdx.x)] = sr;
    part[2 * ((long long)c * slabs + blockIdx.x) + 1] = si;
  }
}

__global__ void k_spinor_dot_finish(const double* __restrict__ part, int slabs, double* __restrict__ out,
                                    int B) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= B) return;
  double re = 0.0, im = 0.0;
  for (int k = 0; k < slabs; ++k) {
    re += part[2 * ((long long)c * slabs + k)];
    im += part[2 * ((long long)c * slabs + k) + 1];
  }
  out[2 * c] = re;
  out[2 * c + 1] = im;
}

// Fermion force f = -Im(A - B) (fermion.py:330-336).  KICK: out = p - dt*(f [+ beta*g])
// (kick_fermion / kick_full, integrators.py:172-186).
template <bool KICK>
__global__ void k_fermion_force(const double2* __restrict__ U, const double2* __restrict__ chi,
                                const double2* __restrict__ xi, const double* __restrict__ q,
                                double beta, const double* __restrict__ p, double dt,
                                double* __restrict__ out, Geo g) {
  long long n = (long long)g.B * g.V;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    long long b = i / g.V;
    int s = (int)(i - b * g.V);
    long long cb = b * g.V;
    const double2* Uc = U + 2 * cb;
    auto lc = [&](int k) { return ld256_spinor_nc(chi, cb + k); };
    auto lx = [&](int k) { return ld256_spinor_nc(xi, cb + k); };
    auto lu = [&](int mu, int k) { return __ldg(Uc + mu * g.V + k); };
    double f0, f1;
    force_site(s, g.L, g.T, lc, lx, lu, f0, f1);
    long long o0 = 2 * cb + s, o1 = o0 + g.V;
    if (KICK) {
      if (q) {   // kick_full: force = gauge_force + fermion_force
        const int x = s / g.T, t = s - x * g.T;
        int xm = x == 0 ? g.L - 1 : x - 1, tm = t == 0 ? g.T - 1 : t - 1;
        const double* qc = q + 2 * cb;
        double s0 = sin(plaq(qc, g.L, g.T, x, t));
        double st = sin(plaq(qc, g.L, g.T, x, tm));
        double sx = sin(plaq(qc, g.L, g.T, xm, t));
        f0 = __dadd_rn(__dmul_rn(beta, __dsub_rn(s0, st)), f0);
        f1 = __dadd_rn(__dmul_rn(beta, __dsub_rn(sx, s0)), f1);
      }
      out[o0] = __dsub_rn(p[o0], __dmul_rn(dt, f0));
      out[o1] = __dsub_rn(p[o1], __dmul_rn(dt, f1));
    } else {
      out[o0] = f0;
      out[o1] = f1;
    }
  }
}

// The two hopping contractions of link (n, mu) as fields (fermion.py:317-327):
// A(n) = conj(w-(a)(n)) U_mu(n) w-(b)(n+mu), B(n) = conj(w+(a)(n+mu)) conj(U_mu(n)) w+(b)(n),
// products evaluated left to right as NumPy does.
__global__ void k_link_bilinears(const double2* __restrict__ U, const double2* __restrict__ a,
                                 const double2* __restrict__ bv, int mu, double2* __restrict__ outA,
                                 double2* __restrict__ outB, Geo g) {
  long long n = (long long)g.B * g.V;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    long long b = i / g.V;
    int s = (int)(i - b * g.V);
    int x = s / g.T, t = s - x * g.T;
    int f = mu == 0 ? (x + 1 == g.L ? 0 : x + 1) * g.T + t : x * g.T + (t + 1 == g.T ? 0 : t + 1);
    long long cb = b * g.V;
    Spinor an = ld256_spinor_nc(a, cb + s), af = ld256_spinor_nc(a, cb + f);
    Spinor bn = ld256_spinor_nc(bv, cb + s), bf = ld256_spinor_nc(bv, cb + f);
    double2 u = __ldg(U + 2 * cb + (long long)mu * g.V + s);
    Bil r = mu == 0 ? bilinear<0>(an, af, bn, bf, u) : bilinear<1>(an, af, bn, bf, u);
    outA[cb + s] = r.A;
    outB[cb + s] = r.B;
  }
}

// Weighted w-sums (fermion.py:362-383, Appendix A5), gather form per site.
__global__ void k_wsums(const double2* __restrict__ U, const double* __restrict__ wt,
                        const double2* __restrict__ chi, const double2* __restrict__ xi,
                        double2* __restrict__ b1, double2* __restrict__ b2, Geo g) {
  long long n = (long long)g.B * g.V;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    long long b = i / g.V;
    int s = (int)(i - b * g.V);
    long long cb = b * g.V;
    const double2* Uc = U + 2 * cb;
    const double* Wc = wt + 2 * cb;
    auto lc = [&](int k) { return ld256_spinor_nc(chi, cb + k); };
    auto lx = [&](int k) { return ld256_spinor_nc(xi, cb + k); };
    auto lu = [&](int mu, int k) { return __ldg(Uc + mu * g.V + k); };
    auto lw = [&](int mu, int k) { return __ldg(Wc + mu * g.V + k); };
    Spinor o1, o2;
    wsums_site(s, g.L, g.T, lc, lx, lu, lw, o1, o2);
    const double2 o10 = o1.s0, o11 = o1.s1, o20 = o2.s0, o21 = o2.s1;
    long long o = cb + s;
    b1[2 * o] = o10;
    b1[2 * o + 1] = o11;
    b2[2 * o] = o20;
    b2[2 * o + 1] = o21;
  }
}

// C = 2Im(A[z1,xi]-B[z1,xi]) + 2Im(A[chi,z2]-B[chi,z2]) - 2Re(A[chi,xi]+B[chi,xi])*w
// (fermion.py:409-417)
__global__ void k_fg_combine(const double2* __restrict__ U, const double2* __restrict__ z1,
                             const double2* __restrict__ z2, const double2* __restrict__ chi,
                             const double2* __restrict__ xi, const double* __restrict__ wt,
                             double* __restrict__ out, Geo g) {
  long long n = (long long)g.B * g.V;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    long long b = i / g.V;
    int s = (int)(i - b * g.V);
    long long cb = b * g.V;
    const double2* Uc = U + 2 * cb;
    auto l1 = [&](int k) { return ld256_spinor_nc(z1, cb + k); };
    auto l2 = [&](int k) { return ld256_spinor_nc(z2, cb + k); };
    auto lc = [&](int k) { return ld256_spinor_nc(chi, cb + k); };
    auto lx = [&](int k) { return ld256_spinor_nc(xi, cb + k); };
    auto lu = [&](int mu, int k) { return __ldg(Uc + mu * g.V + k); };
    auto lw = [&](int mu, int k) { return __ldg(wt + 2 * cb + mu * g.V + k); };
    out[2 * cb + s] = fg_combine_site<0>(s, g.L, g.T, l1, l2, lc, lx, lu, lw);
    out[2 * cb + g.V + s] = fg_combine_site<1>(s, g.L, g.T, l1, l2, lc, lx, lu, lw);
  }
}

}  // namespace

extern "C" {

int sch_links_to_u(sch_ctx* ctx, const double* q, double* U, int B, int L, int T, int fermion_bc) {
  SCH_CHECK_ARG(ctx, q && U && B >= 1 && L >= 2 && T >= 2, "links_to_u: bad args");
  SCH_CHECK_ARG(ctx, fermion_bc == 0 || fermion_bc == 1, "links_to_u: fermion_bc must be 0 or 1");
  Geo g{B, L, T, (long long)L * T};
  k_links_to_u<<<grid_for((long long)B * 2 * g.V), 256, 0, ctx->stream>>>(q, (double2*)U, g,
                                                                         fermion_bc);
  SCH_LAUNCHED(ctx);
  return SCH_OK;
}

int sch_dslash(sch_ctx* ctx, const double* U, int u_batched, const double* psi, double* out, int B,
               int L, int T, double m0, int dagger) {
  SCH_CHECK_ARG(ctx, U && psi && out && B >= 1 && L >= 2 && T >= 2, "dslash: bad args");
  SCH_CHECK_ARG(ctx, psi != out, "dslash: in-place application is not supported");
  Geo g{B, L, T, (long long)L * T};
  long long us = u_batched ? 2 * g.V : 0;
  unsigned grid = grid_for((long long)B * g.V);
  if (dagger)
    k_dslash<true><<<grid, 256, 0, ctx->stream>>>((const double2*)U, us, (const double2*)psi,
                                                   (double2*)out, g, 2.0 + m0);
  else
    k_dslash<false><<<grid, 256, 0, ctx->stream>>>((const double2*)U, us, (const double2*)psi,
                                                    (double2*)out, g, 2.0 + m0);
  SCH_LAUNCHED(ctx);
  return SCH_OK;
}

int sch_ddagd(sch_ctx* ctx, const double* U, const double* psi, double* out, int B, int L, int T,
              double m0) {
  SCH_CHECK_ARG(ctx, U && psi && out && B >= 1 && L >= 2 && T >= 2, "ddagd: bad args");
  SCH_CHECK_ARG(ctx, psi != out, "ddagd: in-place application is not supported");
  TileArgs a{};
  a.U = (const double2*)U;
  a.in = (const double2*)psi;
  a.out = (double2*)out;
  a.B = B;
  a.L = L;
  a.T = T;
  a.diag = 2.0 + m0;
  int TX = 0;
  if (use_tma() && tma_tile_shape(L, T, TX)) {   // persistent TMA-pipelined tiles
    a.tiles_t = 1;
    a.tiles_per_chain = L / TX;
    launch_normal_tma<MODE_PLAIN>(a, ctx->stream, ctx->num_sms);
  } else {
    TileShape sh = pick_tile(L, T);
    a.tiles_t = sh.tiles_t;
    a.tiles_per_chain = sh.tiles_x * sh.tiles_t;
    launch_normal_tile<MODE_PLAIN>(sh, a, ctx->stream);
  }
  SCH_LAUNCHED(ctx);
  return SCH_OK;
}

int sch_spinor_dot(sch_ctx* ctx, const double* a, const double* b, double* out, int B, long long V) {
  SCH_CHECK_ARG(ctx, a && b && out && B >= 1 && V >= 1, "spinor_dot: bad args");
  long long per_chain = 2 * V;   // complex entries per chain
  int slabs = (int)((per_chain + 16383) / 16384);
  if (slabs > 256) slabs = 256;
  void* ws;
  int st = sch_workspace(ctx, sizeof(double) * 2 * (size_t)B * slabs, &ws);
  if (st) return st;
  k_spinor_dot<<<dim3(slabs, B), 256, 0, ctx->stream>>>((const double2*)a, (const double2*)b,
                                                         per_chain, slabs, (double*)ws);
  SCH_LAUNCHED(ctx);
  k_spinor_dot_finish<<<blocks_for(B, 128), 128, 0, ctx->stream>>>((const double*)ws, slabs, out, B);
  SCH_LAUNCHED(ctx);
  return SCH_OK;
}

int sch_fermion_force(sch_ctx* ctx, const double* U, const double* chi, const double* xi,
                      double* out, int B, int L, int T) {
  SCH_CHECK_ARG(ctx, U && chi && xi && out && B >= 1 && L >= 2 && T >= 2, "fermion_force: bad args");
  Geo g{B, L, T, (long long)L * T};
  k_fermion_force<false><<<grid_for((long long)B * g.V), 256, 0, ctx->stream>>>(
      (const double2*)U, (const double2*)chi, (const double2*)xi, nullptr, 0.0, nullptr, 0.0, out, g);
  SCH_LAUNCHED(ctx);
  return SCH_OK;
}

int sch_link_bilinears(sch_ctx* ctx, const double* U, const double* a, const double* b, int mu,
                       double* A, double* Bout, int B, int L, int T) {
  SCH_CHECK_ARG(ctx, U && a && b && A && Bout && (mu == 0 || mu == 1) && B >= 1 && L >= 2 && T >= 2,
                "link_bilinears: bad args");
  Geo g{B, L, T, (long long)L * T};
  k_link_bilinears<<<grid_for((long long)B * g.V), 256, 0, ctx->stream>>>(
      (const double2*)U, (const double2*)a, (const double2*)b, mu, (double2*)A, (double2*)Bout, g);
  SCH_LAUNCHED(ctx);
  return SCH_OK;
}

int sch_kick_fermion(sch_ctx* ctx, const double* U, const double* chi, const double* xi,
                     const double* q, double beta, const double* p, double dt, double* p_out, int B,
                     int L, int T) {
  SCH_CHECK_ARG(ctx, U && chi && xi && p && p_out && B >= 1 && L >= 2 && T >= 2,
                "kick_fermion: bad args");
  Geo g{B, L, T, (long long)L * T};
  k_fermion_force<true><<<grid_for((long long)B * g.V), 256, 0, ctx->stream>>>(
      (const double2*)U, (const double2*)chi, (const double2*)xi, q, beta, p, dt, p_out, g);
  SCH_LAUNCHED(ctx);
  return SCH_OK;
}

int sch_weighted_w_sums(sch_ctx* ctx, const double* U, const double* weight, const double* chi,
                        const double* xi, double* b1, double* b2, int B, int L, int T) {
  SCH_CHECK_ARG(ctx, U && weight && chi && xi && b1 && b2 && B >= 1 && L >= 2 && T >= 2,
                "weighted_w_sums: bad args");
  Geo g{B, L, T, (long long)L * T};
  k_wsums<<<grid_for((long long)B * g.V), 256, 0, ctx->stream>>>(
      (const double2*)U, weight, (const double2*)chi, (const double2*)xi, (double2*)b1, (double2*)b2, g);
  SCH_LAUNCHED(ctx);
  return SCH_OK;
}

int sch_fg_fermion_combine(sch_ctx* ctx, const double* U, const double* z1, const double* z2,
                           const double* chi, const double* xi, const double* weight, double* out,
                           int B, int L, int T) {
  SCH_CHECK_ARG(ctx, U && z1 && z2 && chi && xi && weight && out && B >= 1 && L >= 2 && T >= 2,
                "fg_fermion_combine: bad args");
  Geo g{B, L, T, (long long)L * T};
  k_fg_combine<<<grid_for((long long)B * g.V), 256, 0, ctx->stream>>>(
      (const double2*)U, (const double2*)z1, (const double2*)z2, (const double2*)chi,
      (const double2*)xi, weight, out, g);
  SCH_LAUNCHED(ctx);
  return SCH_OK;
}

}  // extern "C"
