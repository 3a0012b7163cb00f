// Link-field kernels: drift, kicks, gauge action/force, gauge force-gradient
// pieces and per-chain reductions.  Compiled with --fmad=false so every
// real-arithmetic update is evaluated exactly in NumPy's operation order
// (the drift and gauge force are then bit-identical to the reference for
// identical inputs, up to the libm-vs-CUDA sin/cos difference).
#include "common.cuh"
#include "site_ops.cuh"
#include "runtime.hpp"
#include "../../include/schwinger_sm100.h"

namespace {

__global__ void k_rotate(const double* __restrict__ q, const double* __restrict__ p, double h,
                         double* __restrict__ out, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = wrap_angle(q[i] + h * p[i]);
}

__global__ void k_wrap(const double* __restrict__ q, double* __restrict__ out, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = wrap_angle(q[i]);
}

// out = p - (a*f + c*g)  or  p - a*f
__global__ void k_kick(const double* __restrict__ p, const double* __restrict__ f, double a,
                       const double* __restrict__ g, double c, double* __restrict__ out,
                       long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    double k = a * f[i];
    if (g) k = k + c * g[i];
    out[i] = p[i] - k;
  }
}

struct Geo {
  int B, L, T;
  long long V;
};


__global__ void k_plaq_angles(const double* __restrict__ q, double* __restrict__ out, Geo g) {
  long long n = (long long)g.B * g.V;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    int b = (int)(i / g.V);
    int s = (int)(i - (long long)b * g.V);
    int x = s / g.T, t = s - (s / g.T) * g.T;
    out[i] = plaq(q + (long long)b * 2 * g.V, g.L, g.T, x, t);
  }
}

// gauge force beta*g, g0 = s - s(n-t), g1 = s(n-x) - s   (gauge.py:43-59),
// optionally fused with the kick p - dt*(beta*g) (integrators.py:161-164)
template <bool KICK>
__global__ void k_gauge_force(const double* __restrict__ q, double beta, const double* __restrict__ p,
                              double dt, double* __restrict__ out, Geo g) {
  long long n = (long long)g.B * g.V;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    int b = (int)(i / g.V);
    int s = (int)(i - (long long)b * g.V);
    int x = s / g.T, t = s - x * g.T;
    int xm = x == 0 ? g.L - 1 : x - 1;
    int tm = t == 0 ? g.T - 1 : t - 1;
    const double* qc = q + (long long)b * 2 * g.V;
    double s0 = sin(plaq(qc, g.L, g.T, x, t));
    double st = sin(plaq(qc, g.L, g.T, x, tm));
    double sx = sin(plaq(qc, g.L, g.T, xm, t));
    double f0 = beta * (s0 - st);
    double f1 = beta * (sx - s0);
    long long o0 = (long long)b * 2 * g.V + s, o1 = o0 + g.V;
    if (KICK) {
      out[o0] = p[o0] - dt * f0;
      out[o1] = p[o1] - dt * f1;
    } else {
      out[o0] = f0;
      out[o1] = f1;
    }
  }
}

// Fused inner leapfrog (integrators.py:253-259) for chains that fit in one
// CTA's shared memory: q, p and the plaquette sines stay on chip for all m
// micro steps.  Evaluation order per micro step is the reference's:
// kick(0.5*d) ; drift(d) ; kick(0.5*d).
__global__ void k_inner_leapfrog_resident(double* __restrict__ q, double* __restrict__ p,
                                          double beta, double half, double delta, int m, Geo g) {
  extern __shared__ double sm[];
  const int V = (int)g.V;
  double* sq = sm;            // 2V
  double* sp = sq + 2 * V;    // 2V
  double* ss = sp + 2 * V;    // V  (sin theta)
  double* qc = q + (long long)blockIdx.x * 2 * V;
  double* pc = p + (long long)blockIdx.x * 2 * V;
  for (int i = threadIdx.x; i < 2 * V; i += blockDim.x) {
    sq[i] = qc[i];
    sp[i] = pc[i];
  }
  __syncthreads();
  // sin(theta) is recomputed only after a drift: the second half kick of a
  // micro step and the first of the next act at the same links, so they share
  // the force values (the kicks themselves stay separate, as in the reference)
  bool fresh = false;
  auto kick = [&](double dt) {
    if (!fresh) {
      for (int s = threadIdx.x; s < V; s += blockDim.x) {
        int x = s / g.T, t = s - x * g.T;
        ss[s] = sin(plaq(sq, g.L, g.T, x, t));
      }
      __syncthreads();
      fresh = true;
    }
    for (int s = threadIdx.x; s < V; s += blockDim.x) {
      int x = s / g.T, t = s - x * g.T;
      int xm = x == 0 ? g.L - 1 : x - 1;
      int tm = t == 0 ? g.T - 1 : t - 1;
      double s0 = ss[s];
      double f0 = beta * (s0 - ss[x * g.T + tm]);
      double f1 = beta * (ss[xm * g.T + t] - s0);
      sp[s] = sp[s] - dt * f0;
      sp[V + s] = sp[V + s] - dt * f1;
    }
    __syncthreads();
  };
  for (int k = 0; k < m; ++k) {
    if (half != 0.0) kick(half);
    for (int i = threadIdx.x; i < 2 * V; i += blockDim.x) sq[i] = wrap_angle(sq[i] + delta * sp[i]);
    fresh = false;
    __syncthreads();
    if (half != 0.0) kick(half);
  }
  for (int i = threadIdx.x; i < 2 * V; i += blockDim.x) {
    qc[i] = sq[i];
    pc[i] = sp[i];
  }
}

// C_GG (gauge.py:97-107) from the eight translated mu-oriented plaquettes.
__global__ void k_fg_gauge_gauge(const double* __restrict__ q, double beta, double* __restrict__ out,
                                 Geo g) {
  long long n = (long long)g.B * g.V;
  const double bb2 = 2.0 * beta * beta;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    int b = (int)(i / g.V);
    int s = (int)(i - (long long)b * g.V);
    int x = s / g.T, t = s - x * g.T;
    const double* qc = q + (long long)b * 2 * g.V;
    for (int mu = 0; mu < 2; ++mu) {
      // offsets (dx, dt) of P1..P8 for link direction mu, nu = 1 - mu
      const int mx = mu == 0, mt = mu == 1, nx = mu == 1, nt = mu == 0;
      const int ox[8] = {0, -nx, mx, nx, -mx, -mx - nx, -2 * nx, mx - nx};
      const int ot[8] = {0, -nt, mt, nt, -mt, -mt - nt, -2 * nt, mt - nt};
      double re[8], im[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        int xx = x + ox[k], tt = t + ot[k];
        xx = xx < 0 ? xx + g.L : (xx >= g.L ? xx - g.L : xx);   // |offset| <= 2 <= L
        tt = tt < 0 ? tt + g.T : (tt >= g.T ? tt - g.T : tt);
        double th = plaq(qc, g.L, g.T, xx, tt);
        double sn, cs;
        sincos(th, &sn, &cs);
        re[k] = cs;
        im[k] = mu == 0 ? sn : -sn;   // mu = 1 uses the conjugate orientation
      }
      double first = ((((4.0 * im[0] - im[1]) - im[2]) - im[3]) - im[4]) * re[0];
      double second = ((((4.0 * im[1] - im[0]) - im[5]) - im[6]) - im[7]) * re[1];
      out[(long long)b * 2 * g.V + mu * g.V + s] = bb2 * (first - second);
    }
  }
}

// The mu-oriented plaquettes P1(n, mu) = e^{+-i theta} and (K = 8) their
// seven translates P2..P8 attached to link (n, mu) (gauge.py:62-95), as
// complex fields out[k][b][mu][x][t].
__global__ void k_plaquette_stencil(const double* __restrict__ q, double2* __restrict__ out, int K,
                                    Geo g) {
  long long n = (long long)g.B * g.V;
  const long long plane = (long long)g.B * 2 * g.V;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    int b = (int)(i / g.V);
    int s = (int)(i - (long long)b * g.V);
    int x = s / g.T, t = s - x * g.T;
    const double* qc = q + (long long)b * 2 * g.V;
    for (int mu = 0; mu < 2; ++mu) {
      const int mx = mu == 0, mt = mu == 1, nx = mu == 1, nt = mu == 0;
      const int ox[8] = {0, -nx, mx, nx, -mx, -mx - nx, -2 * nx, mx - nx};
      const int ot[8] = {0, -nt, mt, nt, -mt, -mt - nt, -2 * nt, mt - nt};
      for (int k = 0; k < K; ++k) {
        int xx = x + ox[k], tt = t + ot[k];
        xx = xx < 0 ? xx + g.L : (xx >= g.L ? xx - g.L : xx);
        tt = tt < 0 ? tt + g.T : (tt >= g.T ? tt - g.T : tt);
        double sn, cs;
        sincos(plaq(qc, g.L, g.T, xx, tt), &sn, &cs);
        out[k * plane + (long long)b * 2 * g.V + mu * g.V + s] = make_double2(cs, mu == 0 ? sn : -sn);
      }
    }
  }
}

// 2*beta*[(w(n,mu)+w(n+mu,nu)-w(n+nu,mu)-w(n,nu)) Re P1
//        +(w(n,mu)-w(n+mu-nu,nu)-w(n-nu,mu)+w(n-nu,nu)) Re P2]   (gauge.py:110-136)
__global__ void k_gauge_hessian_dot(const double* __restrict__ q, double beta,
                                    const double* __restrict__ w, double* __restrict__ out, Geo g) {
  long long n = (long long)g.B * g.V;
  const double b2 = 2.0 * beta;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    int b = (int)(i / g.V);
    int s = (int)(i - (long long)b * g.V);
    int x = s / g.T, t = s - x * g.T;
    const double* qc = q + (long long)b * 2 * g.V;
    const double* wc = w + (long long)b * 2 * g.V;
    auto at = [&](int dir, int dx, int dtt) {
      int xx = wrapi(x + dx, g.L), tt = wrapi(t + dtt, g.T);
      return wc[dir * g.V + xx * g.T + tt];
    };
    for (int mu = 0; mu < 2; ++mu) {
      const int nu = 1 - mu;
      const int mx = mu == 0, mt = mu == 1, nx = nu == 0, nt = nu == 1;
      double c1 = cos(plaq(qc, g.L, g.T, x, t));
      double c2 = cos(plaq(qc, g.L, g.T, wrapi(x - nx, g.L), wrapi(t - nt, g.T)));
      double wm = at(mu, 0, 0), wn = at(nu, 0, 0);
      double t1 = ((wm + at(nu, mx, mt)) - at(mu, nx, nt)) - wn;
      double t2 = ((wm - at(nu, mx - nx, mt - nt)) - at(mu, -nx, -nt)) + at(nu, -nx, -nt);
      out[(long long)b * 2 * g.V + mu * g.V + s] = b2 * (t1 * c1 + t2 * c2);
    }
  }
}

// ------------------------------------------------------------ reductions
// Per-chain deterministic sums.  One CTA per (chain, slab); the slab
// partials are reduced in a fixed order by a second pass when a chain spans
// more than one slab.
enum RedKind { RED_SQ_HALF = 0, RED_GAUGE_ACTION = 1, RED_AVG_PLAQ = 2 };

template <int KIND>
__device__ __forceinline__ double red_elem(const double* __restrict__ a, long long i, Geo g, int b) {
  if (KIND == RED_SQ_HALF) return a[i] * a[i];
  int s = (int)i;
  int x = s / g.T, t = s - x * g.T;
  double c = cos(plaq(a, g.L, g.T, x, t));
  return KIND == RED_GAUGE_ACTION ? 1.0 - c : c;
}

template <int KIND>
__global__ void k_chain_reduce(const double* __restrict__ a, long long per_chain, long long stride,
                               int slabs, double* __restrict__ part, Geo g) {
  __shared__ double slot[32];
  int b = blockIdx.y;
  long long lo = per_chain * blockIdx.x / slabs, hi = per_chain * (blockIdx.x + 1) / slabs;
  const double* ac = a + (long long)b * stride;
  double acc = 0.0;
  for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x) acc += red_elem<KIND>(ac, i, g, b);
  double s = block_sum_rt(acc, slot);
  if (threadIdx.x == 0) part[(long long)b * slabs + blockIdx.x] = s;
}

__global__ void k_reduce_finish(const double* __restrict__ part, int slabs, double scale_mul,
                                double scale_div, int mode, double* __restrict__ out, int B) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  double s = 0.0;
  for (int k = 0; k < slabs; ++k) s += part[(long long)b * slabs + k];
  // mode 0: s*mul ; mode 1: mul*s ; mode 2: s/div
  out[b] = mode == 0 ? s * scale_mul : (mode == 1 ? scale_mul * s : s / scale_div);
}

template <int KIND>
int chain_reduce(sch_ctx* ctx, const double* a, long long per_chain, long long stride, int B, Geo g,
                 double mul, double div, int mode, double* out) {
  int slabs = (int)((per_chain + 8191) / 8192);
  if (slabs > 256) slabs = 256;
  void* ws;
  int st = sch_workspace(ctx, sizeof(double) * (size_t)B * slabs, &ws);
  if (st) return st;
  double* part = (double*)ws;
  k_chain_reduce<KIND><<<dim3(slabs, B), 256, 0, ctx->stream>>>(a, per_chain, stride, slabs, part, g);
  SCH_LAUNCHED(ctx);
  k_reduce_finish<<<blocks_for(B, 128), 128, 0, ctx->stream>>>(part, slabs, mul, div, mode, out, B);
  SCH_LAUNCHED(ctx);
  return SCH_OK;
}

// Metropolis accept (hmc.py:54-60) with device uniforms: 1 accept, 0 reject,
// -1 non-finite dH (the caller raises ValueError).
__global__ void k_metropolis(const double* __restrict__ dh, const double* __restrict__ u,
                             int* __restrict__ acc, int B) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= B) return;
  double d = dh[c];
  if (!isfinite(d)) acc[c] = -1;
  else if (d <= 0.0) acc[c] = 1;
  else acc[c] = u[c] < exp(-d) ? 1 : 0;
}

// out[c] = accept[c] == 1 ? a[c] : b[c]   (per-chain Metropolis selection)
__global__ void k_select(const int* __restrict__ acc, const double* __restrict__ a,
                         const double* __restrict__ b, double* __restrict__ out, int B,
                         long long per_chain) {
  long long n = (long long)B * per_chain;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    int c = (int)(i / per_chain);
    out[i] = acc[c] == 1 ? a[i] : b[i];
  }
}

unsigned grid_for(long long n, int nt = 256) {
  long long b = (n + nt - 1) / nt;
  if (b > 148LL * 64) b = 148LL * 64;
  if (b < 1) b = 1;
  return (unsigned)b;
}

}  // namespace

extern "C" {

int sch_rotate_links(sch_ctx* ctx, const double* q, const double* p, double h, double* out,
                     long long n) {
  SCH_CHECK_ARG(ctx, q && p && out && n >= 0, "rotate_links: bad args");
  if (n == 0) return SCH_OK;
  k_rotate<<<grid_for(n), 256, 0, ctx->stream>>>(q, p, h, out, n);
  SCH_LAUNCHED(ctx);
  return SCH_OK;
}

int sch_wrap_angles(sch_ctx* ctx, const double* q, double* out, long long n) {
  SCH_CHECK_ARG(ctx, q && out && n >= 0, "wrap_angles: bad args");
  if (n == 0) return SCH_OK;
  k_wrap<<<grid_for(n), 256, 0, ctx->stream>>>(q, out, n);
  SCH_LAUNCHED(ctx);
  return SCH_OK;
}

int sch_kick(sch_ctx* ctx, const double* p, const double* f, double a, const double* g, double c,
             double* out, long long n) {
  SCH_CHECK_ARG(ctx, p && f && out && n >= 0, "kick: bad args");
  if (n == 0) return SCH_OK;
  k_kick<<<grid_for(n), 256, 0, ctx->stream>>>(p, f, a, g, c, out, n);
  SCH_LAUNCHED(ctx);
  return SCH_OK;
}

int sch_kinetic_energy(sch_ctx* ctx, const double* p, double* out, int B, long long per_chain) {
  SCH_CHECK_ARG(ctx, p && out && B >= 1 && per_chain >= 1, "kinetic_energy: bad args");
  Geo g{B, 1, 1, 1};
  // 0.5 * np.sum(p * p): the scalar multiplies the sum (lattice.py:130)
  return chain_reduce<RED_SQ_HALF>(ctx, p, per_chain, per_chain, B, g, 0.5, 1.0, 1, out);
}

int sch_plaquette_angles(sch_ctx* ctx, const double* q, double* out, int B, int L, int T) {
  SCH_CHECK_ARG(ctx, q && out && B >= 1 && L >= 2 && T >= 2, "plaquette_angles: bad args");
  Geo g{B, L, T, (long long)L * T};
  k_plaq_angles<<<grid_for((long long)B * g.V), 256, 0, ctx->stream>>>(q, out, g);
  SCH_LAUNCHED(ctx);
  return SCH_OK;
}

int sch_gauge_force(sch_ctx* ctx, const double* q, double beta, double* out, int B, int L, int T) {
  SCH_CHECK_ARG(ctx, q && out && B >= 1 && L >= 2 && T >= 2, "gauge_force: bad args");
  Geo g{B, L, T, (long long)L * T};
  k_gauge_force<false><<<grid_for((long long)B * g.V), 256, 0, ctx->stream>>>(q, beta, nullptr, 0.0,
                                                                              out, g);
  SCH_LAUNCHED(ctx);
  return SCH_OK;
}

int sch_kick_gauge(sch_ctx* ctx, const double* q, const double* p, double beta, double dt,
                   double* p_out, int B, int L, int T) {
  SCH_CHECK_ARG(ctx, q && p && p_out && B >= 1 && L >= 2 && T >= 2, "kick_gauge: bad args");
  Geo g{B, L, T, (long long)L * T};
  k_gauge_force<true><<<grid_for((long long)B * g.V), 256, 0, ctx->stream>>>(q, beta, p, dt, p_out, g);
  SCH_LAUNCHED(ctx);
  return SCH_OK;
}

int sch_inner_leapfrog(sch_ctx* ctx, double* q, double* p, double beta, double span, int m, int B,
                       int L, int T) {
  SCH_CHECK_ARG(ctx, q && p && B >= 1 && L >= 2 && T >= 2 && m >= 1, "inner_leapfrog: bad args");
  Geo g{B, L, T, (long long)L * T};
  const double delta = span / m;
  const double half = 0.5 * delta;
  size_t smem = sizeof(double) * 5 * (size_t)g.V;
  if (smem <= 200 * 1024) {
    static bool attr_set = false;
    if (!attr_set) {
      cudaFuncSetAttribute(k_inner_leapfrog_resident, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           200 * 1024);
      attr_set = true;
    }
    int nt = g.V >= 512 ? 512 : (g.V >= 256 ? 256 : 128);
    k_inner_leapfrog_resident<<<B, nt, smem, ctx->stream>>>(q, p, beta, half, delta, m, g);
    SCH_LAUNCHED(ctx);
    return SCH_OK;
  }
  long long n = (long long)B * 2 * g.V;
  for (int k = 0; k < m; ++k) {
    if (half != 0.0) {
      k_gauge_force<true><<<grid_for(B * g.V), 256, 0, ctx->stream>>>(q, beta, p, half, p, g);
      SCH_LAUNCHED(ctx);
    }
    k_rotate<<<grid_for(n), 256, 0, ctx->stream>>>(q, p, delta, q, n);
    SCH_LAUNCHED(ctx);
    if (half != 0.0) {
      k_gauge_force<true><<<grid_for(B * g.V), 256, 0, ctx->stream>>>(q, beta, p, half, p, g);
      SCH_LAUNCHED(ctx);
    }
  }
  return SCH_OK;
}

int sch_gauge_action(sch_ctx* ctx, const double* q, double beta, double* out, int B, int L, int T) {
  SCH_CHECK_ARG(ctx, q && out && B >= 1 && L >= 2 && T >= 2, "gauge_action: bad args");
  Geo g{B, L, T, (long long)L * T};
  // beta * np.sum(1 - cos theta)   (gauge.py:40)
  return chain_reduce<RED_GAUGE_ACTION>(ctx, q, g.V, 2 * g.V, B, g, beta, 1.0, 1, out);
}

int sch_avg_plaquette(sch_ctx* ctx, const double* q, double* out, int B, int L, int T) {
  SCH_CHECK_ARG(ctx, q && out && B >= 1 && L >= 2 && T >= 2, "avg_plaquette: bad args");
  Geo g{B, L, T, (long long)L * T};
  return chain_reduce<RED_AVG_PLAQ>(ctx, q, g.V, 2 * g.V, B, g, 1.0, (double)g.V, 2, out);
}

int sch_fg_gauge_gauge(sch_ctx* ctx, const double* q, double beta, double* out, int B, int L, int T) {
  SCH_CHECK_ARG(ctx, q && out && B >= 1 && L >= 2 && T >= 2, "fg_gauge_gauge: bad args");
  Geo g{B, L, T, (long long)L * T};
  k_fg_gauge_gauge<<<grid_for((long long)B * g.V), 256, 0, ctx->stream>>>(q, beta, out, g);
  SCH_LAUNCHED(ctx);
  return SCH_OK;
}

int sch_plaquette_stencil(sch_ctx* ctx, const double* q, double* out, int K, int B, int L, int T) {
  SCH_CHECK_ARG(ctx, q && out && (K == 1 || K == 8) && B >= 1 && L >= 2 && T >= 2,
                "plaquette_stencil: bad args");
  Geo g{B, L, T, (long long)L * T};
  k_plaquette_stencil<<<grid_for((long long)B * g.V), 256, 0, ctx->stream>>>(q, (double2*)out, K, g);
  SCH_LAUNCHED(ctx);
  return SCH_OK;
}

int sch_gauge_hessian_dot(sch_ctx* ctx, const double* q, double beta, const double* w, double* out,
                          int B, int L, int T) {
  SCH_CHECK_ARG(ctx, q && w && out && B >= 1 && L >= 2 && T >= 2, "gauge_hessian_dot: bad args");
  Geo g{B, L, T, (long long)L * T};
  k_gauge_hessian_dot<<<grid_for((long long)B * g.V), 256, 0, ctx->stream>>>(q, beta, w, out, g);
  SCH_LAUNCHED(ctx);
  return SCH_OK;
}

int sch_metropolis(sch_ctx* ctx, const double* dh, const double* u, int* accept, int B) {
  SCH_CHECK_ARG(ctx, dh && u && accept && B >= 1, "metropolis: bad args");
  k_metropolis<<<blocks_for(B, 128), 128, 0, ctx->stream>>>(dh, u, accept, B);
  SCH_LAUNCHED(ctx);
  return SCH_OK;
}

int sch_select_chains(sch_ctx* ctx, const int* accept, const double* a, const double* b,
                      double* out, int B, long long per_chain) {
  SCH_CHECK_ARG(ctx, accept && a && b && out && B >= 1 && per_chain >= 1, "select_chains: bad args");
  k_select<<<grid_for((long long)B * per_chain), 256, 0, ctx->stream>>>(accept, a, b, out, B, per_chain);
  SCH_LAUNCHED(ctx);
  return SCH_OK;
}

}  // extern "C"
