// Trajectory megakernel: one CTA runs a whole HMC
// trajectory of one 16x16 chain — both Hamiltonians, every kick, inner flow
// and CG solve of the adapted nested force-gradient scheme — in a single
// launch for the whole ensemble.
//
// What it removes from the batched path (hmc.py _ensemble_update): the ~90
// kernel launches per update and, more importantly, the 17 per-solve
// waves of the resident CG (each launch ends in a tail where SMs idle while
// the slowest chains finish).  Here a CTA that finishes early simply starts
// its next phase; the only tail is the trajectory's.
//
// Schedule (integrators.py:341-349, adapted-nested-fg, n macro steps of h,
// M micro steps per inner flow), with the batched path's solve reuse:
//   H0 = (kin + S_G) + Re<eta, xi>,  xi = CG(eta) at q0, chi = D xi
//   step j:  Kf(h/6) [the pair at q_j]  I(h/2)
//            G(2h/3): xi = CG(eta), chi = D xi, f, (b1, b2) = wsums(f),
//                     Z1 = D CG(b1), Z2 = CG(D^dag(b2 + Z1)), C = combine,
//                     p -= (2h/3) f + (FG_KICK_SIGN fgc h^3) C
//            I(h/2)   xi = CG(eta) at q_{j+1}, chi = D xi   Kf(h/6)
//   H1 from the last pair.
// Every per-site formula is the batched kernels' (site_ops.cuh, wilson_site,
// cg_resblk_run); the Hamiltonian sums reproduce the batched reductions'
// summation trees (256-thread block sums) exactly, so dH and the final links
// equal the batched path's.
//
// State: q, p, the plaquette sines, U, xi and chi in shared memory (50 KB
// per CTA, 4 CTAs per SM as the batched CG); the FG fields and the solves'
// right-hand sides in a per-chain global scratch (L2-resident while the
// chain runs).  Fields written inside the kernel are read back with generic
// coherent loads.
#include "common.cuh"
#include "resident_col.cuh"
#include "runtime.hpp"
#include "site_ops.cuh"
#include "../../include/schwinger_sm100.h"

namespace {

constexpr int ML = 16, MT = 16, MV = ML * MT;
constexpr int MNT = 64;                       // threads per chain (2x2 sites each in the CG)
constexpr int MPL = 2 * (2 * 2 + 2 * 2) * MNT;   // CG exchange planes (double2)
// per-chain global scratch, in double2 units
enum { SC_Y = 0, SC_Z1 = 2 * MV, SC_Z2 = 4 * MV, SC_B1 = 6 * MV, SC_B2 = 8 * MV, SC_RHS = 10 * MV,
       SC_F = 12 * MV, SC_FG = 13 * MV, SC_SIZE = 14 * MV };
// shared memory, in double2 units: CG planes | q p (2V doubles each) | sines (V doubles) | U | xi | chi
constexpr int SM_Q = MPL, SM_SS = SM_Q + 2 * MV, SM_U = SM_SS + MV / 2, SM_XI = SM_U + 2 * MV,
              SM_CHI = SM_XI + 2 * MV, SM_SIZE = SM_CHI + 2 * MV;

// generic (shared or global) spinor access: two 128-bit loads / stores
SCH_DEV Spinor ldg_any(const double2* p, int k) {
  Spinor v;
  v.s0 = p[2 * k];
  v.s1 = p[2 * k + 1];
  return v;
}
SCH_DEV void stg_any(double2* p, int k, const Spinor& v) {
  p[2 * k] = v.s0;
  p[2 * k + 1] = v.s1;
}

struct MegaArgs {
  const double* q_in;    // [B][2][V]
  const double* p_in;    // [B][2][V]
  const double2* eta;    // [B][V][2]
  double* q_out;         // [B][2][V]
  double2* scratch;      // [B][SC_SIZE]
  double* dh;            // [B]
  int* status;           // [B]: 1 if a CG hit maxiter
  int* iters;            // [B]: CG iterations of the trajectory
  int* cg_it;            // [B] per-solve outputs of cg_resblk_run
  double* cg_rel;        // [B]
  int* cg_st;            // [B]
  double beta, diag, tol;
  int maxiter;
  double dt_kf, b_g, c_g, span_i;   // h/6, 2h/3, FG_KICK_SIGN*fgc*h^3, h/2 (host-computed)
  int n_steps, micro;
  int B;
};

// 256-thread block sum (common.cuh block_sum_rt) emulated by 64 threads, so
// the Hamiltonian pieces carry the batched reductions' bits: virtual thread
// v = tid + 64 j holds vals[j]; virtual warp (v / 32) = warp + 2 j.
SCH_DEV double block_sum_256(const double* vals, double* slot8) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const double s = warp_sum(vals[j]);
    if (lane == 0) slot8[w + 2 * j] = s;
  }
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += slot8[k];
  __syncthreads();
  return s;
}

__global__ void __launch_bounds__(MNT, 4) k_traj_anfg16(MegaArgs a) {
  extern __shared__ double2 smem[];
  double2* cgsm = smem;                                    // MPL double2
  double* sq = reinterpret_cast<double*>(smem + SM_Q);     // 2V
  double* sp = sq + 2 * MV;                                // 2V
  double* ss = reinterpret_cast<double*>(smem + SM_SS);    // V plaquette sines
  double2* U = smem + SM_U;
  double2* xi = smem + SM_XI;
  double2* chi = smem + SM_CHI;
  __shared__ double slot8[8];
  const int c = blockIdx.x;
  const int tid = threadIdx.x;
  double2* scr = a.scratch + (long long)c * SC_SIZE;
  double* F = reinterpret_cast<double*>(scr + SC_F);
  double* FG = reinterpret_cast<double*>(scr + SC_FG);
  const double2* eta = a.eta + (long long)c * 2 * MV;

#pragma unroll
  for (int i = tid; i < 2 * MV; i += MNT) {
    sq[i] = a.q_in[(long long)c * 2 * MV + i];
    sp[i] = a.p_in[(long long)c * 2 * MV + i];
  }
  __syncthreads();

  // coherent loaders of per-chain fields
  auto lsp = [](const double2* f) { return [f](int k) { return ldg_any(f, k); }; };
  auto lu = [&](int mu, int k) { return U[mu * MV + k]; };

  auto links = [&]() {   // U = exp(i q)  (fermion.py:94; k_links_to_u)
#pragma unroll
    for (int i = tid; i < 2 * MV; i += MNT) {
      double sn, cs;
      sincos(sq[i], &sn, &cs);
      U[i] = make_double2(cs, sn);
    }
    __syncthreads();
  };
  auto dslash = [&](auto dag, const double2* in, double2* out) {   // k_dslash
    constexpr bool DAG = decltype(dag)::value;
#pragma unroll
    for (int s = tid; s < MV; s += MNT) {
      const Nbr n = nbr(s, ML, MT);
      const Spinor cv = ldg_any(in, s);
      const Spinor vxp = ldg_any(in, n.xp * MT + n.t), vxm = ldg_any(in, n.xm * MT + n.t);
      const Spinor vtp = ldg_any(in, n.x * MT + n.tp), vtm = ldg_any(in, n.x * MT + n.tm);
      const double2 u0 = U[s], u1 = U[MV + s];
      const double2 u0m = U[n.xm * MT + n.t], u1m = U[MV + n.x * MT + n.tm];
      stg_any(out, s, wilson_site<DAG>(cv, vxp, vxm, vtp, vtm, u0, u0m, u1, u1m, a.diag));
    }
    __syncthreads();
  };
  // trajectory state that lives across the solves is kept in shared memory,
  // so the inlined solver keeps the register file (it is FP64-latency bound
  // and loses ILP with fewer registers)
  __shared__ int sh_it, sh_st;
  __shared__ double sh_h0;
  if (tid == 0) {
    sh_it = 0;
    sh_st = 0;
  }
  auto cg = [&](const double2* b, double2* x) {   // cg_normal, per-chain stop (resident engine)
    ResArgs r{};
    r.U = U;
    r.b = b;
    r.x0 = nullptr;
    r.x = x;
    r.iters = a.cg_it;
    r.relres = a.cg_rel;
    r.status = a.cg_st;
    r.L = ML;
    r.T = MT;
    r.diag = a.diag;
    r.tol = a.tol;
    r.maxiter = a.maxiter;
    cg_resblk_run<ML, MT, 2, 2, 1, true, true>(r, c, 0, cgsm);
    __syncthreads();
    if (tid == 0) {
      sh_it += a.cg_it[c];
      sh_st |= a.cg_st[c];
    }
  };
  auto kick_fermion = [&](double dt) {   // p -= dt f(chi, xi)  (k_fermion_force<true>)
#pragma unroll
    for (int s = tid; s < MV; s += MNT) {
      double f0, f1;
      force_site(s, ML, MT, lsp(chi), lsp(xi), lu, f0, f1);
      sp[s] = kick_elem(sp[s], dt, f0);
      sp[MV + s] = kick_elem(sp[MV + s], dt, f1);
    }
    __syncthreads();
  };
  auto inner_leapfrog = [&](double span, int m) {   // k_inner_leapfrog_resident
    const double delta = span / m;
    const double half = 0.5 * delta;
    bool fresh = false;
    auto kick = [&](double dt) {
      if (!fresh) {
#pragma unroll
        for (int s = tid; s < MV; s += MNT) {
          const int x = s / MT, t = s - x * MT;
          ss[s] = sin(plaq(sq, ML, MT, x, t));
        }
        __syncthreads();
        fresh = true;
      }
#pragma unroll
      for (int s = tid; s < MV; s += MNT) {
        const Nbr n = nbr(s, ML, MT);
        double f0, f1;
        gauge_force_from_sines(a.beta, ss[s], ss[n.x * MT + n.tm], ss[n.xm * MT + n.t], f0, f1);
        sp[s] = kick_elem(sp[s], dt, f0);
        sp[MV + s] = kick_elem(sp[MV + s], dt, f1);
      }
      __syncthreads();
    };
    for (int k = 0; k < m; ++k) {
      if (half != 0.0) kick(half);
#pragma unroll
      for (int i = tid; i < 2 * MV; i += MNT) sq[i] = rotate_elem(sq[i], sp[i], delta);
      fresh = false;
      __syncthreads();
      if (half != 0.0) kick(half);
    }
  };
  auto hamiltonian = [&]() {   // (kin + S_G) + Re<eta, xi>  (hmc.py:44-51)
    double v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {   // kinetic: 0.5 * sum p^2 (k_chain_reduce, fmad off)
      const int k = tid + MNT * j;
      double acc = __dadd_rn(0.0, __dmul_rn(sp[k], sp[k]));
      v[j] = __dadd_rn(acc, __dmul_rn(sp[k + MV], sp[k + MV]));
    }
    const double kin = __dmul_rn(0.5, block_sum_256(v, slot8));
#pragma unroll
    for (int j = 0; j < 4; ++j) {   // gauge action: beta * sum(1 - cos theta)
      const int s = tid + MNT * j;
      const int x = s / MT, t = s - x * MT;
      v[j] = __dadd_rn(0.0, __dsub_rn(1.0, cos(plaq(sq, ML, MT, x, t))));
    }
    const double sg = __dmul_rn(a.beta, block_sum_256(v, slot8));
#pragma unroll
    for (int j = 0; j < 4; ++j) {   // Re sum conj(eta) xi (k_spinor_dot: entries k, k + 256)
      const int k = tid + MNT * j;
      double re = 0.0;
      for (int e = k; e < 2 * MV; e += 256) {
        const double2 x = eta[e], y = xi[e];
        re += x.x * y.x + x.y * y.y;
      }
      v[j] = re;
    }
    const double sf = 0.0 + block_sum_256(v, slot8);
    return __dadd_rn(__dadd_rn(kin, sg), sf);
  };

  // One CG call site for all 1 + 4n solves (a single inlined copy of the
  // solver); role of solve k: 4 = the pair at q0 (H0), then per macro step
  // 0 = the G kick's pair, 1 = CG(b1) for Z1, 2 = CG(D^dag(b2 + Z1)) = Z2,
  // 3 = the pair at the step's end (its last Kf and the next step's first).
  double2* b1 = scr + SC_B1;
  double2* b2 = scr + SC_B2;
  double2* y = scr + SC_Y;
  double2* z1 = scr + SC_Z1;
  double2* z2 = scr + SC_Z2;
  double2* rhs = scr + SC_RHS;
  using Fd = std::integral_constant<bool, false>;
  using Td = std::integral_constant<bool, true>;
  const int nsolves = 1 + 4 * a.n_steps;
  for (int k = 0; k < nsolves; ++k) {
    const int role = k == 0 ? 4 : (k - 1) % 4;
    const double2* b = eta;
    double2* x = xi;
    if (role == 0) {   // Kf(h/6) with the pair at q_j, then I(h/2), then the G pair
      kick_fermion(a.dt_kf);
      inner_leapfrog(a.span_i, a.micro);
    }
    if (role == 0 || role == 3 || role == 4) links();
    if (role == 1) { b = b1; x = y; }
    if (role == 2) { b = rhs; x = z2; }
    cg(b, x);
    if (role == 0 || role == 3 || role == 4) dslash(Fd{}, xi, chi);
    if (role == 4) {
      const double h = hamiltonian();
      if (tid == 0) sh_h0 = h;
    }
    if (role == 3) kick_fermion(a.dt_kf);
    if (role == 0) {   // f and the weighted w-sums (fermion.py:362-383)
#pragma unroll
      for (int s = tid; s < MV; s += MNT) {
        double f0, f1;
        force_site(s, ML, MT, lsp(chi), lsp(xi), lu, f0, f1);
        F[s] = f0;
        F[MV + s] = f1;
      }
      __syncthreads();
#pragma unroll
      for (int s = tid; s < MV; s += MNT) {
        Spinor o1, o2;
        wsums_site(s, ML, MT, lsp(chi), lsp(xi), lu, [&](int mu, int q) { return F[mu * MV + q]; },
                   o1, o2);
        stg_any(b1, s, o1);
        stg_any(b2, s, o2);
      }
      __syncthreads();
    }
    if (role == 1) {   // Z1 = D y; rhs = D^dag (b2 + Z1)  (fermion.py:386-394)
      dslash(Fd{}, y, z1);
#pragma unroll
      for (int e = tid; e < 2 * MV; e += MNT) {
        const double2 u = b2[e], w = z1[e];
        b2[e] = make_double2(__dadd_rn(u.x, w.x), __dadd_rn(u.y, w.y));
      }
      __syncthreads();
      dslash(Td{}, b2, rhs);
    }
    if (role == 2) {   // C (k_fg_combine), the FG kick (k_kick), I(h/2)
#pragma unroll
      for (int s = tid; s < MV; s += MNT) {
        auto lw = [&](int mu, int q) { return F[mu * MV + q]; };
        FG[s] = fg_combine_site<0>(s, ML, MT, lsp(z1), lsp(z2), lsp(chi), lsp(xi), lu, lw);
        FG[MV + s] = fg_combine_site<1>(s, ML, MT, lsp(z1), lsp(z2), lsp(chi), lsp(xi), lu, lw);
      }
      __syncthreads();
#pragma unroll
      for (int i = tid; i < 2 * MV; i += MNT) sp[i] = kick2_elem(sp[i], a.b_g, F[i], a.c_g, FG[i]);
      __syncthreads();
      inner_leapfrog(a.span_i, a.micro);
    }
  }
  const double h1 = hamiltonian();
#pragma unroll
  for (int i = tid; i < 2 * MV; i += MNT) a.q_out[(long long)c * 2 * MV + i] = sq[i];
  if (tid == 0) {
    a.dh[c] = __dsub_rn(h1, sh_h0);
    a.status[c] = sh_st;
    a.iters[c] = sh_it;
  }
}

}  // namespace

extern "C" {

// One adapted-nested-fg trajectory of B independent 16x16 chains (periodic
// fermion boundaries, per-chain CG stop), one CTA per chain: q_in, p, eta in;
// q_out, dh = H(end) - H(start), status (1: a CG hit maxiter) and the CG
// iterations per chain out.  Scalars as the batched path computes them:
// dt_kf = h/6, b_g = 2h/3, c_g = FG_KICK_SIGN * fgc * h^3, span = h/2.
int sch_traj_anfg16(sch_ctx* ctx, const double* q_in, const double* p, const double* eta,
                    double* q_out, double* dh, int* status, int* iters, int B, double beta, double m0,
                    double tol, int maxiter, double dt_kf, double b_g, double c_g, double span,
                    int n_steps, int micro) {
  SCH_CHECK_ARG(ctx, q_in && p && eta && q_out && dh && status && iters && B >= 1 && n_steps >= 1 &&
                         micro >= 1 && maxiter >= 1,
                "traj_anfg16: bad args");
  SCH_CHECK_ARG(ctx, q_out != q_in, "traj_anfg16: q_out aliases q_in");
  const size_t scr = sizeof(double2) * (size_t)SC_SIZE * B;
  const size_t small = 3 * sizeof(double) * (size_t)B + 256;
  void* ws;
  int rc = sch_workspace(ctx, scr + small, &ws);
  if (rc) return rc;
  MegaArgs a{};
  a.q_in = q_in;
  a.p_in = p;
  a.eta = (const double2*)eta;
  a.q_out = q_out;
  a.scratch = (double2*)ws;
  char* tail = (char*)ws + scr;
  a.cg_rel = (double*)tail;
  a.cg_it = (int*)(tail + sizeof(double) * B);
  a.cg_st = (int*)(tail + sizeof(double) * B + sizeof(int) * B);
  a.dh = dh;
  a.status = status;
  a.iters = iters;
  a.beta = beta;
  a.diag = 2.0 + m0;
  a.tol = tol;
  a.maxiter = maxiter;
  a.dt_kf = dt_kf;
  a.b_g = b_g;
  a.c_g = c_g;
  a.span_i = span;
  a.n_steps = n_steps;
  a.micro = micro;
  a.B = B;
  const size_t smem = sizeof(double2) * SM_SIZE;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_traj_anfg16, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return sch_fail(ctx, SCH_ERR_CUDA, "traj smem attr: %s", cudaGetErrorString(e));
    attr = true;
  }
  k_traj_anfg16<<<B, MNT, smem, ctx->stream>>>(a);
  SCH_LAUNCHED(ctx);
  return SCH_OK;
}

}  // extern "C"
