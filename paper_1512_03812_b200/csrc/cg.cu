// Conjugate gradient on the Wilson normal operator D^dag D, with the exact
// stopping semantics of the reference cg_normal (fermion.py:171-217):
//
//   normb = ||b||, target = tol*normb;  x = 0 | x0;  r = b - A x;  p = r
//   for it = 1..maxiter:
//     ap = A p;  alpha = <p,ap> > 0 ? rs/<p,ap> : 0;  x += alpha p
//     r = (it % 50 == 0) ? b - A x : r - alpha ap;   rs' = ||r||^2
//     if sqrt(rs') <= target:                        (true-residual re-check)
//        tr = b - A x; if ||tr|| <= target: return;  r = tr; rs' = ||tr||^2
//     beta = rs > 0 ? rs'/rs : 0;  p = r + beta p;  rs = rs'
//
// Two engines:
//  * resident  : one CTA owns one chain for the whole solve (V <= 2048).  U,
//                p and D p live in shared memory, x and r in registers; the
//                solve is a single launch with no host round trips.  Used for
//                per-chain stopping (the hmc_update semantics) — the 16^2 and
//                32^2 ensembles of BASELINE configs 1-3.
//  * streaming : HBM-resident vectors, one fused D^dag D tile pass + one
//                fused update pass per iteration (352 B/site/iteration, SURVEY
//                §8(d)), tiny per-chain control kernels, and a host loop that
//                enqueues iterations in chunks and polls a device flag.  Used
//                for batch_global stopping (measure_dh semantics) and lattices
//                too large for one CTA (configs 4-5).
#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"
#include "runtime.hpp"
#include "tile.cuh"
#include "tma_tile.cuh"
#include "resident.cuh"
#include "resident_col.cuh"
#include "resident_cluster.cuh"
#include <cstdio>
#include <cstdlib>
#include "../../include/schwinger_sm100.h"

namespace {

constexpr int kReplace = kResReplace;   // residual replacement period (fermion.py:199)

// ============================================================ resident CG
// (kernel in resident.cuh)

template <int NT, int SPT, int MINB, int LC = 0, int TC = 0>
int launch_resident(sch_ctx* ctx, const ResArgs& a, int B) {
  const size_t smem = sizeof(double2) * 8 * (size_t)a.L * a.T;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_cg_resident<NT, SPT, MINB, LC, TC>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return sch_fail(ctx, SCH_ERR_CUDA, "smem attr: %s", cudaGetErrorString(e));
    attr = true;
  }
  k_cg_resident<NT, SPT, MINB, LC, TC><<<B, NT, smem, ctx->stream>>>(a);
  SCH_LAUNCHED(ctx);
  return SCH_OK;
}

template <int LC, int TC, int BX, int BT, int MINB, int TSH = 0, bool ROT = false>
int launch_resblk(sch_ctx* ctx, const ResArgs& a, int B) {
  constexpr int NT = LC * TC / (BX * BT);
  const size_t smem = sizeof(double2) * 2 * (2 * BT + 2 * BX) * NT;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_cg_resblk<LC, TC, BX, BT, MINB, TSH, ROT>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return sch_fail(ctx, SCH_ERR_CUDA, "smem attr: %s", cudaGetErrorString(e));
    attr = true;
  }
  k_cg_resblk<LC, TC, BX, BT, MINB, TSH, ROT><<<B, NT, smem, ctx->stream>>>(a);
  SCH_LAUNCHED(ctx);
  return SCH_OK;
}

// Resident-engine instantiation for V sites.  16x16 and 32x32 run the
// block-owned kernel (2x2 sites per thread; resident_col.cuh: 16^2 2.26 ns,
// 32^2 10.76 ns per chain-iteration); other shapes the strided kernel
// (resident.cuh).  SCH_RESIDENT="NTxSPTxMINBxSPEC" forces a strided
// instantiation for tuning runs (SPEC 1 = compile-time shape, 0 = generic).
// Resident CG in the sigma1-diagonal spin basis (block_stencil.cuh; default,
// measured 16^2 2.25 -> 2.07 ns and 32^2 10.48 -> 9.32 ns per chain-iteration);
// SCH_RESBLK_ROT=0 runs the reference basis.
bool resblk_rot() {
  static int rot = -1;
  if (rot < 0) {
    const char* e = getenv("SCH_RESBLK_ROT");
    rot = (e && e[0] == '0') ? 0 : 1;
  }
  return rot != 0;
}

struct ResidentForce {
  int nt = 0, spt = 0, minb = 0, spec = 1;
};
const ResidentForce& resident_force() {
  static ResidentForce f;
  static bool read = false;
  if (!read) {
    read = true;
    if (const char* e = getenv("SCH_RESIDENT")) sscanf(e, "%dx%dx%dx%d", &f.nt, &f.spt, &f.minb, &f.spec);
  }
  return f;
}
bool resident_forced(long long V) {
  const ResidentForce& f = resident_force();
  return f.nt > 0 && (long long)f.nt * f.spt >= V;
}
int resident_dispatch(sch_ctx* ctx, const ResArgs& a, int B, long long V) {
  const ResidentForce& rf = resident_force();
  const int fnt = rf.nt, fspt = rf.spt, fminb = rf.minb, fspec = rf.spec;
  const bool forced = resident_forced(V);
  const bool rot = resblk_rot();
  if (!forced && a.L == 16 && a.T == 16) {
    if (rot) return launch_resblk<16, 16, 2, 2, 4, 1, true>(ctx, a, B);
    return launch_resblk<16, 16, 2, 2, 4, 1>(ctx, a, B);
  }
  if (!forced && a.L == 32 && a.T == 32) {
    if (rot) return launch_resblk<32, 32, 2, 2, 1, 1, true>(ctx, a, B);
    return launch_resblk<32, 32, 2, 2, 1, 1>(ctx, a, B);
  }
  int nt, spt, minb;
  bool spec = true;
  if (forced) {
    nt = fnt; spt = fspt; minb = fminb; spec = fspec != 0;
  } else if (V <= 128) { nt = 128; spt = 1; minb = 1; }
  else if (V <= 256) { nt = 128; spt = 2; minb = 4; }
  else if (V <= 512) { nt = 256; spt = 2; minb = 1; }
  else { nt = 256; spt = 4; minb = 1; }
  const bool s16 = spec && a.L == 16 && a.T == 16 && (long long)nt * spt == 256;
  const bool s32 = spec && a.L == 32 && a.T == 32 && (long long)nt * spt == 1024;
#define SCH_RES(N, S, M) \
  if (nt == N && spt == S && minb == M) return launch_resident<N, S, M>(ctx, a, B);
#define SCH_RES16(N, S, M) \
  if (s16 && nt == N && spt == S && minb == M) return launch_resident<N, S, M, 16, 16>(ctx, a, B);
#define SCH_RES32(N, S, M) \
  if (s32 && nt == N && spt == S && minb == M) return launch_resident<N, S, M, 32, 32>(ctx, a, B);
  SCH_RES16(128, 2, 4) SCH_RES32(256, 4, 1)
  SCH_RES(128, 1, 1) SCH_RES(128, 2, 1) SCH_RES(128, 2, 4)
  SCH_RES(256, 1, 4) SCH_RES(256, 2, 1) SCH_RES(256, 4, 1) SCH_RES(512, 2, 1)
#undef SCH_RES
#undef SCH_RES16
#undef SCH_RES32
  return sch_fail(ctx, SCH_ERR_ARG, "no resident CG instantiation %dx%dx%d", nt, spt, minb);
}

// Cluster-resident CG (resident_cluster.cuh): CS CTAs per chain.
template <int LC, int TC, int CS, int BX, int BT, int MINB, bool ROT = true>
int launch_cluster_tx(sch_ctx* ctx, const ResArgs& a, int B) {
  constexpr int NT = LC * TC / (CS * BX * BT);
  constexpr int PL = (2 * BT + 2 * BX) * NT;
  constexpr int FACE = BT * (TC / BT);
  const size_t smem = sizeof(double2) * (2 * PL + 8 * FACE);
  auto kern = k_cg_cluster_tx<LC, TC, CS, BX, BT, MINB, ROT>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e == cudaSuccess && CS > 8)
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return sch_fail(ctx, SCH_ERR_CUDA, "cluster attr: %s", cudaGetErrorString(e));
    attr = true;
  }
  kern<<<B * CS, NT, smem, ctx->stream>>>(a);
  SCH_LAUNCHED(ctx);
  return SCH_OK;
}

// 64^2 (cfg4): the 4-CTA cluster kernel (measured: 62.2 ns per chain-
// iteration; 8-CTA clusters 62.6, the cluster-barrier variant 78.5)
int cluster_dispatch(sch_ctx* ctx, const ResArgs& a, int B) {
  if (a.L == 64 && a.T == 64)
    return resblk_rot() ? launch_cluster_tx<64, 64, 4, 2, 2, 1>(ctx, a, B)
                        : launch_cluster_tx<64, 64, 4, 2, 2, 1, false>(ctx, a, B);
  return -1;   // no cluster instantiation: use the streaming engine
}

// =========================================================== streaming CG
struct StreamState {
  // per chain
  double *normb, *target, *rs, *rs_new, *alpha, *beta, *best;
  int *active, *need_x, *pass;
  // per chain outputs (caller-owned)
  int* iters;
  double* relres;
  int* status;
  // global
  int* n_active;   // chains still iterating; 0 => done
  int* n_active_init;
  int* it;         // current iteration (1-based), advanced on the device
                   // so a captured chunk of iterations can be replayed
  // partials [B][tpc]
  double *part_pap, *part_rr, *part_rr2, *part_bb;
  int B, tpc, global_mode;
  double tol;
  int maxiter;
};

// Elementwise pass over the same tiles as the stencil (so partials align).
struct ElemArgs {
  const double2* __restrict__ b;
  const double2* __restrict__ x0;
  double2* __restrict__ x;
  double2* __restrict__ r;
  double2* __restrict__ p;
  const double2* __restrict__ ap;
  int L, T, TX, TT, tiles_t, tpc;
};

__device__ __forceinline__ bool tile_site(const ElemArgs& e, int tile, int k, long long& s) {
  const int tx = tile / e.tiles_t, tt = tile - (tile / e.tiles_t) * e.tiles_t;
  const int li = k / e.TT, lj = k - (k / e.TT) * e.TT;
  const int X = tx * e.TX + li, Tt = tt * e.TT + lj;
  if (X >= e.L || Tt >= e.T) return false;
  s = (long long)X * e.T + Tt;
  return true;
}

// init: x = x0|0; r = b; p = b; partial ||b||^2
__global__ void k_cg_init(ElemArgs e, StreamState st) {
  __shared__ double slot[32];
  const int c = blockIdx.x / e.tpc, tile = blockIdx.x - c * e.tpc;
  const long long cb = (long long)c * e.L * e.T;
  double acc = 0.0;
  for (int k = threadIdx.x; k < e.TX * e.TT; k += blockDim.x) {
    long long s;
    if (!tile_site(e, tile, k, s)) continue;
    Spinor bv = ld256_spinor_nc(e.b, cb + s);
    acc += spinor_norm2(bv);
    Spinor xv;
    if (e.x0) xv = ld256_spinor_nc(e.x0, cb + s);
    else xv.s0 = xv.s1 = make_double2(0, 0);
    st256_spinor(e.x, cb + s, xv);
    st256_spinor(e.r, cb + s, bv);
    st256_spinor(e.p, cb + s, bv);
  }
  double s = block_sum_rt(acc, slot);
  if (threadIdx.x == 0) st.part_bb[blockIdx.x] = s;
}

// p = r (after r = b - A x0)
__global__ void k_copy_r_to_p(ElemArgs e) {
  const int c = blockIdx.x / e.tpc, tile = blockIdx.x - c * e.tpc;
  const long long cb = (long long)c * e.L * e.T;
  for (int k = threadIdx.x; k < e.TX * e.TT; k += blockDim.x) {
    long long s;
    if (!tile_site(e, tile, k, s)) continue;
    st256_spinor(e.p, cb + s, ld256_spinor(e.r, cb + s));
  }
}

// update: p = r + beta p; x += alpha p; (non-replacement) r -= alpha ap, partial ||r||^2
// With few tiles per chain (FUSE_ALPHA) every thread forms alpha itself from
// the chain's <p,Ap> tile partials, in the same fixed order as k_ctrl_alpha.
template <bool FUSE_ALPHA>
__global__ void k_cg_update(ElemArgs e, StreamState st) {
  pdl_enter();
  __shared__ double slot[32];
  const int repl = (*st.it % kReplace) == 0;
  const int c = blockIdx.x / e.tpc, tile = blockIdx.x - c * e.tpc;
  if (!st.active[c]) return;
  double al;
  if (FUSE_ALPHA) {
    double den = 0.0;
    for (int k = 0; k < e.tpc; ++k) den += st.part_pap[(long long)c * e.tpc + k];
    al = den > 0.0 ? st.rs[c] / den : 0.0;
  } else {
    al = st.alpha[c];
  }
  const double be = st.beta[c];
  const long long cb = (long long)c * e.L * e.T;
  double acc = 0.0;
  for (int k = threadIdx.x; k < e.TX * e.TT; k += blockDim.x) {
    long long s;
    if (!tile_site(e, tile, k, s)) continue;
    Spinor rv = ld256_spinor(e.r, cb + s), pv = ld256_spinor(e.p, cb + s);
    Spinor xv = ld256_spinor(e.x, cb + s);
    pv = sp_fma(be, pv, rv);
    xv = sp_fma(al, pv, xv);
    st256_spinor(e.p, cb + s, pv);
    st256_spinor(e.x, cb + s, xv);
    if (!repl) {
      rv = sp_fma(-al, ld256_spinor_nc(e.ap, cb + s), rv);
      st256_spinor(e.r, cb + s, rv);
      acc += spinor_norm2(rv);
    }
  }
  if (!repl) {
    double s = block_sum_rt(acc, slot);
    if (threadIdx.x == 0) st.part_rr[blockIdx.x] = s;
  }
}

// Per-chain sum of tile partials in a fixed order.  Control kernels run in
// one of two layouts: one thread per chain (few tiles per chain, sequential
// sum) or one CTA per chain (many tiles, tree sum).
constexpr int kSmallTpc = 16;

template <bool PER_THREAD>
__device__ __forceinline__ int ctrl_chain() {
  return PER_THREAD ? (int)(blockIdx.x * blockDim.x + threadIdx.x) : (int)blockIdx.x;
}

template <bool PER_THREAD>
__device__ __forceinline__ bool ctrl_leader() {
  return PER_THREAD ? true : threadIdx.x == 0;
}

template <bool PER_THREAD>
__device__ __forceinline__ double sum_partials(const double* part, int tpc, int c, double* slot) {
  if (PER_THREAD) {
    double acc = 0.0;
    for (int k = 0; k < tpc; ++k) acc += part[(long long)c * tpc + k];
    return acc;
  }
  double acc = 0.0;
  for (int k = threadIdx.x; k < tpc; k += blockDim.x) acc += part[(long long)c * tpc + k];
  return block_sum_rt(acc, slot);
}

// init control: normb, target, rs, flags
template <bool PT>
__global__ void k_ctrl_init(StreamState st, int have_x0) {
  __shared__ double slot[2][32];
  const int c = ctrl_chain<PT>();
  if (c >= st.B) return;
  double nb2 = sum_partials<PT>(st.part_bb, st.tpc, c, slot[0]);
  double rr = have_x0 ? sum_partials<PT>(st.part_rr2, st.tpc, c, slot[1]) : nb2;
  if (ctrl_leader<PT>()) {
    double nb = sqrt(nb2);
    st.normb[c] = nb;
    st.target[c] = st.tol * nb;
    st.rs[c] = rr;
    st.beta[c] = 0.0;
    st.alpha[c] = 0.0;
    st.best[c] = INFINITY;
    st.iters[c] = 0;
    st.relres[c] = 0.0;
    st.status[c] = 0;
    st.need_x[c] = 0;
    st.pass[c] = 0;
    st.active[c] = st.global_mode ? 1 : (nb > 0.0 ? 1 : 0);
  }
}

// one CTA: count active chains; global mode: all-zero rhs => done (fermion.py:181)
__global__ void k_ctrl_init_global(StreamState st) {
  __shared__ int cnt;
  __shared__ int nz;
  if (threadIdx.x == 0) {
    cnt = 0;
    nz = 0;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < st.B; c += blockDim.x) {
    if (st.active[c]) atomicAdd(&cnt, 1);
    if (st.normb[c] != 0.0) atomicAdd(&nz, 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) *st.it = 1;
  if (st.global_mode && nz == 0) {
    for (int c = threadIdx.x; c < st.B; c += blockDim.x) st.active[c] = 0;
    if (threadIdx.x == 0) *st.n_active = *st.n_active_init = 0;
    return;
  }
  if (threadIdx.x == 0) *st.n_active = *st.n_active_init = cnt;
}

// after the stencil pass: alpha = <p,Ap> > 0 ? rs/<p,Ap> : 0
template <bool PT>
__global__ void k_ctrl_alpha(StreamState st) {
  pdl_enter();
  __shared__ double slot[32];
  const int c = ctrl_chain<PT>();
  if (c >= st.B || !st.active[c]) return;
  double den = sum_partials<PT>(st.part_pap, st.tpc, c, slot);
  if (ctrl_leader<PT>()) st.alpha[c] = den > 0.0 ? st.rs[c] / den : 0.0;
}

// after the update: rs' and the convergence check
template <bool PT>
__global__ void k_ctrl_check(StreamState st) {
  pdl_enter();
  __shared__ double slot[32];
  const int repl = (*st.it % kReplace) == 0;
  const int c = ctrl_chain<PT>();
  if (c >= st.B || !st.active[c]) return;
  if (repl) {
    if (ctrl_leader<PT>()) {
      st.pass[c] = 1;
      st.need_x[c] = 1;
    }
    return;
  }
  double rsn = sum_partials<PT>(st.part_rr, st.tpc, c, slot);
  if (ctrl_leader<PT>()) {
    st.rs_new[c] = rsn;
    int ok = sqrt(rsn) <= st.target[c];
    st.pass[c] = ok;
    st.need_x[c] = st.global_mode ? 0 : ok;
  }
}

// global mode: the true-residual branch runs only when every chain passes
__global__ void k_ctrl_check_global(StreamState st) {
  pdl_enter();
  const int repl = (*st.it % kReplace) == 0;
  __shared__ int fails;
  if (threadIdx.x == 0) fails = 0;
  __syncthreads();
  if (!repl)
    for (int c = threadIdx.x; c < st.B; c += blockDim.x)
      if (st.active[c] && !st.pass[c]) atomicAdd(&fails, 1);
  __syncthreads();
  const int all = fails == 0;
  for (int c = threadIdx.x; c < st.B; c += blockDim.x)
    if (st.active[c]) st.need_x[c] = repl ? 1 : all;
}

// after the (optional) true-residual pass
template <bool PT>
__global__ void k_ctrl_final(StreamState st) {
  pdl_enter();
  __shared__ double slot[32];
  const int it = *st.it;
  const int c = ctrl_chain<PT>();
  if (c >= st.B || !st.active[c]) return;
  const int nx = st.need_x[c];
  double tn2 = nx ? sum_partials<PT>(st.part_rr2, st.tpc, c, slot) : 0.0;
  if (!ctrl_leader<PT>()) return;
  double rs_new = nx ? tn2 : st.rs_new[c];
  st.rs_new[c] = rs_new;
  if (st.global_mode) return;   // decisions in k_ctrl_final_global
  if (nx) {
    const double tn = sqrt(tn2);
    const int repl = (it % kReplace) == 0;
    if (!repl || tn <= st.target[c]) st.best[c] = tn / st.normb[c];
    if (tn <= st.target[c]) {
      st.active[c] = 0;
      st.iters[c] = it;
      st.relres[c] = tn / st.normb[c];
      atomicSub(st.n_active, 1);
      return;
    }
  }
  const double rs = st.rs[c];
  st.beta[c] = rs > 0.0 ? rs_new / rs : 0.0;
  st.rs[c] = rs_new;
  st.need_x[c] = 0;
  if (it >= st.maxiter) {
    st.active[c] = 0;
    st.iters[c] = it;
    st.status[c] = 1;
    st.relres[c] = fmin(st.best[c], sqrt(rs_new) / st.normb[c]);
    atomicSub(st.n_active, 1);
  }
}

__global__ void k_ctrl_final_global(StreamState st) {
  pdl_enter();
  const int it = *st.it;
  __shared__ int fails, any_x;
  __shared__ double worst;
  if (threadIdx.x == 0) {
    fails = 0;
    any_x = 0;
    worst = 0.0;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < st.B; c += blockDim.x) {
    if (!st.active[c]) continue;
    if (st.need_x[c]) {
      atomicOr(&any_x, 1);
      if (!(sqrt(st.rs_new[c]) <= st.target[c])) atomicAdd(&fails, 1);
    }
  }
  __syncthreads();
  // worst relative true residual of this check (fermion.py:207), fixed order
  if (any_x && threadIdx.x == 0) {
    double w = 0.0;
    for (int c = 0; c < st.B; ++c)
      if (st.active[c] && st.normb[c] > 0) w = fmax(w, sqrt(st.rs_new[c]) / st.normb[c]);
    worst = w;
  }
  __syncthreads();
  const bool converged = any_x && fails == 0;
  for (int c = threadIdx.x; c < st.B; c += blockDim.x) {
    if (!st.active[c]) continue;
    if (any_x && (!((it % kReplace) == 0) || converged)) st.best[c] = worst;
    if (converged) {
      st.active[c] = 0;
      st.iters[c] = it;
      st.relres[c] = st.normb[c] > 0 ? sqrt(st.rs_new[c]) / st.normb[c] : 0.0;
      continue;
    }
    const double rs = st.rs[c], rsn = st.rs_new[c];
    st.beta[c] = rs > 0.0 ? rsn / rs : 0.0;
    st.rs[c] = rsn;
    st.need_x[c] = 0;
    if (it >= st.maxiter) {
      st.active[c] = 0;
      st.iters[c] = it;
      st.status[c] = 1;
      st.relres[c] = fmin(st.best[c], sqrt(rsn) / (st.normb[c] > 0 ? st.normb[c] : 1.0));
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && (converged || it >= st.maxiter)) *st.n_active = 0;
}

__global__ void k_iter_inc(StreamState st) {
  pdl_enter();
  if (threadIdx.x == 0) ++*st.it;
}

// Body tail of the device-side CG loop: keep iterating while a chain is
// active (the WHILE node of the conditional graph re-evaluates this).
__global__ void k_set_continue(StreamState st, cudaGraphConditionalHandle h) {
  pdl_enter();
  if (threadIdx.x == 0)
    cudaGraphSetConditional(h, (*st.n_active > 0 && *st.it <= st.maxiter + 1) ? 1u : 0u);
}

// Chains whose rhs is exactly zero return x = 0 (fermion.py:181-182): per
// chain in per-chain mode, and for the whole batch in global mode when every
// rhs is zero.
__global__ void k_zero_x_if_null(ElemArgs e, StreamState st) {
  const int c = blockIdx.x / e.tpc, tile = blockIdx.x - c * e.tpc;
  if (st.normb[c] != 0.0) return;
  if (st.global_mode && *st.n_active_init != 0) return;
  const long long cb = (long long)c * e.L * e.T;
  for (int k = threadIdx.x; k < e.TX * e.TT; k += blockDim.x) {
    long long s;
    if (!tile_site(e, tile, k, s)) continue;
    Spinor z;
    z.s0 = z.s1 = make_double2(0, 0);
    st_spinor(e.x, cb + s, z);
  }
}

int cg_streaming(sch_ctx* ctx, const double2* U, const double2* b, double2* x, const double2* x0,
                 int B, int L, int T, double m0, double tol, int maxiter, int global_mode, int* iters,
                 double* relres, int* status) {
  const TileShape sh = pick_tile(L, T);
  const int tpc = sh.tiles_x * sh.tiles_t;
  const long long V = (long long)L * T;
  const size_t nvec = (size_t)B * V * 2;   // double2 per vector
  size_t bytes = 3 * nvec * sizeof(double2) + 7 * (size_t)B * sizeof(double) +
                 3 * (size_t)B * sizeof(int) + 4 * (size_t)B * tpc * sizeof(double) + 64 * 256;
  void* ws;
  int rc = sch_workspace(ctx, bytes, &ws);
  if (rc) return rc;
  char* w = (char*)ws;
  auto take = [&](size_t n) {
    char* p = w;
    w += (n + 255) & ~size_t(255);
    return (void*)p;
  };
  double2* r = (double2*)take(nvec * sizeof(double2));
  double2* p = (double2*)take(nvec * sizeof(double2));
  double2* ap = (double2*)take(nvec * sizeof(double2));
  StreamState st;
  st.normb = (double*)take(B * 8);
  st.target = (double*)take(B * 8);
  st.rs = (double*)take(B * 8);
  st.rs_new = (double*)take(B * 8);
  st.alpha = (double*)take(B * 8);
  st.beta = (double*)take(B * 8);
  st.best = (double*)take(B * 8);
  st.active = (int*)take(B * 4);
  st.need_x = (int*)take(B * 4);
  st.pass = (int*)take(B * 4);
  st.n_active = (int*)take(4);
  st.n_active_init = (int*)take(4);
  st.it = (int*)take(4);
  st.part_pap = (double*)take((size_t)B * tpc * 8);
  st.part_rr = (double*)take((size_t)B * tpc * 8);
  st.part_rr2 = (double*)take((size_t)B * tpc * 8);
  st.part_bb = (double*)take((size_t)B * tpc * 8);
  if ((size_t)(w - (char*)ws) > ctx->ws_bytes)
    return sch_fail(ctx, SCH_ERR_ARG, "cg workspace layout overflow");
  st.iters = iters;
  st.relres = relres;
  st.status = status;
  st.B = B;
  st.tpc = tpc;
  st.global_mode = global_mode;
  st.tol = tol;
  st.maxiter = maxiter;

  ElemArgs e{b, x0, x, r, p, ap, L, T, sh.TX, sh.TT, sh.tiles_t, tpc};
  TileArgs ta{};
  ta.U = U;
  ta.B = B;
  ta.L = L;
  ta.T = T;
  ta.tiles_t = sh.tiles_t;
  ta.tiles_per_chain = tpc;
  ta.diag = 2.0 + m0;
  const unsigned ngrid = (unsigned)B * tpc;
  cudaStream_t s = ctx->stream;

  k_cg_init<<<ngrid, 256, 0, s>>>(e, st);
  SCH_LAUNCHED(ctx);
  if (x0) {   // r = b - A x0 ; p = r
    TileArgs tx = ta;
    tx.in = x;
    tx.bvec = b;
    tx.out = r;
    tx.flag = nullptr;
    tx.partial = st.part_rr2;
    launch_normal_tile<MODE_X>(sh, tx, s);
    SCH_LAUNCHED(ctx);
    k_copy_r_to_p<<<ngrid, 256, 0, s>>>(e);
    SCH_LAUNCHED(ctx);
  }
  // control-kernel layout: one thread per chain when chains have few tiles
  const bool pt = tpc <= kSmallTpc;
  const unsigned cgrid = pt ? blocks_for(B, 128) : (unsigned)B;
  const int sparse = ctx->num_sms * 2;   // persistent grid of the true-residual pass
  if (pt) k_ctrl_init<true><<<cgrid, 128, 0, s>>>(st, x0 != nullptr);
  else k_ctrl_init<false><<<cgrid, 128, 0, s>>>(st, x0 != nullptr);
  SCH_LAUNCHED(ctx);
  k_ctrl_init_global<<<1, 1024, 0, s>>>(st);
  SCH_LAUNCHED(ctx);

  TileArgs tp = ta;   // stencil pass: p formed on the fly from r, p_old
  tp.in = r;
  tp.in2 = p;
  tp.out = ap;
  tp.flag = st.active;
  tp.beta = st.beta;
  tp.partial = st.part_pap;
  TileArgs txx = ta;  // true residual / replacement pass
  txx.in = x;
  txx.bvec = b;
  txx.out = r;
  txx.flag = st.need_x;
  txx.partial = st.part_rr2;

  // One CG iteration; every decision (replacement, convergence, maxiter)
  // is made on the device from st.it, so the sequence can be captured once
  // and replayed.  Returns the number of kernels enqueued.
  // Every launch but the first of a solve uses programmatic stream
  // serialization (runtime.hpp launch_k): its CTAs are scheduled while the
  // previous kernel drains and wait in pdl_enter().
  const bool pdl = use_pdl();
  auto enqueue_iteration = [&](cudaStream_t q) -> int {
    int n = 0;
    launch_normal_tile<MODE_P>(sh, tp, q, 0, pdl);
    ++n;
    if (pt) {
      launch_k(pdl, k_cg_update<true>, dim3(ngrid), dim3(256), 0, q, e, st);
      launch_k(pdl, k_ctrl_check<true>, dim3(cgrid), dim3(128), 0, q, st);
      n += 2;
    } else {
      launch_k(pdl, k_ctrl_alpha<false>, dim3(cgrid), dim3(128), 0, q, st);
      launch_k(pdl, k_cg_update<false>, dim3(ngrid), dim3(256), 0, q, e, st);
      launch_k(pdl, k_ctrl_check<false>, dim3(cgrid), dim3(128), 0, q, st);
      n += 3;
    }
    if (global_mode) {
      launch_k(pdl, k_ctrl_check_global, dim3(1), dim3(1024), 0, q, st);
      ++n;
    }
    launch_normal_tile<MODE_X>(sh, txx, q, sparse, pdl);
    ++n;
    if (pt) launch_k(pdl, k_ctrl_final<true>, dim3(cgrid), dim3(128), 0, q, st);
    else launch_k(pdl, k_ctrl_final<false>, dim3(cgrid), dim3(128), 0, q, st);
    ++n;
    if (global_mode) {
      launch_k(pdl, k_ctrl_final_global, dim3(1), dim3(1024), 0, q, st);
      ++n;
    }
    launch_k(pdl, k_iter_inc, dim3(1), dim3(32), 0, q, st);
    return n + 1;
  };
  auto poll_done = [&]() -> int {
    SCH_CUDA(ctx, cudaMemcpyAsync(ctx->h_flag, st.n_active, sizeof(int), cudaMemcpyDeviceToHost, s));
    SCH_CUDA(ctx, cudaStreamSynchronize(s));
    return *ctx->h_flag == 0 ? 1 : 0;
  };

  if (use_cg_graph() && use_cg_while()) {
    // The whole loop on the device: a conditional WHILE node whose body is
    // kBody captured iterations plus k_set_continue.  One graph launch per
    // solve, no host polling: the call returns without synchronising.
    // 4 iterations per pass of the WHILE body: the conditional node costs
    // ~3.5 us per evaluation, a converged iteration is a few no-op launches
    constexpr int kBody = 4;
    if (!ctx->cap_stream)
      SCH_CUDA(ctx, cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking));
    cudaGraph_t graph;
    SCH_CUDA(ctx, cudaGraphCreate(&graph, 0));
    cudaGraphConditionalHandle handle;
    SCH_CUDA(ctx, cudaGraphConditionalHandleCreate(&handle, graph, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = handle;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t cnode;
    SCH_CUDA(ctx, cudaGraphAddNode(&cnode, graph, nullptr, 0, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    SCH_CUDA(ctx, cudaStreamBeginCaptureToGraph(ctx->cap_stream, body, nullptr, nullptr, 0,
                                                cudaStreamCaptureModeRelaxed));
    int per = 0;
    for (int j = 0; j < kBody; ++j) per += enqueue_iteration(ctx->cap_stream);
    launch_k(pdl, k_set_continue, dim3(1), dim3(32), 0, ctx->cap_stream, st, handle);
    cudaError_t ce = cudaGetLastError();
    SCH_CUDA(ctx, cudaStreamEndCapture(ctx->cap_stream, &body));
    if (ce != cudaSuccess) {
      cudaGraphDestroy(graph);
      return sch_fail(ctx, SCH_ERR_CUDA, "cg while-capture: %s", cudaGetErrorString(ce));
    }
    cudaGraphExec_t exec;
    cudaError_t ie = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ie != cudaSuccess) return sch_fail(ctx, SCH_ERR_CUDA, "cg while-instantiate: %s", cudaGetErrorString(ie));
    cudaError_t le = cudaGraphLaunch(exec, s);
    cudaGraphExecDestroy(exec);   // released once the launch completes
    if (le != cudaSuccess) return sch_fail(ctx, SCH_ERR_CUDA, "cg graph launch: %s", cudaGetErrorString(le));
    ctx->launches += per + 1;     // per body pass; the trip count is decided on the device
  } else if (use_cg_graph()) {
    // capture kChunk iterations once on a private stream, replay on s
    constexpr int kChunk = 8;
    if (!ctx->cap_stream)
      SCH_CUDA(ctx, cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking));
    cudaGraph_t graph;
    SCH_CUDA(ctx, cudaStreamBeginCapture(ctx->cap_stream, cudaStreamCaptureModeRelaxed));
    int per = 0;
    for (int j = 0; j < kChunk; ++j) per += enqueue_iteration(ctx->cap_stream);
    cudaError_t ce = cudaGetLastError();
    SCH_CUDA(ctx, cudaStreamEndCapture(ctx->cap_stream, &graph));
    if (ce != cudaSuccess)
      return sch_fail(ctx, SCH_ERR_CUDA, "cg capture: %s", cudaGetErrorString(ce));
    cudaGraphExec_t exec;
    SCH_CUDA(ctx, cudaGraphInstantiate(&exec, graph, 0));
    cudaGraphDestroy(graph);
    const int max_chunks = maxiter / kChunk + 2;
    int rc2 = SCH_OK;
    for (int k = 0; k < max_chunks; ++k) {
      cudaError_t le = cudaGraphLaunch(exec, s);
      if (le != cudaSuccess) {
        rc2 = sch_fail(ctx, SCH_ERR_CUDA, "cg graph launch: %s", cudaGetErrorString(le));
        break;
      }
      ctx->launches += per;
      if (poll_done()) break;
    }
    cudaGraphExecDestroy(exec);
    if (rc2) return rc2;
  } else {
    int done_iters = 0, chunk = 4;
    while (done_iters < maxiter + 1) {
      for (int j = 0; j < chunk; ++j) ctx->launches += enqueue_iteration(s);
      SCH_LAUNCHED(ctx);
      done_iters += chunk;
      if (poll_done()) break;
      chunk = std::min(chunk * 2, 32);
    }
  }
  k_zero_x_if_null<<<ngrid, 256, 0, s>>>(e, st);
  SCH_LAUNCHED(ctx);
  return SCH_OK;
}

}  // namespace

extern "C" int sch_cg_normal(sch_ctx* ctx, const double* U, const double* b, double* x,
                             const double* x0, int B, int L, int T, double m0, double tol,
                             int maxiter, int stop_mode, int* iters, double* relres, int* status,
                             int* h_iters_out) {
  SCH_CHECK_ARG(ctx, U && b && x && iters && relres && status, "cg_normal: null pointer");
  SCH_CHECK_ARG(ctx, B >= 1 && L >= 2 && T >= 2 && maxiter >= 1, "cg_normal: bad geometry");
  SCH_CHECK_ARG(ctx, stop_mode == 0 || stop_mode == 1, "cg_normal: stop_mode must be 0 or 1");
  SCH_CHECK_ARG(ctx, x != b && x != x0, "cg_normal: x must not alias b or x0");
  const long long V = (long long)L * T;
  const bool per_chain = stop_mode == 1 || B == 1;
  int rc = SCH_OK;
  if (per_chain && V <= 1024) {
    ResArgs a{(const double2*)U, (const double2*)b, (const double2*)x0, (double2*)x, iters, relres,
              status, L, T, 2.0 + m0, tol, maxiter};
    rc = resident_dispatch(ctx, a, B, V);
  } else if (per_chain && (rc = cluster_dispatch(ctx, ResArgs{(const double2*)U, (const double2*)b,
                                                              (const double2*)x0, (double2*)x, iters,
                                                              relres, status, L, T, 2.0 + m0, tol,
                                                              maxiter}, B)) >= 0) {
    // cluster-resident engine ran (rc = its status)
  } else {
    rc = SCH_OK;
    rc = cg_streaming(ctx, (const double2*)U, (const double2*)b, (double2*)x, (const double2*)x0, B,
                      L, T, m0, tol, maxiter, per_chain ? 0 : 1, iters, relres, status);
  }
  if (rc) return rc;
  if (h_iters_out) {
    std::vector<int> hi(B), hs(B);
    SCH_CUDA(ctx, cudaMemcpyAsync(hi.data(), iters, sizeof(int) * B, cudaMemcpyDeviceToHost, ctx->stream));
    SCH_CUDA(ctx, cudaMemcpyAsync(hs.data(), status, sizeof(int) * B, cudaMemcpyDeviceToHost, ctx->stream));
    SCH_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    *h_iters_out = *std::max_element(hi.begin(), hi.end());
    for (int c = 0; c < B; ++c)
      if (hs[c]) return sch_fail(ctx, SCH_ERR_SOLVER, "CG exceeded %d iterations (chain %d)", maxiter, c);
  }
  return SCH_OK;
}

// chi_xi (fermion.py:300-310): xi = CG(eta), chi = D xi in one call.
// (Forming chi inside the resident solve from the registers was measured:
// the solver's loop compiles ~12 % slower with the epilogue, more than the
// 44 us D launch it saves on 8192 x 16^2 — DESIGN.md §5.)
extern "C" int sch_chi_xi(sch_ctx* ctx, const double* U, const double* eta, double* chi, double* xi,
                          const double* x0, int B, int L, int T, double m0, double tol, int maxiter,
                          int stop_mode, int* iters, double* relres, int* status) {
  SCH_CHECK_ARG(ctx, U && eta && chi && xi && iters && relres && status, "chi_xi: null pointer");
  SCH_CHECK_ARG(ctx, xi != eta && xi != x0 && chi != eta && chi != xi && chi != x0,
                "chi_xi: outputs alias inputs");
  int rc = sch_cg_normal(ctx, U, eta, xi, x0, B, L, T, m0, tol, maxiter, stop_mode, iters, relres,
                         status, nullptr);
  if (rc) return rc;
  return sch_dslash(ctx, U, 1, xi, chi, B, L, T, m0, 0);
}
