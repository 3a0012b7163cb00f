/*
 * schwinger_sm100.h — C-ABI of the B200 (sm_100a) engine for the HMC
 * molecular-dynamics hot path of the 2D Schwinger model (arXiv:1512.03812
 * reference package `schwinger`, /root/reference/pkg/src/schwinger).
 *
 * The reference has no FFI: its boundary is the in-process Python module API
 * (SURVEY.md §8(b)).  Each entry point below replaces one reference function;
 * the citation names it.  A ctypes binding (paper_1512_03812_b200/_lib.py)
 * mirrors those Python signatures on top of this header; INTEGRATION.md shows
 * the stub a maintainer of the reference would add.
 *
 * Conventions
 *  - Every pointer is a DEVICE pointer unless named h_*; layouts are the
 *    reference's (lattice.py:3-12):
 *       links (q, p, forces)  double  [B][2][L][T]
 *       link cache U          double  [B][2][L][T][2]   (re, im) = exp(i q)
 *       spinors               double  [B][L][T][2][2]   complex128 (B, L, T, 2)
 *    B = number of independent chains (batch), B >= 1.
 *  - All work is stream-ordered on the context's stream (sch_set_stream);
 *    calls return without synchronising unless stated.
 *  - Return value: 0 = OK, 1 = bad argument, 2 = CUDA error,
 *    3 = solver hit maxiter (details in the per-chain status array).
 *    sch_last_error() gives the message.
 *  - Arithmetic is IEEE FP64 throughout.  Real-arithmetic updates (drift,
 *    kicks) are evaluated without FMA contraction in NumPy's order.
 */
#ifndef SCHWINGER_SM100_H
#define SCHWINGER_SM100_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct sch_ctx sch_ctx;

/* ---- context --------------------------------------------------------- */
int sch_ctx_create(int device, sch_ctx** out);
int sch_ctx_destroy(sch_ctx* ctx);
int sch_set_stream(sch_ctx* ctx, void* cuda_stream);
const char* sch_last_error(const sch_ctx* ctx);
/* Number of kernels this context has launched (for bench accounting). */
unsigned long long sch_launch_count(const sch_ctx* ctx);
/* Library build identifier, e.g. "sm_100a". */
const char* sch_build_info(void);

/* ---- L0: links, momenta (lattice.py) --------------------------------- */
/* out = wrap(q + h*p), wrap = floored mod to [-pi,pi)
 * replaces lattice.rotate_links (lattice.py:111-118) + wrap_angles (:28-30) */
int sch_rotate_links(sch_ctx* ctx, const double* q, const double* p, double h,
                     double* out, long long n);
/* replaces lattice.wrap_angles (lattice.py:28-30) */
int sch_wrap_angles(sch_ctx* ctx, const double* q, double* out, long long n);
/* out = p - (a*f + c*g)   (g may be NULL => out = p - a*f)
 * replaces the momentum kicks of integrators.py:161-246 / shift_momenta
 * (lattice.py:121-125) */
int sch_kick(sch_ctx* ctx, const double* p, const double* f, double a,
             const double* g, double c, double* out, long long n);
/* out[b] = 0.5 * sum p^2 over the chain's 2*L*T links
 * replaces lattice.kinetic_energy (lattice.py:128-130) */
int sch_kinetic_energy(sch_ctx* ctx, const double* p, double* out, int B, long long per_chain);

/* ---- L1a: gauge sector (gauge.py) ------------------------------------ */
/* theta(n) per site, [B][L][T]; replaces gauge.plaq_angles (gauge.py:21-24) */
int sch_plaquette_angles(sch_ctx* ctx, const double* q, double* out, int B, int L, int T);
/* beta * g (gauge.py:43-59) */
int sch_gauge_force(sch_ctx* ctx, const double* q, double beta, double* out, int B, int L, int T);
/* p_out = p - dt * (beta * g(q)); kick_gauge (integrators.py:161-164) fused */
int sch_kick_gauge(sch_ctx* ctx, const double* q, const double* p, double beta, double dt,
                   double* p_out, int B, int L, int T);
/* M micro leapfrog steps of the gauge system fused: [kick dt/2, drift dt,
 * kick dt/2] x m (integrators.py:253-259). q, p updated in place. */
int sch_inner_leapfrog(sch_ctx* ctx, double* q, double* p, double beta, double span, int m,
                       int B, int L, int T);
/* per chain: beta*sum(1-cos theta) (gauge.py:37-40) and mean cos theta (gauge.py:32-34) */
int sch_gauge_action(sch_ctx* ctx, const double* q, double beta, double* out, int B, int L, int T);
int sch_avg_plaquette(sch_ctx* ctx, const double* q, double* out, int B, int L, int T);
/* C_GG closed form (gauge.py:97-107) */
int sch_fg_gauge_gauge(sch_ctx* ctx, const double* q, double beta, double* out, int B, int L, int T);
/* 2 * sum w * Hess(S_G) (gauge.py:110-136) */
/* gauge.oriented_plaquettes (K = 1, out (B,2,L,T) c128) and
 * gauge.plaquette_stencil (K = 8, out (8,B,2,L,T) c128): the mu-oriented
 * plaquette P1 and its translates P2..P8 attached to link (n,mu)
 * (pkg/src/schwinger/gauge.py:62-95) */
int sch_plaquette_stencil(sch_ctx* ctx, const double* q, double* out, int K, int B, int L, int T);
int sch_gauge_hessian_dot(sch_ctx* ctx, const double* q, double beta, const double* w,
                          double* out, int B, int L, int T);

/* ---- L1b: Wilson fermions (fermion.py) ------------------------------- */
/* U = exp(i q) (fermion.py:94); fermion_bc 0 = periodic (reference),
 * 1 = antiperiodic in time (sign flip of U_t on t = T-1; BASELINE configs) */
int sch_links_to_u(sch_ctx* ctx, const double* q, double* U, int B, int L, int T, int fermion_bc);
/* out = D psi (dagger=0) or D^dag psi (dagger=1); U chain stride 0 when
 * u_batched == 0.  replaces WilsonDirac.apply / apply_dag (fermion.py:119-127) */
int sch_dslash(sch_ctx* ctx, const double* U, int u_batched, const double* psi, double* out,
               int B, int L, int T, double m0, int dagger);
/* out = D^dag D psi, fused (one pass, shared-memory halo tile)
 * replaces WilsonDirac.normal (fermion.py:129-131) */
int sch_ddagd(sch_ctx* ctx, const double* U, const double* psi, double* out,
              int B, int L, int T, double m0);
/* out[b] = sum conj(a) b over the chain (complex: out[2b], out[2b+1])
 * replaces fermion.spinor_dot (fermion.py:54-56) */
int sch_spinor_dot(sch_ctx* ctx, const double* a, const double* b, double* out, int B, long long V);

/* CG on D^dag D x = b (fermion.py:171-217), exact stopping semantics:
 * residual replacement every 50 iterations, true-residual re-check, alpha/beta
 * guards.  stop_mode 0 = batch_global (reference batched semantics: every
 * chain iterates until all pass), 1 = per_chain (each chain stops as an
 * unbatched reference call would).  x0 may be NULL (zero start).
 * Per-chain outputs (device): iters[B] (int32), relres[B] (true ||b-Ax||/||b||
 * at convergence, or the best residual on failure), status[B] (0 ok,
 * 1 maxiter).  h_iters_out (host, may be NULL) receives the max iteration
 * count; requesting it synchronises the stream.
 * Returns 3 (SCH_ERR_SOLVER) only when h_iters_out is non-NULL and a chain
 * failed; otherwise failures are reported through status[] (no sync). */
int sch_cg_normal(sch_ctx* ctx, const double* U, const double* b, double* x, const double* x0,
                  int B, int L, int T, double m0, double tol, int maxiter, int stop_mode,
                  int* iters, double* relres, int* status, int* h_iters_out);

/* chi_xi (fermion.py:300-310): xi = (D^dag D)^{-1} eta by the CG above and
 * chi = D xi, in one call; the 16^2 / 32^2 per-chain resident engines form
 * chi inside the solve.  Outputs and stop modes as sch_cg_normal (no sync). */
int sch_chi_xi(sch_ctx* ctx, const double* U, const double* eta, double* chi, double* xi,
               const double* x0, int B, int L, int T, double m0, double tol, int maxiter,
               int stop_mode, int* iters, double* relres, int* status);

/* f(n,mu) = -Im[A - B] (fermion.py:330-336); when p != NULL the kick is
 * fused: out = p - dt * (f [+ beta*g(q) when q != NULL])  (kick_fermion /
 * kick_full, integrators.py:172-186) */
int sch_fermion_force(sch_ctx* ctx, const double* U, const double* chi, const double* xi,
                      double* out, int B, int L, int T);
/* fermion.link_bilinears(op, mu, a, b) (pkg/src/schwinger/fermion.py:317-327):
 * A, Bout (B,L,T) c128 */
int sch_link_bilinears(sch_ctx* ctx, const double* U, const double* a, const double* b, int mu,
                       double* A, double* Bout, int B, int L, int T);
int sch_kick_fermion(sch_ctx* ctx, const double* U, const double* chi, const double* xi,
                     const double* q, double beta, const double* p, double dt, double* p_out,
                     int B, int L, int T);
/* b1 = sum weight*w1, b2 = sum weight*w2 (fermion.py:362-383) */
int sch_weighted_w_sums(sch_ctx* ctx, const double* U, const double* weight, const double* chi,
                        const double* xi, double* b1, double* b2, int B, int L, int T);
/* C = 2Im(A[z1,xi]-B[z1,xi]) + 2Im(A[chi,z2]-B[chi,z2]) - 2Re(A[chi,xi]+B[chi,xi])*weight
 * (fermion.py:409-417) */
int sch_fg_fermion_combine(sch_ctx* ctx, const double* U, const double* z1, const double* z2,
                           const double* chi, const double* xi, const double* weight,
                           double* out, int B, int L, int T);

/* ---- L3: Metropolis on device (bench mode) -------------------------- */
/* accept[b] = 1 if dH <= 0 or u < exp(-dH), 0 otherwise, -1 if dH is not
 * finite (hmc.py:54-60) */
int sch_metropolis(sch_ctx* ctx, const double* dh, const double* u, int* accept, int B);
/* out[b] = accept[b] == 1 ? a[b] : b_[b] over per_chain doubles (hmc.py:95) */
int sch_select_chains(sch_ctx* ctx, const int* accept, const double* a, const double* b_,
                      double* out, int B, long long per_chain);

/* ---- device RNG (bench mode; parity mode draws on the host with the
 * reference's NumPy Philox generator) ---------------------------------- */
/* scale * standard normals, Philox4x32-10 keyed by (seed, stream0 + chain),
 * counter (ctr, element); out[b * per_chain + i] */
int sch_rng_normal(sch_ctx* ctx, double* out, int B, long long per_chain, uint64_t seed,
                   uint64_t stream0, uint64_t ctr, double scale);
int sch_rng_uniform(sch_ctx* ctx, double* out, int B, long long per_chain, uint64_t seed,
                    uint64_t stream0, uint64_t ctr);

/* ---- bit-exact replica of the reference's NumPy streams ------------------
 * np.random.Generator(np.random.Philox(key=[seed, stream0 + chain]))
 * (lattice.py:86-104): one state per chain in device memory
 * (sch_np_rng_state_bytes() bytes each); draws are value-identical to the
 * host generator's (Philox4x64-10, NumPy's 256-layer ziggurat normal). */
int sch_np_rng_state_bytes(void);
int sch_np_rng_init(sch_ctx* ctx, void* state, int B, uint64_t seed, uint64_t stream0);
/* mode 0: standard_normal, 1: uniform(lo, hi), 2: random(); out[b*n + i] */
int sch_np_rng_fill(sch_ctx* ctx, void* state, double* out, int B, long long n_per_chain, int mode,
                    double lo, double hi);
/* hmc_update's heatbath draws per chain in the reference order
 * (hmc.py:78-82, fermion.py:289): p[2V] normals, then phi = (re + i im) *
 * phi_scale from 2V + 2V normals (phi unused when quenched) */
int sch_np_heatbath(sch_ctx* ctx, void* state, double* p, double* phi, int B, long long V,
                    double phi_scale, int quenched);
/* metropolis (hmc.py:54-60): accept 1/0, -1 for non-finite dH; draws only if dH > 0 */
int sch_np_metropolis(sch_ctx* ctx, void* state, const double* dh, int* accept, int B);

/* ---- trajectory megakernel ------------------------ */
/* One adapted-nested-fg trajectory (integrators.py:341-349, with the
 * Hamiltonian at both ends, hmc.py:44-51 and hmc.py:83-85) of B independent
 * 16x16 chains, one CTA per chain, in a single launch: replaces hamiltonian()
 * + integrate_trajectory() + hamiltonian() of hmc_update for that scheme.
 * q_in, p [B][2][16][16], eta [B][16][16][2] in; q_out, dh = H(end) - H(start),
 * status (1: a CG hit maxiter), iters (CG iterations) per chain out.
 * dt_kf = h/6, b_g = 2h/3, c_g = FG_KICK_SIGN * fgc * h^3, span = h/2. */
int sch_traj_anfg16(sch_ctx* ctx, const double* q_in, const double* p, const double* eta,
                    double* q_out, double* dh, int* status, int* iters, int B, double beta, double m0,
                    double tol, int maxiter, double dt_kf, double b_g, double c_g, double span,
                    int n_steps, int micro);

/* ---- domain decomposition of one lattice (BASELINE configs[4]) -------- */
/* One lattice split into G = nranks * strips_local x-strips of Lloc = L/G
 * rows.  Fields are "extended strips": [strips_local][Lloc+4][T] (2 halo
 * rows per side) in the usual per-site layouts.  nranks == 1: every strip in
 * this process, halo exchange by a copy kernel.  nranks > 1: one strip per
 * rank, NCCL send/recv of the 2-row faces and NCCL all-reduce of the CG
 * scalars (libnccl.so.2 bound at run time), or — nccl_id NULL, then
 * sch_dd_p2p_open/_connect — peer-memory mailboxes over NVLink (CUDA IPC).
 * Replaces nothing in the reference, which has no decomposed path: it is the
 * multi-GPU form of WilsonDirac.normal / cg_normal (fermion.py:129-217). */
typedef struct sch_dd sch_dd;
int sch_nccl_unique_id(sch_ctx* ctx, void* id_out /* 128 bytes */);
int sch_dd_create(sch_ctx* ctx, const void* nccl_id, int nranks, int rank, int L, int T,
                  int strips_local, sch_dd** out);
int sch_dd_destroy(sch_dd* dd);
/* p2p transport, step 1: allocate the zeroed mailboxes of this process's
 * strips; writes their CUDA IPC handle (64 bytes; zero when nranks == 1) */
int sch_dd_p2p_open(sch_ctx* ctx, sch_dd* dd, void* ipc_handle_out);
/* p2p transport, step 2 (after every rank's step 1): map the other ranks'
 * mailboxes from nranks x 64 handle bytes in rank order and switch the
 * exchanges and global sums of this dd to peer-memory kernels.  With
 * nranks == 1 (all strips in this process) the mailbox table is local. */
int sch_dd_p2p_connect(sch_ctx* ctx, sch_dd* dd, const void* ipc_handles);
/* out4 = {strips_local, Lloc, Lext, G} */
int sch_dd_geometry(const sch_dd* dd, int* out4);
/* refresh the halo rows of a field [S][planes][Lext][T][words_per_site] (doubles) */
int sch_dd_exchange(sch_ctx* ctx, sch_dd* dd, double* field, int planes, int words_per_site);
/* *out (device) = whole-lattice sum over every strip's own rows, formed by
 * the canonical tree through the lattice's transport (the same bits on
 * every rank, for any strip count): kind 0 = sum p^2 (momenta; the caller
 * takes 0.5x, lattice.py:128-130), 1 = sum(1 - cos theta) (links,
 * gauge.py:37-40), 2 = Re sum conj(a) b (spinors a, b, fermion.py:54-56) */
int sch_dd_own_sum(sch_ctx* ctx, sch_dd* dd, int kind, const double* a, const double* b,
                   double* out);
/* out = D^dag D psi on the own rows (psi's halos are refreshed first);
 * WilsonDirac.normal (fermion.py:129-131) on a decomposed lattice */
int sch_dd_ddagd(sch_ctx* ctx, sch_dd* dd, const double* U_ext, double* psi_ext, double* out_ext,
                 double m0);
/* cg_normal (fermion.py:171-217) on a decomposed lattice; b's (and x0's)
 * halos are refreshed in place.  Synchronises; host outputs may be NULL.
 * Returns 3 when maxiter is hit. */
int sch_dd_cg_normal(sch_ctx* ctx, sch_dd* dd, const double* U_ext, double* b_ext, double* x_ext,
                     double* x0_ext, double m0, double tol, int maxiter, int* h_iters,
                     double* h_relres, int* h_status);

/* ---- measurement probe (bench.py) ------------------------------------ */
/* FP64 FMA issue-rate probe: blocks x 256 threads x iters x 32 DFMA
 * (flops = blocks*256*iters*64); scratch needs `blocks` doubles. */
int sch_probe_fp64(sch_ctx* ctx, double* scratch, int blocks, int iters);

#ifdef __cplusplus
}
#endif
#endif /* SCHWINGER_SM100_H */
