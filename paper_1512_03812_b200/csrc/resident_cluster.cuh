// Cluster-resident per-chain CG for lattices too large for one CTA's
// registers (cfg4: 64^2 chains, 4096 sites = 786 KB of CG state).
//
// One thread-block cluster of CS CTAs owns one chain for the whole solve.
// CTA `rank` owns the x-rows [rank*R, (rank+1)*R), R = L/CS, every t; each
// thread a BX x BT block of sites, with the block-owned exchange of
// resident_col.cuh: faces are exported to shared memory, hops between a
// thread's own sites stay in registers.  The x-faces of a CTA's first and
// last row go to the neighbouring CTAs' shared memory (DSMEM), so the
// exchange never touches L2/HBM; the global sums are published into every
// CTA of the cluster and summed there in lane order (identical in every
// thread of the cluster, so all CTAs take the same branch at every stopping
// test).  Stopping rule, residual replacement and true-residual check are
// those of the reference cg_normal (fermion.py:171-217), as in resident.cuh.
//
// ROT = true (the dispatch default, cg.cu resblk_rot) runs the solve in the
// sigma1-diagonal spin basis of block_stencil.cuh (SiteBlockRot): b' = T b
// in, x = T x' / 2 out, u0 prescaled by -1; 64^2 67.1 -> 62.2 ns per
// chain-iteration.  (A variant synchronising with cluster-wide barriers
// measured 78.5 ns, 8-CTA clusters 67.8: removed.)
#pragma once

#include <cooperative_groups.h>

#include "block_stencil.cuh"
#include "tma_tile.cuh"

// Phase stamps of the iteration for tools/micro/cluster_phases.cu (clock
// reads by thread 0 of the cluster's first CTA); nothing in the library build.
#ifndef RES_STAMP
#define RES_STAMP(i)
#define RES_STAMP_BEGIN()
#define RES_STAMP_END(iters)
#endif

SCH_DEV void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory"); }
SCH_DEV void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory"); }
SCH_DEV void cluster_barrier() {
  cluster_arrive();
  cluster_wait();
}

// ---------------------------------------------------------------------------
// k_cg_cluster_tx: no cluster-wide barrier inside the loop.
//
// The neighbouring CTAs' x-faces and every CTA's reduction partials are
// PUSHED into the consumer's shared memory with st.async, each store
// completing bytes on an mbarrier of the receiving CTA
// (mbarrier::complete_tx); a consumer waits only on its own mbarrier for the
// bytes it needs, so no CTA ever waits for the whole cluster and no release
// fence drains the memory system.  Faces are double-buffered by use parity;
// a producer can be at most one use ahead of a consumer (each stage needs
// the consumer's partial sums of the previous one), so two buffers suffice.
// Intra-CTA planes use __syncthreads as in k_cg_resblk.
SCH_DEV uint32_t mapa_addr(uint32_t local_smem, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local_smem), "r"(rank));
  return r;
}
SCH_DEV void st_async_v2f64(uint32_t addr, double2 v, uint32_t mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];"
               ::"r"(addr), "d"(v.x), "d"(v.y), "r"(mbar)
               : "memory");
}
SCH_DEV void st_async_f64(uint32_t addr, double v, uint32_t mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];"
               ::"r"(addr), "d"(v), "r"(mbar)
               : "memory");
}
SCH_DEV void mbar_wait_cluster(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAITC_%=;\n}" ::"r"(bar),
      "r"(parity)
      : "memory");
}

template <int LC, int TC, int CS, int BX, int BT, int MINB, bool ROT = false>
__global__ void __cluster_dims__(CS, 1, 1) __launch_bounds__(LC * TC / (CS * BX * BT), MINB)
    k_cg_cluster_tx(ResArgs a) {
  namespace cgx = cooperative_groups;
  constexpr int R = LC / CS;
  constexpr int SPT = BX * BT;
  constexpr int NT = R * TC / SPT;
  constexpr int NBT = TC / BT, NBX = R / BX;
  constexpr int V = LC * TC;
  constexpr int NW = NT / 32;
  constexpr int NP = CS * NW;
  constexpr int PL = (2 * BT + 2 * BX) * NT;
  constexpr int FACE = BT * NBT;                      // double2 per pushed x-face
  constexpr uint32_t FACE_TX = 2u * FACE * 16u;       // both neighbours' faces
  constexpr uint32_t RED_TX = NP * 8u;
  static_assert(LC % CS == 0 && R % BX == 0 && TC % BT == 0 && NT % 32 == 0, "block shape");
  static_assert(NP <= 32 && NBX >= 2 && BX >= 2 && BT >= 2, "shape");
  constexpr int O0 = 0, O1 = BT * NT, O2 = 2 * BT * NT, O3 = (2 * BT + BX) * NT;
  extern __shared__ double2 sm[];
  double2* E0 = sm;                       // [2 stages][PL] local planes
  double2* RXp = sm + 2 * PL;             // [2 stages][2 par][FACE] from rank+1
  double2* RXm = RXp + 4 * FACE;          // [2 stages][2 par][FACE] from rank-1
  __shared__ double red[3][2][NP];
  __shared__ __align__(8) uint64_t mbx[2][2], mbr[3][2];
  const int rank = (int)cgx::this_cluster().block_rank();
  const int tid = threadIdx.x;
  const int c = blockIdx.x / CS;
  const long long cb = (long long)c * V;
  const int bx = tid / NBT, bt = tid % NBT;
  auto site = [&](int k) { return (rank * R + bx * BX + k / BT) * TC + bt * BT + k % BT; };
  const int ttp = bx * NBT + (bt + 1) % NBT;
  const int ttm = bx * NBT + (bt + NBT - 1) % NBT;
  const int rnext = (rank + 1) % CS, rprev = (rank + CS - 1) % CS;
  // remote targets of this thread's face pushes (edge block rows only), for
  // buffer (stage s, parity q) at +(2s+q)*FACE*16 B / +(2s+q)*8 B
  const uint32_t pushP = mapa_addr(smem_u32(RXp + bt), rprev);   // my first row -> rank-1
  const uint32_t pushM = mapa_addr(smem_u32(RXm + bt), rnext);   // my last row -> rank+1
  const uint32_t barP = mapa_addr(smem_u32(&mbx[0][0]), rprev);
  const uint32_t barM = mapa_addr(smem_u32(&mbx[0][0]), rnext);

  if (tid == 0) {
    for (int s = 0; s < 2; ++s)
      for (int q = 0; q < 2; ++q) mbar_init(&mbx[s][q], 1);
    for (int j = 0; j < 3; ++j)
      for (int q = 0; q < 2; ++q) mbar_init(&mbr[j][q], 1);
    fence_mbar_init();
    for (int s = 0; s < 2; ++s)
      for (int q = 0; q < 2; ++q) mbar_arrive_expect_tx(&mbx[s][q], FACE_TX);
    for (int j = 0; j < 3; ++j)
      for (int q = 0; q < 2; ++q) mbar_arrive_expect_tx(&mbr[j][q], RED_TX);
  }
  cluster_barrier();   // every CTA's barriers exist before anyone pushes

  // uses of each face stage / reduction slot so far (identical in every
  // thread of the cluster): buffer = use & 1, mbarrier phase parity = (use >> 1) & 1
  int ufx[2] = {0, 0}, ured[3] = {0, 0, 0};

  auto publish = [&](double v, int j) {
    v = warp_sum(v);
    const int q = ured[j] & 1;
    if ((tid & 31) == 0) {
      const uint32_t slot = smem_u32(&red[j][q][rank * NW + (tid >> 5)]);
      const uint32_t bar = smem_u32(&mbr[j][q]);
#pragma unroll
      for (int r = 0; r < CS; ++r) st_async_f64(mapa_addr(slot, r), v, mapa_addr(bar, r));
    }
  };
  auto total = [&](int j) {
    const int q = ured[j] & 1;
    const uint32_t par = (ured[j] >> 1) & 1;
    mbar_wait_cluster(smem_u32(&mbr[j][q]), par);
    if (tid == 0) mbar_arrive_expect_tx(&mbr[j][q], RED_TX);   // arm this buffer's next use
    const int l = tid & 31;
    const double v = warp_sum(l < NP ? red[j][q][l] : 0.0);
    ++ured[j];
    return v;
  };

  double2 u0[SPT], u1[SPT];
  Spinor x[SPT], r[SPT], p[SPT];
  double bb = 0.0;
#pragma unroll
  for (int k = 0; k < SPT; ++k) {
    u0[k] = cscale(ROT ? -1.0 : -0.5, __ldg(a.U + 2 * cb + site(k)));   // exact: power-of-two scale
    u1[k] = cscale(-0.5, __ldg(a.U + 2 * cb + V + site(k)));
    r[k] = rot_in<ROT>(ldg_spinor(a.b, cb + site(k)));
    x[k].s0 = x[k].s1 = make_double2(0, 0);
    bb += spinor_norm2(r[k]);
  }
  publish(bb, 2);
  const double normb2 = total(2);
  const double normb = sqrt(normb2);
  const double target = a.tol * normb;
  if (normb == 0.0) {
#pragma unroll
    for (int k = 0; k < SPT; ++k) st_spinor(a.x, cb + site(k), rot_out<ROT>(x[k]));
    if (tid == 0 && rank == 0) {
      a.iters[c] = 0;
      a.relres[c] = 0.0;
      a.status[c] = 0;
    }
    cluster_barrier();
    return;
  }
  const double t2 = target * target;
  const double t2lo = t2 * (1.0 - 4e-15), t2hi = t2 * (1.0 + 4e-15);

  using Blk = std::conditional_t<ROT, SiteBlockRot<BX, BT>, SiteBlock<BX, BT>>;   // ROT: block_stencil.cuh
  // produce stage s: local planes, and the CTA's edge rows pushed to the
  // neighbouring CTAs' receive buffers
  auto produce = [&](auto dag, int s, const Spinor* v) {
    double2* E = E0 + s * PL;
    const int q = ufx[s] & 1;
    Blk::template produce<decltype(dag)::value>(u0, u1, v, [&](int plane, int idx, double2 val) {
      if (plane == 0 && bx == 0)   // read by rank-1's last block row as its forward-x hop
        st_async_v2f64(pushP + 16u * ((s * 2 + q) * FACE + idx * NBT), val, barP + 8u * (s * 2 + q));
      else if (plane == 1 && bx == NBX - 1)   // read by rank+1's first block row (backward-x)
        st_async_v2f64(pushM + 16u * ((s * 2 + q) * FACE + idx * NBT), val, barM + 8u * (s * 2 + q));
      else {
        constexpr int off[4] = {O0, O1, O2, O3};
        E[off[plane] + idx * NT + tid] = val;
      }
    });
  };
  auto interior = [&](auto dag, const Spinor* v, Spinor* out) {
    Blk::template interior<decltype(dag)::value>(u0, u1, v, out, a.diag);
  };
  auto faces = [&](auto dag, int s, Spinor* out) {
    constexpr bool DAG = decltype(dag)::value;
    const double2* E = E0 + s * PL;
    const int q = ufx[s] & 1;
    if (bx == 0 || bx == NBX - 1) {   // whole warps (NBT = 32 threads per block row)
      mbar_wait_cluster(smem_u32(&mbx[s][q]), (ufx[s] >> 1) & 1);
      if (tid == 0) mbar_arrive_expect_tx(&mbx[s][q], FACE_TX);
    }
    double2 fx[SPT], ft[SPT];
#pragma unroll
    for (int k = 0; k < SPT; ++k) {
      const int i = k / BT, j = k % BT;
      if (i == BX - 1) fx[k] = bx == NBX - 1 ? RXp[(s * 2 + q) * FACE + j * NBT + bt] : E[O0 + j * NT + tid + NBT];
      if (i == 0) fx[k] = bx == 0 ? RXm[(s * 2 + q) * FACE + j * NBT + bt] : E[O1 + j * NT + tid - NBT];
      if (j == BT - 1) ft[k] = E[O2 + i * NT + ttp];
      if (j == 0) ft[k] = E[O3 + i * NT + ttm];
    }
    Blk::template faces<DAG>(u0, u1, fx, ft, out);
    ++ufx[s];
  };
  using F = std::integral_constant<bool, false>;
  using T = std::integral_constant<bool, true>;

  // out = D^dag D v; `dd` (if given) receives this thread's ||D v||^2 partial
  auto apply = [&](const Spinor* v, Spinor* out, double* dd) {
    Spinor t[SPT];
    produce(F{}, 0, v);
    __syncthreads();
    interior(F{}, v, t);
    faces(F{}, 0, t);
    if (dd) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < SPT; ++k) s += spinor_norm2(t[k]);
      *dd = s;
    }
    produce(T{}, 1, t);
    __syncthreads();
    interior(T{}, t, out);
    faces(T{}, 1, out);
  };

  Spinor w[SPT];
  double rs = normb2;
  if (a.x0) {
#pragma unroll
    for (int k = 0; k < SPT; ++k) x[k] = rot_in<ROT>(ldg_spinor(a.x0, cb + site(k)));
    apply(x, w, nullptr);
    double rr = 0.0;
#pragma unroll
    for (int k = 0; k < SPT; ++k) {
      r[k] = sp_sub(r[k], w[k]);
      rr += spinor_norm2(r[k]);
    }
    publish(rr, 1);
    rs = total(1);
  }
#pragma unroll
  for (int k = 0; k < SPT; ++k) p[k] = r[k];

  double best = INFINITY;
  double inv_rs = __drcp_rn(rs);
  int it = 1;
  int status = 1;
  double relres = 0.0;
  RES_STAMP_BEGIN();
  for (; it <= a.maxiter; ++it) {
    RES_STAMP(0);
    double dd;
    {
      Spinor t[SPT];
      produce(F{}, 0, p);
      RES_STAMP(1);
      __syncthreads();
      interior(F{}, p, t);
      RES_STAMP(2);
      faces(F{}, 0, t);
      RES_STAMP(3);
      dd = 0.0;
#pragma unroll
      for (int k = 0; k < SPT; ++k) dd += spinor_norm2(t[k]);
      produce(T{}, 1, t);
      publish(dd, 0);
      RES_STAMP(4);
      __syncthreads();
      interior(T{}, t, w);
      RES_STAMP(5);
      faces(T{}, 1, w);
      RES_STAMP(6);
    }
    const double den = total(0);
    RES_STAMP(7);
    const double alpha = den > 0.0 ? rs / den : 0.0;
    const bool repl = (it % kResReplace) == 0;
    double rsn = 0.0;
#pragma unroll
    for (int k = 0; k < SPT; ++k) {
      if (!repl) {
        r[k] = sp_fma(-alpha, w[k], r[k]);
        rsn += spinor_norm2(r[k]);
      }
    }
    double rs_new = 0.0;
    bool check = true;
    if (!repl) {
      publish(rsn, 1);
#pragma unroll
      for (int k = 0; k < SPT; ++k) x[k] = sp_fma(alpha, p[k], x[k]);
      RES_STAMP(8);
      rs_new = total(1);
      RES_STAMP(9);
      check = rs_new <= t2lo;
      if (!check && rs_new <= t2hi) {
        double sq;
        asm volatile("sqrt.rn.f64 %0, %1;" : "=d"(sq) : "d"(rs_new));
        check = sq <= target;
      }
    } else {
#pragma unroll
      for (int k = 0; k < SPT; ++k) x[k] = sp_fma(alpha, p[k], x[k]);
    }
    if (check) {
      apply(x, w, nullptr);
      double tn2 = 0.0;
#pragma unroll
      for (int k = 0; k < SPT; ++k) {
        w[k] = sp_sub(rot_in<ROT>(ldg_spinor(a.b, cb + site(k))), w[k]);
        tn2 += spinor_norm2(w[k]);
      }
      publish(tn2, 2);
      tn2 = total(2);
      const double tn = sqrt(tn2);
      if (!repl || tn <= target) best = tn / normb;
      if (tn <= target) {
        status = 0;
        relres = tn / normb;
        break;
      }
#pragma unroll
      for (int k = 0; k < SPT; ++k) r[k] = w[k];
      rs_new = tn2;
    }
    double beta = 0.0;
    if (rs > 0.0) {
      const double q0 = rs_new * inv_rs;
      beta = __fma_rn(__fma_rn(-rs, q0, rs_new), inv_rs, q0);
    }
#pragma unroll
    for (int k = 0; k < SPT; ++k) p[k] = sp_fma(beta, p[k], r[k]);
    rs = rs_new;
    inv_rs = __drcp_rn(rs);
    RES_STAMP(10);
  }
  RES_STAMP_END(a.maxiter);
#pragma unroll
  for (int k = 0; k < SPT; ++k) st_spinor(a.x, cb + site(k), rot_out<ROT>(x[k]));
  if (tid == 0 && rank == 0) {
    a.iters[c] = status == 0 ? it : a.maxiter;
    a.relres[c] = status == 0 ? relres : fmin(best, sqrt(rs) / normb);
    a.status[c] = status;
  }
  cluster_barrier();   // every push addressed to this CTA has landed and been consumed
}
