// Domain decomposition of ONE lattice into x-strips (BASELINE configs[4],
// SURVEY §8(e) mode 2): halo exchange inside every D^dag D application and
// global reductions inside every CG iteration.
//
// Layout: each strip holds its Lloc own rows plus H = 2 halo rows on each
// side (the fused D^dag D reaches two sites), as an "extended strip" of
// Lext = Lloc + 4 rows x T:
//     rows 0,1            <- rows Lloc, Lloc+1 of the left neighbour strip
//     rows 2 .. Lloc+1    own rows (global rows x0 .. x0+Lloc-1)
//     rows Lloc+2, Lloc+3 <- rows 2, 3 of the right neighbour strip
// so an x-face is a contiguous run of T sites and the exchange is zero-copy.
// The stencil kernels run unchanged on the extended strip; rows outside the
// own range are masked out of outputs and reductions.
//
// Transports:
//   local : all S strips live in this process as a batch [S][Lext][T]; the
//           exchange is one copy kernel, reductions are plain sums (this is
//           how the path is exercised on one GPU);
//   nccl  : one strip per rank; ncclSend/ncclRecv of the 2-row faces with
//           the +-x neighbours (grouped), ncclAllReduce of the CG scalars.
//           libnccl.so.2 is bound at run time (dlopen), so the library still
//           loads on machines without NCCL.
//   p2p   : peer memory over NVLink, no NCCL on the data path.  Every strip
//           has a mailbox in its owner's HBM (face slots, arrival / ack
//           counters, reduction slots and flags); the mailboxes of the other
//           ranks are mapped with CUDA IPC (sch_dd_p2p_open / _connect).  A
//           face exchange is a push kernel that stores the strip's two edge
//           rows straight into the neighbours' mailboxes (NVLink stores) and
//           bumps their arrival counters with a system-scope release, and a
//           pull kernel that waits on its own counters and copies the slots
//           into the halo rows, then acknowledges to the producer (credit for
//           slot reuse, two slots per side).  A global sum is one kernel that
//           reduces the strip's partials and stores the value into slot
//           [strip] of every mailbox with a release flag, and one that waits
//           for all G flags and sums the G slots in strip order — identical
//           on every rank, deterministic.  The same kernels serve S strips
//           held by one process (loopback: mailbox table = local pointers;
//           every wait is already satisfied by the preceding push in stream
//           order), which is how the protocol is exercised on one GPU.
//
// CG semantics are the reference's (fermion.py:171-217) for a single chain.
// p and x are updated on halo rows too (from exchanged r and their own
// previous halos, bit-identical to the owner's values), so each iteration
// exchanges only r.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>

#include "common.cuh"
#include "runtime.hpp"
#include "tile.cuh"
#include "march.cuh"
#include "tma_tile.cuh"
#include "../../include/schwinger_sm100.h"

namespace {

constexpr int kHalo = 2;
constexpr int kDDReplace = 50;

// ---------------------------------------------------------------- NCCL (dlopen)
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
};

NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    api.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (api.h) {
      auto sym = [&](const char* n) { return dlsym(api.h, n); };
      api.GetUniqueId = (decltype(api.GetUniqueId))sym("ncclGetUniqueId");
      api.CommInitRank = (decltype(api.CommInitRank))sym("ncclCommInitRank");
      api.CommDestroy = (decltype(api.CommDestroy))sym("ncclCommDestroy");
      api.GroupStart = (decltype(api.GroupStart))sym("ncclGroupStart");
      api.GroupEnd = (decltype(api.GroupEnd))sym("ncclGroupEnd");
      api.Send = (decltype(api.Send))sym("ncclSend");
      api.Recv = (decltype(api.Recv))sym("ncclRecv");
      api.AllReduce = (decltype(api.AllReduce))sym("ncclAllReduce");
      api.AllGather = (decltype(api.AllGather))sym("ncclAllGather");
      api.GetErrorString = (decltype(api.GetErrorString))sym("ncclGetErrorString");
      api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.GroupStart &&
               api.GroupEnd && api.Send && api.Recv && api.AllReduce && api.AllGather;
    }
  }
  return api;
}

#define SCH_NCCL(ctx, expr)                                                               \
  do {                                                                                    \
    ncclResult_t _r = (expr);                                                             \
    if (_r != ncclSuccess)                                                                \
      return sch_fail((ctx), SCH_ERR_CUDA, "%s:%d %s: %s", __FILE__, __LINE__, #expr,     \
                      nccl().GetErrorString ? nccl().GetErrorString(_r) : "nccl error");  \
  } while (0)

}  // namespace

struct sch_dd {
  int nranks = 1, rank = 0;   // transport ranks
  int S = 1;                  // strips held by this process
  int G = 1;                  // strips in the whole lattice
  int L = 0, T = 0, Lloc = 0, Lext = 0;
  ncclComm_t comm = nullptr;  // null => local transport (unless p2p)
  // p2p transport (peer-memory mailboxes)
  bool p2p = false;
  char* box_mem = nullptr;            // this process's S mailboxes
  size_t box_bytes = 0;               // one mailbox
  char** box_tab = nullptr;           // device table: G mailbox pointers
  std::vector<void*> ipc_opened;      // peer allocations mapped with cudaIpcOpenMemHandle
  // device counters: [0] exchanges done, [1] global sums done, [2] pull CTAs
  // finished in the current exchange.  Kept on the device so the kernels
  // find their sequence number themselves and a CG loop can be captured.
  unsigned long long* seq_dev = nullptr;
  // canonical global sums (see "Decomposition-invariant sums" below)
  int CW = 0, NC = 0;                 // row-chunk width and chunks per row (T / CW)
  int* red_ctr = nullptr;             // last-CTA ticket of k_dd_rowred (self-resetting)
  double* red_blk = nullptr;          // [S][nb] 64-row block values
  double* red_all = nullptr;          // [0]: this rank's strip value, [1..G]: all-gathered (NCCL)
  double* own_part = nullptr;         // [S][Lloc][NC] row partials of sch_dd_own_sum
};

namespace {

// ------------------------------------------------------------- CG state
struct DDState {
  double* sc;   // scalars: see SC_* below
  int* flag;    // [S] need_x (X pass) per local strip (all equal)
  double* beta; // [S] beta per local strip (all equal)
  int* ctl;     // [0] done, [1] iters, [2] status, [3] current iteration (device-side loop)
};
enum { SC_NORMB2 = 0, SC_PAP, SC_RR, SC_TN2, SC_RS, SC_RSNEW, SC_ALPHA, SC_NORMB, SC_TARGET,
       SC_BEST, SC_RELRES, SC_COUNT };

SCH_DEV bool own_row(long long i, int T, int Lext, int lo, int hi) {
  const int row = (int)((i / T) % Lext);
  return row >= lo && row < hi;
}


// Scalar control of the decomposed CG (fermion.py:171-217), run by one
// thread right after the global sum it needs — fused into the sum's kernel
// (local and p2p transports) or a 1-thread kernel after the NCCL all-reduce.
SCH_DEV void dd_alpha(DDState st) {
  if (st.ctl[0]) return;
  const double den = st.sc[SC_PAP];
  st.sc[SC_ALPHA] = den > 0.0 ? st.sc[SC_RS] / den : 0.0;
}

SCH_DEV void dd_check(DDState st, int S) {
  if (st.ctl[0]) return;
  const int repl = (st.ctl[3] % kDDReplace) == 0;
  int need;
  if (repl) {
    need = 1;
  } else {
    const double rsn = st.sc[SC_RR];
    st.sc[SC_RSNEW] = rsn;
    need = sqrt(rsn) <= st.sc[SC_TARGET];
  }
  for (int s = 0; s < S; ++s) st.flag[s] = need;
}

SCH_DEV void dd_final(DDState st, int S, int maxiter) {
  if (st.ctl[0]) return;
  const int it = st.ctl[3];
  const int nx = st.flag[0];
  double rs_new = st.sc[SC_RSNEW];
  if (nx) {
    const double tn2 = st.sc[SC_TN2];
    const double tn = sqrt(tn2);
    const int repl = (it % kDDReplace) == 0;
    if (!repl || tn <= st.sc[SC_TARGET]) st.sc[SC_BEST] = tn / st.sc[SC_NORMB];
    if (tn <= st.sc[SC_TARGET]) {
      st.ctl[0] = 1;
      st.ctl[1] = it;
      st.sc[SC_RELRES] = tn / st.sc[SC_NORMB];
      for (int s = 0; s < S; ++s) st.flag[s] = 0;
      return;
    }
    rs_new = tn2;
  }
  const double rs = st.sc[SC_RS];
  const double beta = rs > 0.0 ? rs_new / rs : 0.0;
  for (int s = 0; s < S; ++s) {
    st.beta[s] = beta;
    st.flag[s] = 0;
  }
  st.sc[SC_RS] = rs_new;
  if (it >= maxiter) {
    st.ctl[0] = 1;
    st.ctl[1] = it;
    st.ctl[2] = 1;
    st.sc[SC_RELRES] = fmin(st.sc[SC_BEST], sqrt(rs_new) / st.sc[SC_NORMB]);
  }
}

enum { POST_NONE = 0, POST_ALPHA, POST_CHECK, POST_FINAL };
struct DDPost {
  int kind = POST_NONE;
  DDState st{};
  int S = 1, maxiter = 0;
  int set_cond = 0;                    // POST_FINAL inside the WHILE graph: drive its condition
  cudaGraphConditionalHandle h = 0;
};

SCH_DEV void dd_post_run(const DDPost& p) {
  if (p.kind == POST_ALPHA) {
    dd_alpha(p.st);
  } else if (p.kind == POST_CHECK) {
    dd_check(p.st, p.S);
  } else if (p.kind == POST_FINAL) {
    dd_final(p.st, p.S, p.maxiter);
    ++p.st.ctl[3];
    if (p.set_cond)   // iterate while not done (and below the cap)
      cudaGraphSetConditional(p.h, (p.st.ctl[0] == 0 && p.st.ctl[3] <= p.maxiter) ? 1u : 0u);
  }
}

__global__ void k_dd_post(DDPost p) { dd_post_run(p); }

// ---------------------------------------------------------- halo exchange
// Field layout [S][P planes][Lext][T][W doubles]; copy the 4 halo rows of
// every strip from its periodic neighbours (local transport).
__global__ void k_dd_exchange_local(double* __restrict__ f, int S, int P, int Lext, int Lloc, int T,
                                    int W) {
  const long long row = (long long)T * W;
  const long long n = (long long)S * P * 4 * row;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const long long e = i % row;
    long long q = i / row;
    const int h = (int)(q % 4);
    q /= 4;
    const int pl = (int)(q % P);
    const int s = (int)(q / P);
    // destination halo row and its source strip/row
    int dst_row, src_strip, src_row;
    if (h < 2) {                    // rows 0,1 <- left's Lloc, Lloc+1
      dst_row = h;
      src_strip = (s - 1 + S) % S;
      src_row = Lloc + h;
    } else {                        // rows Lloc+2, Lloc+3 <- right's 2, 3
      dst_row = Lloc + h;
      src_strip = (s + 1) % S;
      src_row = h;
    }
    const long long plane = (long long)Lext * row;
    f[((long long)s * P + pl) * plane + dst_row * row + e] =
        f[((long long)src_strip * P + pl) * plane + src_row * row + e];
  }
}

int p2p_exchange(sch_ctx* ctx, sch_dd* dd, double* f, int P, int W);

int dd_exchange(sch_ctx* ctx, sch_dd* dd, double* f, int P, int W) {
  if (dd->p2p) return p2p_exchange(ctx, dd, f, P, W);
  if (dd->comm == nullptr) {
    if (dd->nranks > 1) return sch_fail(ctx, SCH_ERR_ARG, "dd: no transport (NCCL id or p2p connect)");
    const long long n = (long long)dd->S * P * 4 * dd->T * W;
    unsigned grid = (unsigned)std::min<long long>((n + 255) / 256, 148 * 16);
    k_dd_exchange_local<<<grid, 256, 0, ctx->stream>>>(f, dd->S, P, dd->Lext, dd->Lloc, dd->T, W);
    SCH_LAUNCHED(ctx);
    return SCH_OK;
  }
  NcclApi& n = nccl();
  const int left = (dd->rank - 1 + dd->nranks) % dd->nranks;
  const int right = (dd->rank + 1) % dd->nranks;
  const size_t face = (size_t)2 * dd->T * W;   // two rows
  const size_t row = (size_t)dd->T * W;
  const size_t plane = (size_t)dd->Lext * row;
  SCH_NCCL(ctx, n.GroupStart());
  for (int pl = 0; pl < P; ++pl) {
    double* base = f + pl * plane;
    SCH_NCCL(ctx, n.Send(base + dd->Lloc * row, face, ncclDouble, right, dd->comm, ctx->stream));
    SCH_NCCL(ctx, n.Recv(base, face, ncclDouble, left, dd->comm, ctx->stream));
    SCH_NCCL(ctx, n.Send(base + 2 * row, face, ncclDouble, left, dd->comm, ctx->stream));
    SCH_NCCL(ctx, n.Recv(base + (dd->Lloc + 2) * row, face, ncclDouble, right, dd->comm, ctx->stream));
  }
  SCH_NCCL(ctx, n.GroupEnd());
  return SCH_OK;
}

// ------------------------------------------------------ p2p transport
// Mailbox of one strip (in its owner's HBM), byte offsets from P2PBox:
//   [0]    u64 arrived[2]   push CTAs that delivered into face side d
//   [16]   u64 acked[2]     pull CTAs of the neighbour that consumed what
//                           this strip pushed right (0) / left (1)
//   [256]  u64 redflag[G]   last global-sum sequence number stored by strip g
//   [..]   f64 red[2][G]    global-sum slots (two, by sequence parity)
//   [..]   f64 face[2][2][2*T*kFW]  side (0 = from the left neighbour,
//                           1 = from the right) x slot (sequence parity) x
//                           two rows of up to kFW words per site
constexpr int kFW = 4;          // words per site a face slot holds (P*W <= 4)
constexpr int kNBuf = 2;        // face / sum slots per side (credit window)
constexpr int kP2PBlk = 16;     // CTAs per side of a push / pull launch (counting unit)
constexpr long long kSpinCap = 1ll << 27;   // ~10 s of polling, then trap (no silent hang)

struct P2PGeom {
  size_t off_redflag, off_red, off_face, bytes;
  long long slot_words;
};

P2PGeom p2p_geom(int G, int T) {
  P2PGeom g;
  auto al = [](size_t v) { return (v + 255) & ~size_t(255); };
  g.off_redflag = 256;
  g.off_red = al(g.off_redflag + sizeof(unsigned long long) * G);
  g.off_face = al(g.off_red + sizeof(double) * kNBuf * G);
  g.slot_words = 2ll * T * kFW;
  g.bytes = al(g.off_face + sizeof(double) * 2 * kNBuf * g.slot_words);
  return g;
}

SCH_DEV unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
SCH_DEV void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
SCH_DEV void add_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
SCH_DEV void spin_until(const unsigned long long* p, unsigned long long target) {
  long long n = 0;
  while (ld_acquire_sys(p) < target) {
    __nanosleep(64);
    if (++n > kSpinCap) __trap();   // a peer never arrived: fail the launch, do not hang
  }
}

struct P2PArgs {
  char* const* tab;   // G mailbox pointers (local or IPC-mapped)
  unsigned long long* seq;   // sch_dd::seq_dev
  int strip0, S, G, Lext, Lloc, T;
  size_t off_redflag, off_red, off_face;
  long long slot_words;
};

SCH_DEV unsigned long long* box_u64(const P2PArgs& a, int g, size_t off) {
  return (unsigned long long*)(a.tab[g] + off);
}

// grid (kP2PBlk, S, 2): d = 0 pushes rows Lloc, Lloc+1 into the right
// neighbour's side-0 slot, d = 1 rows 2, 3 into the left neighbour's side-1 slot
__global__ void k_p2p_push(const double* __restrict__ f, int P, int W, P2PArgs a) {
  const int s = blockIdx.y, d = blockIdx.z, g = a.strip0 + s;
  const unsigned long long seq = *(volatile unsigned long long*)a.seq + 1;
  const int tgt = d == 0 ? (g + 1) % a.G : (g - 1 + a.G) % a.G;
  if (threadIdx.x == 0 && seq > kNBuf)   // credit: the slot's previous content was consumed
    spin_until(box_u64(a, g, 16 + 8 * d), (unsigned long long)kP2PBlk * (seq - kNBuf));
  __syncthreads();
  double* slot = (double*)(a.tab[tgt] + a.off_face) + (d * kNBuf + seq % kNBuf) * a.slot_words;
  const long long row = (long long)a.T * W, per_plane = 2 * row;
  const long long plane = (long long)a.Lext * row;
  const double* src = f + (long long)s * P * plane + (long long)(d == 0 ? a.Lloc : 2) * row;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < P * per_plane;
       i += (long long)gridDim.x * blockDim.x) {
    const long long pl = i / per_plane, e = i - pl * per_plane;
    slot[i] = src[pl * plane + e];   // NVLink store when tgt is remote
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    add_release_sys(box_u64(a, tgt, 8 * d), 1ull);
  }
}

// grid (kP2PBlk, S, 2): d = 0 fills rows 0, 1 from side 0, d = 1 rows
// Lloc+2, Lloc+3 from side 1, then returns the credit to the producer
__global__ void k_p2p_pull(double* __restrict__ f, int P, int W, P2PArgs a) {
  const int s = blockIdx.y, d = blockIdx.z, g = a.strip0 + s;
  const unsigned long long seq = *(volatile unsigned long long*)a.seq + 1;
  const int src_strip = d == 0 ? (g - 1 + a.G) % a.G : (g + 1) % a.G;
  if (threadIdx.x == 0) spin_until(box_u64(a, g, 8 * d), (unsigned long long)kP2PBlk * seq);
  __syncthreads();
  const double* slot = (const double*)(a.tab[g] + a.off_face) + (d * kNBuf + seq % kNBuf) * a.slot_words;
  const long long row = (long long)a.T * W, per_plane = 2 * row;
  const long long plane = (long long)a.Lext * row;
  double* dst = f + (long long)s * P * plane + (long long)(d == 0 ? 0 : a.Lloc + 2) * row;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < P * per_plane;
       i += (long long)gridDim.x * blockDim.x) {
    const long long pl = i / per_plane, e = i - pl * per_plane;
    dst[pl * plane + e] = __ldcg(slot + i);   // L2: the peer's stores land there, not in L1
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    add_release_sys(box_u64(a, src_strip, 16 + 8 * d), 1ull);
    // the last CTA out advances the exchange counter (every CTA has read it)
    const unsigned long long total = (unsigned long long)gridDim.x * gridDim.y * gridDim.z;
    if (atomicAdd(a.seq + 2, 1ull) == total - 1) {
      a.seq[2] = 0;
      __threadfence();
      *(volatile unsigned long long*)a.seq = seq;
    }
  }
}

// Canonical tree (balanced, index order, zero padded) of n <= 256 values in
// global memory by one warp: lane l owns [l*K, l*K + K), K = the power of two
// >= n/32; every lane returns the sum.
SCH_DEV double warp_canon(const double* v, int n, int lane) {
  if (n > 64 && (n & 1) == 0) {
    // long rows (the marching pass writes T/4 partials per row): coalesced
    // 16-B loads, chunk by chunk.  Lane l of chunk c holds values 64c + 2l,
    // 64c + 2l + 1: their sum is the tree's first level, the xor butterfly
    // the next five, so every lane ends with the subtree of the aligned
    // 64-chunk; lane c keeps chunk c's value and the butterfly over the lanes
    // (zero padded) is the top of the tree.  n <= 2048.
    double keep = 0.0;
    const int nc = (n + 63) / 64;
    for (int c0 = 0; c0 < nc; c0 += 4) {
      double a[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int i = 64 * (c0 + j) + 2 * lane;
        a[j] = 0.0;
        if (i < n) {
          const double2 q = __ldcg(reinterpret_cast<const double2*>(v + i));
          a[j] = q.x + q.y;
        }
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        a[j] = warp_tree_sum(a[j]);
        if (lane == c0 + j) keep = a[j];
      }
    }
    return warp_tree_sum(keep);
  }
  int K = 1;
  while (32 * K < n) K <<= 1;
  double a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int i = lane * K + k;
    a[k] = (k < K && i < n) ? __ldcg(v + i) : 0.0;
  }
#pragma unroll
  for (int w = 4; w >= 1; w >>= 1)
#pragma unroll
    for (int k = 0; k < w; ++k) a[k] = a[2 * k] + a[2 * k + 1];
  return warp_tree_sum(a[0]);
}

// wait for the G strip values of sum `seq` in the first local strip's
// mailbox and combine them by the canonical tree (the same bits on every rank)
__global__ void k_p2p_red_finish(P2PArgs a, double* __restrict__ out, DDPost post) {
  const int g0 = a.strip0;
  const unsigned long long seq = *(volatile unsigned long long*)(a.seq + 1) + 1;
  for (int h = threadIdx.x; h < a.G; h += blockDim.x) spin_until(box_u64(a, g0, a.off_redflag) + h, seq);
  __syncwarp();
  const double* red = (const double*)(a.tab[g0] + a.off_red) + (seq % kNBuf) * a.G;
  const double v = warp_canon(red, a.G, threadIdx.x & 31);
  if (threadIdx.x == 0) {
    *out = v;
    dd_post_run(post);
  }
  __syncwarp();
  if (threadIdx.x == 0) *(volatile unsigned long long*)(a.seq + 1) = seq;   // one warp: all have read it
}

P2PArgs p2p_args(const sch_dd* dd) {
  const P2PGeom pg = p2p_geom(dd->G, dd->T);
  P2PArgs a;
  a.tab = dd->box_tab;
  a.seq = dd->seq_dev;
  a.strip0 = dd->rank * dd->S;
  a.S = dd->S;
  a.G = dd->G;
  a.Lext = dd->Lext;
  a.Lloc = dd->Lloc;
  a.T = dd->T;
  a.off_redflag = pg.off_redflag;
  a.off_red = pg.off_red;
  a.off_face = pg.off_face;
  a.slot_words = pg.slot_words;
  return a;
}

int p2p_exchange(sch_ctx* ctx, sch_dd* dd, double* f, int P, int W) {
  if (P * W > kFW) return sch_fail(ctx, SCH_ERR_ARG, "p2p exchange: %d words per site > %d", P * W, kFW);
  const P2PArgs a = p2p_args(dd);
  const dim3 grid(kP2PBlk, dd->S, 2);
  k_p2p_push<<<grid, 256, 0, ctx->stream>>>(f, P, W, a);
  k_p2p_pull<<<grid, 256, 0, ctx->stream>>>(f, P, W, a);
  ctx->launches += 2;
  return SCH_OK;
}

// ------------------------------------------ decomposition-invariant sums
// Every global sum of the decomposed lattice (the CG's <p,Ap>, ||r||^2,
// ||b - Ax||^2, ||b||^2 and the Hamiltonian's terms) is one fixed
// expression of its site values:
//     sum = C_x ( C_c ( C_t (site value) ) )
// C is the canonical tree — a balanced binary tree over the values in index
// order, zero padded to a power of two; x runs over the L global rows, c
// over the T/CW chunks of a row, t over the CW sites of a chunk.  The
// producing kernels write one partial per (own row, chunk) (row_chunk_sum,
// tile.cuh, and the warp-per-chunk passes below); k_dd_rowred forms each
// strip's value, C over its rows (64-row blocks, then the blocks), and the
// strips' values are combined by C over the G strips: inside the kernel for
// the local transport, by k_p2p_red_finish after the mailbox pushes, or by
// k_dd_tree_post after an ncclAllGather of the G values.  With a power-of-
// two strip height Lloc every strip is a subtree of C over the L rows, so
// each sum — and with it every CG iteration count, stopping decision and
// Hamiltonian — is bit-identical for every number of strips G and every
// transport.
enum { RED_LOCAL = 0, RED_P2P = 1, RED_NCCL = 2 };
constexpr int kRowBlk = 8;      // rows per CTA of k_dd_rowred (one per warp: 64 rows per CTA,
                                // eight per warp in sequence, measured 13 us per sum at 2048 rows)
constexpr int kMaxCanon = 1024; // values one CTA combines (blocks per strip, strips)

struct RowRed {
  const double* part;   // [S][Lloc][nch] row-chunk partials
  int S, Lloc, nch, nb; // nb = ceil(Lloc / kRowBlk)
  double* blk;          // [S][nb]
  const int* need;      // when set and need[0] == 0 the sum is not used: nothing is read
  int* ctr;             // last-CTA ticket (reset by the last CTA)
  int mode;
  double* out;          // local: the global sum; NCCL: this rank's strip value
  DDPost post;          // local transport: the CG control fused into the sum
  P2PArgs pa;           // p2p transport: mailboxes
};

// C over n <= kMaxCanon values (global when GLOBAL, else shared), by the
// whole CTA, ping-pong through two shared buffers; every thread returns it
template <bool GLOBAL>
SCH_DEV double block_canon(const double* v, int n, double* t0, double* t1) {
  int P = 1;
  while (P < n) P <<= 1;
  for (int i = threadIdx.x; i < P; i += blockDim.x)
    t0[i] = i < n ? (GLOBAL ? __ldcg(v + i) : v[i]) : 0.0;
  __syncthreads();
  for (int w = P >> 1; w >= 1; w >>= 1) {
    for (int i = threadIdx.x; i < w; i += blockDim.x) t1[i] = t0[2 * i] + t0[2 * i + 1];
    __syncthreads();
    double* tmp = t0;
    t0 = t1;
    t1 = tmp;
  }
  const double r = t0[0];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(256) k_dd_rowred(RowRed a) {
  __shared__ double rv[kRowBlk];
  __shared__ double t0[kMaxCanon], t1[kMaxCanon], sv[kMaxCanon];
  __shared__ int last;
  const int b = blockIdx.x, s = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // The true-residual sum of an iteration whose stop test did not ask for it
  // (its pass wrote nothing, dd_final ignores the value; `need` is the same
  // on every rank, and is rewritten only by the post of this kernel's last
  // CTA, after every CTA has read it).  Local transport: only the control
  // runs; the others keep their protocol and push zeros.
  const bool skip = a.need != nullptr && a.need[0] == 0;
  if (skip && a.mode == RED_LOCAL) {
    if (b == 0 && s == 0 && threadIdx.x == 0) dd_post_run(a.post);
    return;
  }
  constexpr int RPW = kRowBlk / 8;   // rows per warp (8 warps)
  for (int i = 0; i < RPW; ++i) {
    const int y = b * kRowBlk + warp * RPW + i;
    double v = 0.0;
    if (y < a.Lloc && !skip) v = warp_canon(a.part + ((long long)s * a.Lloc + y) * a.nch, a.nch, lane);
    if (lane == 0) rv[warp * RPW + i] = v;
  }
  __syncthreads();
  if (warp == 0) {   // C over the block's rows (zero padded: exact)
    const double v = warp_tree_sum(2 * lane + 1 < kRowBlk ? rv[2 * lane] + rv[2 * lane + 1] : 0.0);
    if (lane == 0) {
      a.blk[(long long)s * a.nb + b] = v;
      __threadfence();
      last = atomicAdd(a.ctr, 1) == a.nb * a.S - 1;
    }
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int st = 0; st < a.S; ++st) {
    const double v = block_canon<true>(a.blk + (long long)st * a.nb, a.nb, t0, t1);
    if (threadIdx.x == 0) sv[st] = v;
  }
  __syncthreads();
  if (a.mode == RED_LOCAL) {
    const double v = block_canon<false>(sv, a.S, t0, t1);
    if (threadIdx.x == 0) {
      *a.out = v;
      dd_post_run(a.post);
    }
  } else if (a.mode == RED_NCCL) {
    if (threadIdx.x == 0) *a.out = sv[0];
  } else if (threadIdx.x == 0) {   // p2p: strip values -> slot [seq parity][g] of every mailbox
    const P2PArgs& pa = a.pa;
    const unsigned long long seq = *(volatile unsigned long long*)(pa.seq + 1) + 1;
    for (int st = 0; st < a.S; ++st) {
      const int g = pa.strip0 + st;
      for (int h = 0; h < pa.G; ++h) ((double*)(pa.tab[h] + pa.off_red))[(seq % kNBuf) * pa.G + g] = sv[st];
    }
    __threadfence_system();
    for (int st = 0; st < a.S; ++st)
      for (int h = 0; h < pa.G; ++h) st_release_sys(box_u64(pa, h, pa.off_redflag) + pa.strip0 + st, seq);
  }
  if (threadIdx.x == 0) *a.ctr = 0;
}

// NCCL transport: C over the G all-gathered strip values
__global__ void k_dd_tree_post(const double* __restrict__ vals, int G, double* __restrict__ out,
                               DDPost post) {
  const double v = warp_canon(vals, G, threadIdx.x & 31);
  if (threadIdx.x == 0) {
    *out = v;
    dd_post_run(post);
  }
}

// the global sum of the row partials `part` ([S][Lloc][NC]) into *out (on
// the device, every rank); `post` runs on the sum
int dd_allsum(sch_ctx* ctx, sch_dd* dd, const double* part, double* out,
              const DDPost& post = DDPost{}, int nch = 0, const int* need = nullptr) {
  if (!dd->p2p && dd->comm == nullptr && dd->nranks > 1)
    return sch_fail(ctx, SCH_ERR_ARG, "dd: no transport (NCCL id or p2p connect)");
  RowRed a;
  a.part = part;
  a.S = dd->S;
  a.Lloc = dd->Lloc;
  a.nch = nch > 0 ? nch : dd->NC;   // chunks per row of `part` (any power-of-two width: same tree)
  a.nb = (dd->Lloc + kRowBlk - 1) / kRowBlk;
  a.blk = dd->red_blk;
  a.need = need;
  a.ctr = dd->red_ctr;
  a.mode = dd->p2p ? RED_P2P : dd->comm ? RED_NCCL : RED_LOCAL;
  a.out = a.mode == RED_NCCL ? dd->red_all : out;
  a.post = a.mode == RED_LOCAL ? post : DDPost{};
  a.pa = dd->p2p ? p2p_args(dd) : P2PArgs{};
  k_dd_rowred<<<dim3(a.nb, dd->S), 256, 0, ctx->stream>>>(a);
  SCH_LAUNCHED(ctx);
  if (a.mode == RED_P2P) {
    k_p2p_red_finish<<<1, 32, 0, ctx->stream>>>(a.pa, out, post);
    SCH_LAUNCHED(ctx);
  } else if (a.mode == RED_NCCL) {
    SCH_NCCL(ctx, nccl().AllGather(dd->red_all, dd->red_all + 1, 1, ncclDouble, dd->comm, ctx->stream));
    k_dd_tree_post<<<1, 32, 0, ctx->stream>>>(dd->red_all + 1, dd->G, out, post);
    SCH_LAUNCHED(ctx);
  }
  return SCH_OK;
}

// Warp-per-chunk passes: a work item is (strip s, extended row xr, chunk ch);
// lane l owns sites ch*CW + l*K + k (k < K; K = 2 for CW = 64, else 1 and
// lanes >= CW idle), and an own row's chunk partial is C over its CW site
// values — the same tree as row_chunk_sum in the tile kernels.
struct ChunkItem {
  int s, xr, ch;
};
SCH_DEV ChunkItem chunk_item(long long w, int nch, int rows) {
  ChunkItem c;
  c.ch = (int)(w % nch);
  const long long sr = w / nch;
  c.xr = (int)(sr % rows);
  c.s = (int)(sr / rows);
  return c;
}

// x = x0|0, r = p = b on every row (b's halos already exchanged); the row
// partials of ||b||^2 on the own rows
__global__ void k_dd_init(const double2* __restrict__ b, const double2* __restrict__ x0,
                          double2* __restrict__ x, double2* __restrict__ r, double2* __restrict__ p,
                          int S, int Lext, int T, int CW, int lo, int hi, double* __restrict__ rowpart) {
  const int lane = threadIdx.x & 31, K = CW > 32 ? 2 : 1, nch = T / CW;
  const long long items = (long long)S * Lext * nch;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < items; w += nw) {
    const ChunkItem c = chunk_item(w, nch, Lext);
    double v[2] = {0.0, 0.0};
    for (int k = 0; k < K; ++k) {
      const int j = lane * K + k;
      if (j >= CW) continue;
      const long long i = ((long long)c.s * Lext + c.xr) * T + c.ch * CW + j;
      Spinor bv = ld256_spinor_nc(b, i);
      Spinor xv;
      if (x0) xv = ld256_spinor_nc(x0, i);
      else xv.s0 = xv.s1 = make_double2(0, 0);
      st256_spinor(x, i, xv);
      st256_spinor(r, i, bv);
      st256_spinor(p, i, bv);
      v[k] = spinor_norm2(bv);
    }
    if (c.xr >= lo && c.xr < hi) {   // warp-uniform
      const double t = warp_tree_sum(v[0] + v[1]);
      if (lane == 0) rowpart[((long long)c.s * (hi - lo) + (c.xr - lo)) * nch + c.ch] = t;
    }
  }
}

__global__ void k_dd_copy(const double2* __restrict__ src, double2* __restrict__ dst, long long nsites) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nsites;
       i += (long long)gridDim.x * blockDim.x)
    st256_spinor(dst, i, ld256_spinor(src, i));
}

__global__ void k_dd_ctrl_init(DDState st, int S, double tol, int have_x0) {
  const double nb2 = st.sc[SC_NORMB2];
  const double nb = sqrt(nb2);
  st.sc[SC_NORMB] = nb;
  st.sc[SC_TARGET] = tol * nb;
  st.sc[SC_RS] = have_x0 ? st.sc[SC_RR] : nb2;
  st.sc[SC_BEST] = INFINITY;
  st.sc[SC_RELRES] = 0.0;
  for (int s = 0; s < S; ++s) {
    st.beta[s] = 0.0;
    st.flag[s] = 0;
  }
  st.ctl[0] = nb == 0.0 ? 1 : 0;   // zero rhs: x = 0, 0 iterations (fermion.py:181-182)
  st.ctl[1] = 0;
  st.ctl[2] = 0;
  st.ctl[3] = 1;
}

// p = r + beta p, x += alpha p on every row; r -= alpha ap and the row
// partials of ||r||^2 on the own rows (not on residual-replacement
// iterations, where the true-residual pass forms r)
__global__ void k_dd_update(double2* __restrict__ r, double2* __restrict__ p, double2* __restrict__ x,
                            const double2* __restrict__ ap, DDState st, int S, int Lext, int T, int CW,
                            int lo, int hi, double* __restrict__ rowpart) {
  if (st.ctl[0]) return;
  const int repl = (st.ctl[3] % kDDReplace) == 0;
  const double al = st.sc[SC_ALPHA], be = st.beta[0];
  const int lane = threadIdx.x & 31, K = CW > 32 ? 2 : 1, nch = T / CW;
  const long long items = (long long)S * Lext * nch;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < items; w += nw) {
    const ChunkItem c = chunk_item(w, nch, Lext);
    const bool own = c.xr >= lo && c.xr < hi;
    double v[2] = {0.0, 0.0};
    for (int k = 0; k < K; ++k) {
      const int j = lane * K + k;
      if (j >= CW) continue;
      const long long i = ((long long)c.s * Lext + c.xr) * T + c.ch * CW + j;
      Spinor rv = ld256_spinor(r, i), pv = ld256_spinor(p, i), xv = ld256_spinor(x, i);
      pv = sp_fma(be, pv, rv);
      xv = sp_fma(al, pv, xv);
      st256_spinor(p, i, pv);
      st256_spinor(x, i, xv);
      if (!repl && own) {
        rv = sp_fma(-al, ld256_spinor_nc(ap, i), rv);
        st256_spinor(r, i, rv);
        v[k] = spinor_norm2(rv);
      }
    }
    if (own) {
      const double t = warp_tree_sum(v[0] + v[1]);
      if (lane == 0) rowpart[((long long)c.s * (hi - lo) + (c.xr - lo)) * nch + c.ch] = t;
    }
  }
}

// Row partials of the Hamiltonian's sums over the own rows (site values:
// kind 0 p_0^2 + p_1^2, kind 1 1 - cos theta, kind 2 Re conj(a) b over the
// two spin components)
__global__ void k_dd_own_sum(int kind, const double* __restrict__ a, const double* __restrict__ b,
                             int S, int Lext, int T, int CW, int lo, int hi,
                             double* __restrict__ rowpart) {
  const int lane = threadIdx.x & 31, K = CW > 32 ? 2 : 1, nch = T / CW, own = hi - lo;
  const long long plane = (long long)Lext * T;
  const long long items = (long long)S * own * nch;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < items; w += nw) {
    const ChunkItem c = chunk_item(w, nch, own);
    const int x = lo + c.xr;
    double v[2] = {0.0, 0.0};
    for (int k = 0; k < K; ++k) {
      const int j = lane * K + k;
      if (j >= CW) continue;
      const int t = c.ch * CW + j;
      if (kind == 0) {
        const double* ps = a + (long long)c.s * 2 * plane + (long long)x * T + t;
        v[k] = ps[0] * ps[0] + ps[plane] * ps[plane];
      } else if (kind == 1) {
        v[k] = 1.0 - cos(plaq(a + (long long)c.s * 2 * plane, Lext, T, x, t));
      } else {
        const long long e = 2 * ((long long)c.s * plane + (long long)x * T + t);
        const double2* as = (const double2*)a;
        const double2* bs = (const double2*)b;
        v[k] = redot(as[e], bs[e]) + redot(as[e + 1], bs[e + 1]);
      }
    }
    const double t = warp_tree_sum(v[0] + v[1]);
    if (lane == 0) rowpart[((long long)c.s * own + c.xr) * nch + c.ch] = t;
  }
}

// grid of the warp-per-chunk passes: enough warps for one wave
inline unsigned chunk_grid(long long items) {
  return (unsigned)std::max<long long>(1, std::min<long long>((items + 7) / 8, 148 * 8));
}

// The stencil pass of the decomposed lattice: the warp-marching register
// kernel (march.cuh), else — SCH_DD_MARCH=0, or rows beyond 8192 sites — the
// one-tile-per-CTA halo kernel.  Both write canonical row-chunk partials;
// only the chunk width differs.  (Round 2's TMA 2-D tile kernel, 55 % of HBM
// on cfg5 against the marching pass's 80-89 %, was removed.)
enum { ST_TILE = 0, ST_MARCH = 2 };
int dd_stencil_kind(const sch_dd* dd) {
  return march_enabled() && march_shape_ok(dd->T) ? ST_MARCH : ST_TILE;
}
// chunks per row of the stencil pass's partials (0: the lattice's own NC)
int dd_stencil_nch(const sch_dd* dd, int kind) { return kind == ST_MARCH ? march_nch(dd->T) : 0; }
template <int MODE>
void dd_stencil_launch(int kind, const TileShape& sh, const TileArgs& a, cudaStream_t st, int num_sms) {
  if (kind == ST_MARCH && launch_dd_march<MODE>(a, st, num_sms)) return;
  launch_dd_tile<MODE>(sh, a, st);
}

TileArgs dd_tile_args(sch_dd* dd, const TileShape& sh, const double2* U, double m0) {
  TileArgs a{};
  a.U = U;
  a.B = dd->S;
  a.L = dd->Lext;
  a.T = dd->T;
  a.tiles_t = sh.tiles_t;
  a.tiles_per_chain = sh.tiles_x * sh.tiles_t;
  a.diag = 2.0 + m0;
  a.own_lo = kHalo;
  a.own_hi = kHalo + dd->Lloc;
  return a;
}

}  // namespace

extern "C" {

int sch_nccl_unique_id(sch_ctx* ctx, void* id_out) {
  SCH_CHECK_ARG(ctx, id_out != nullptr, "nccl_unique_id: null output");
  if (!nccl().ok) return sch_fail(ctx, SCH_ERR_CUDA, "libnccl.so.2 not available");
  ncclUniqueId id;
  SCH_NCCL(ctx, nccl().GetUniqueId(&id));
  memcpy(id_out, id.internal, sizeof(id.internal));
  return SCH_OK;
}

int sch_dd_create(sch_ctx* ctx, const void* nccl_id, int nranks, int rank, int L, int T,
                  int strips_local, sch_dd** out) {
  SCH_CHECK_ARG(ctx, out && nranks >= 1 && rank >= 0 && rank < nranks && strips_local >= 1,
                "dd_create: bad ranks");
  const int G = nranks * strips_local;
  SCH_CHECK_ARG(ctx, L % G == 0 && L / G >= 2 && T >= 2, "dd_create: L must split into strips of >= 2 rows");
  SCH_CHECK_ARG(ctx, nranks == 1 || strips_local == 1, "dd_create: multi-rank transports hold one strip per rank");
  sch_dd* dd = new sch_dd();
  dd->nranks = nranks;
  dd->rank = rank;
  dd->S = strips_local;
  dd->G = G;
  dd->L = L;
  dd->T = T;
  dd->Lloc = L / G;
  dd->Lext = dd->Lloc + 2 * kHalo;
  TileShape sh;
  if (dd_tile_shape(dd->Lext, T, sh)) {   // else: halo exchange only (stencils need T % 8 == 0)
    dd->CW = sh.TT;
    dd->NC = T / sh.TT;
  } else {
    dd->CW = 8;
    dd->NC = 1;
  }
  {
    const int nb = (dd->Lloc + kRowBlk - 1) / kRowBlk;
    if (nb > kMaxCanon || dd->S > kMaxCanon || dd->NC > 256 || G > 256) {
      delete dd;
      return sch_fail(ctx, SCH_ERR_ARG, "dd_create: lattice too large for the canonical sums");
    }
    cudaError_t e = cudaMalloc(&dd->red_ctr, sizeof(int));
    if (e == cudaSuccess) e = cudaMemset(dd->red_ctr, 0, sizeof(int));
    if (e == cudaSuccess) e = cudaMalloc(&dd->red_blk, sizeof(double) * (size_t)nb * dd->S);
    if (e == cudaSuccess) e = cudaMalloc(&dd->red_all, sizeof(double) * (G + 1));
    if (e == cudaSuccess)
      e = cudaMalloc(&dd->own_part, sizeof(double) * (size_t)dd->S * dd->Lloc * dd->NC);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      sch_dd_destroy(dd);
      return sch_fail(ctx, SCH_ERR_CUDA, "dd_create: %s", cudaGetErrorString(e));
    }
  }
  if (nccl_id != nullptr) {   // NCCL transport (else: local, or p2p connected later); one rank
                              // is allowed: its faces go to itself by ncclSend/ncclRecv
    if (!nccl().ok) {
      delete dd;
      return sch_fail(ctx, SCH_ERR_CUDA, "libnccl.so.2 not available");
    }
    ncclUniqueId id;
    memcpy(id.internal, nccl_id, sizeof(id.internal));
    ncclResult_t r = nccl().CommInitRank(&dd->comm, nranks, id, rank);
    if (r != ncclSuccess) {
      delete dd;
      return sch_fail(ctx, SCH_ERR_CUDA, "ncclCommInitRank: %s", nccl().GetErrorString(r));
    }
  }
  *out = dd;
  return SCH_OK;
}

int sch_dd_destroy(sch_dd* dd) {
  if (!dd) return SCH_OK;
  if (dd->comm) nccl().CommDestroy(dd->comm);
  for (void* ptr : dd->ipc_opened) cudaIpcCloseMemHandle(ptr);
  if (dd->box_tab) cudaFree(dd->box_tab);
  if (dd->seq_dev) cudaFree(dd->seq_dev);
  if (dd->box_mem) cudaFree(dd->box_mem);
  if (dd->red_ctr) cudaFree(dd->red_ctr);
  if (dd->red_blk) cudaFree(dd->red_blk);
  if (dd->red_all) cudaFree(dd->red_all);
  if (dd->own_part) cudaFree(dd->own_part);
  delete dd;
  return SCH_OK;
}

// p2p transport, step 1: allocate (zeroed) the mailboxes of this process's
// S strips and return their CUDA IPC handle (64 bytes) for the other ranks.
int sch_dd_p2p_open(sch_ctx* ctx, sch_dd* dd, void* ipc_handle_out) {
  SCH_CHECK_ARG(ctx, dd && ipc_handle_out, "dd_p2p_open: bad args");
  SCH_CHECK_ARG(ctx, !dd->box_mem, "dd_p2p_open: already open");
  const P2PGeom pg = p2p_geom(dd->G, dd->T);
  dd->box_bytes = pg.bytes;
  SCH_CUDA(ctx, cudaMalloc(&dd->box_mem, pg.bytes * dd->S));
  SCH_CUDA(ctx, cudaMemset(dd->box_mem, 0, pg.bytes * dd->S));
  SCH_CUDA(ctx, cudaMalloc(&dd->box_tab, sizeof(char*) * dd->G));
  SCH_CUDA(ctx, cudaMalloc(&dd->seq_dev, 4 * sizeof(unsigned long long)));
  SCH_CUDA(ctx, cudaMemset(dd->seq_dev, 0, 4 * sizeof(unsigned long long)));
  cudaIpcMemHandle_t h;
  memset(&h, 0, sizeof(h));
  if (dd->nranks > 1) SCH_CUDA(ctx, cudaIpcGetMemHandle(&h, dd->box_mem));
  memcpy(ipc_handle_out, &h, sizeof(h));
  SCH_CUDA(ctx, cudaDeviceSynchronize());   // mailboxes zeroed before any peer maps them
  return SCH_OK;
}

// p2p transport, step 2: map every other rank's mailboxes (handles: nranks
// x 64 bytes in rank order, as all-gathered by the host layer) and switch
// this dd to the p2p transport.  All ranks must have finished step 1.
int sch_dd_p2p_connect(sch_ctx* ctx, sch_dd* dd, const void* ipc_handles) {
  SCH_CHECK_ARG(ctx, dd && ipc_handles && dd->box_mem, "dd_p2p_connect: open first");
  std::vector<char*> tab(dd->G);
  for (int r = 0; r < dd->nranks; ++r) {
    char* base = dd->box_mem;
    if (r != dd->rank) {
      cudaIpcMemHandle_t h;
      memcpy(&h, (const char*)ipc_handles + 64 * (size_t)r, sizeof(h));
      void* ptr = nullptr;
      SCH_CUDA(ctx, cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
      dd->ipc_opened.push_back(ptr);
      base = (char*)ptr;
    }
    for (int s = 0; s < dd->S; ++s) tab[r * dd->S + s] = base + s * dd->box_bytes;
  }
  SCH_CUDA(ctx, cudaMemcpy(dd->box_tab, tab.data(), sizeof(char*) * dd->G, cudaMemcpyHostToDevice));
  dd->p2p = true;
  return SCH_OK;
}

int sch_dd_geometry(const sch_dd* dd, int* out4) {
  if (!dd || !out4) return SCH_ERR_ARG;
  out4[0] = dd->S;
  out4[1] = dd->Lloc;
  out4[2] = dd->Lext;
  out4[3] = dd->G;
  return SCH_OK;
}

// Whole-lattice sums over the own rows of extended fields (the
// Hamiltonian's reductions on a decomposed lattice), through the canonical
// tree and the lattice's transport, so every rank holds the same value:
//   kind 0: sum p^2               a = momenta [S][2][Lext][T]      (lattice.py:128-130, x 0.5 by the caller)
//   kind 1: sum (1 - cos theta)   a = links   [S][2][Lext][T]      (gauge.py:37-40)
//   kind 2: Re sum conj(a) b      a, b = spinors [S][Lext][T][2]   (fermion.py:54-56)
int sch_dd_own_sum(sch_ctx* ctx, sch_dd* dd, int kind, const double* a, const double* b,
                   double* out) {
  SCH_CHECK_ARG(ctx, dd && a && out && kind >= 0 && kind <= 2 && (kind != 2 || b),
                "dd_own_sum: bad args");
  SCH_CHECK_ARG(ctx, dd->T % 8 == 0, "dd_own_sum: T must be a multiple of 8");
  const long long items = (long long)dd->S * dd->Lloc * dd->NC;
  k_dd_own_sum<<<chunk_grid(items), 256, 0, ctx->stream>>>(kind, a, b, dd->S, dd->Lext, dd->T, dd->CW,
                                                           kHalo, kHalo + dd->Lloc, dd->own_part);
  SCH_LAUNCHED(ctx);
  return dd_allsum(ctx, dd, dd->own_part, out);
}

int sch_dd_exchange(sch_ctx* ctx, sch_dd* dd, double* field, int planes, int words_per_site) {
  SCH_CHECK_ARG(ctx, dd && field && planes >= 1 && words_per_site >= 1, "dd_exchange: bad args");
  return dd_exchange(ctx, dd, field, planes, words_per_site);
}

int sch_dd_ddagd(sch_ctx* ctx, sch_dd* dd, const double* U_ext, double* psi_ext, double* out_ext,
                 double m0) {
  SCH_CHECK_ARG(ctx, dd && U_ext && psi_ext && out_ext && psi_ext != out_ext, "dd_ddagd: bad args");
  SCH_CHECK_ARG(ctx, dd->T % 8 == 0, "dd_ddagd: T must be a multiple of 8");
  int rc = dd_exchange(ctx, dd, psi_ext, 1, 4);
  if (rc) return rc;
  TileShape sh;
  dd_tile_shape(dd->Lext, dd->T, sh);
  TileArgs a = dd_tile_args(dd, sh, (const double2*)U_ext, m0);
  a.in = (const double2*)psi_ext;
  a.out = (double2*)out_ext;
  dd_stencil_launch<MODE_PLAIN>(dd_stencil_kind(dd), sh, a, ctx->stream, ctx->num_sms);
  SCH_LAUNCHED(ctx);
  return SCH_OK;
}

int sch_dd_cg_normal(sch_ctx* ctx, sch_dd* dd, const double* U_ext, double* b_ext, double* x_ext,
                     double* x0_ext, double m0, double tol, int maxiter, int* h_iters,
                     double* h_relres, int* h_status) {
  SCH_CHECK_ARG(ctx, dd && U_ext && b_ext && x_ext && maxiter >= 1, "dd_cg_normal: bad args");
  SCH_CHECK_ARG(ctx, x_ext != b_ext && x_ext != x0_ext, "dd_cg_normal: x aliases an input");
  SCH_CHECK_ARG(ctx, dd->T % 8 == 0, "dd_cg_normal: T must be a multiple of 8");
  TileShape sh;
  dd_tile_shape(dd->Lext, dd->T, sh);
  const long long nsites = (long long)dd->S * dd->Lext * dd->T;
  const size_t vec = (size_t)nsites * 2 * sizeof(double2);
  const int skind = dd_stencil_kind(dd);
  const int nch_s = dd_stencil_nch(dd, skind);              // chunks per row of the stencil pass (0: NC)
  const int nch_p = nch_s ? nch_s : dd->NC;
  const size_t npart = (size_t)dd->S * dd->Lloc * std::max(dd->NC, nch_p);   // row partials
  const size_t bytes = 3 * vec + sizeof(double) * (2 * npart + SC_COUNT + dd->S + 64) +
                       sizeof(int) * (dd->S + 8) + 8 * 256;
  void* ws;
  int rc = sch_workspace(ctx, bytes, &ws);
  if (rc) return rc;
  char* w = (char*)ws;
  auto take = [&](size_t n) {
    char* p = w;
    w += (n + 255) & ~size_t(255);
    return (void*)p;
  };
  double2* r = (double2*)take(vec);
  double2* p = (double2*)take(vec);
  double2* ap = (double2*)take(vec);
  double* part_a = (double*)take(sizeof(double) * npart);
  double* part_b = (double*)take(sizeof(double) * npart);
  DDState st;
  st.sc = (double*)take(sizeof(double) * SC_COUNT);
  st.beta = (double*)take(sizeof(double) * dd->S);
  st.flag = (int*)take(sizeof(int) * dd->S);
  st.ctl = (int*)take(sizeof(int) * 8);
  cudaStream_t s = ctx->stream;
  const int lo = kHalo, hi = kHalo + dd->Lloc;
  const unsigned egrid = chunk_grid((long long)dd->S * dd->Lext * dd->NC);   // warp-per-chunk passes

  // init: b (and x0) halos, then x, r, p on every row
  if ((rc = dd_exchange(ctx, dd, b_ext, 1, 4))) return rc;
  if (x0_ext && (rc = dd_exchange(ctx, dd, x0_ext, 1, 4))) return rc;
  k_dd_init<<<egrid, 256, 0, s>>>((const double2*)b_ext, (const double2*)x0_ext, (double2*)x_ext, r, p,
                                  dd->S, dd->Lext, dd->T, dd->CW, lo, hi, part_a);
  SCH_LAUNCHED(ctx);
  if ((rc = dd_allsum(ctx, dd, part_a, st.sc + SC_NORMB2))) return rc;
  TileArgs base = dd_tile_args(dd, sh, (const double2*)U_ext, m0);
  if (x0_ext) {   // r = b - A x0 on own rows, then p = r, both with fresh halos
    TileArgs tx = base;
    tx.in = (const double2*)x_ext;
    tx.bvec = (const double2*)b_ext;
    tx.out = r;
    tx.rowpart = part_b;
    dd_stencil_launch<MODE_X>(skind, sh, tx, s, ctx->num_sms);
    SCH_LAUNCHED(ctx);
    if ((rc = dd_allsum(ctx, dd, part_b, st.sc + SC_RR, DDPost{}, nch_s))) return rc;
    if ((rc = dd_exchange(ctx, dd, (double*)r, 1, 4))) return rc;
    k_dd_copy<<<egrid, 256, 0, s>>>(r, p, nsites);
    SCH_LAUNCHED(ctx);
  }
  k_dd_ctrl_init<<<1, 1, 0, s>>>(st, dd->S, tol, x0_ext != nullptr);
  SCH_LAUNCHED(ctx);

  TileArgs tp = base;   // stencil pass: p = r + beta p formed on the fly
  tp.in = r;
  tp.in2 = p;
  tp.out = ap;
  tp.beta = st.beta;
  tp.rowpart = part_a;
  TileArgs txx = base;  // true residual / replacement pass
  txx.in = (const double2*)x_ext;
  txx.bvec = (const double2*)b_ext;
  txx.out = r;
  txx.flag = st.flag;
  txx.rowpart = part_b;

  // One iteration; the iteration number lives on the device (ctl[3]), so the
  // body is the same every time and can be captured.
  auto post = [&](int kind, cudaGraphConditionalHandle h = 0) {
    DDPost p;
    p.kind = kind;
    p.st = st;
    p.S = dd->S;
    p.maxiter = maxiter;
    p.set_cond = h != 0;
    p.h = h;
    return p;
  };
  auto iteration = [&](cudaStream_t q, cudaGraphConditionalHandle h) -> int {
    const cudaStream_t saved = ctx->stream;
    ctx->stream = q;   // dd_exchange / dd_allsum enqueue on ctx->stream
    int e = SCH_OK;
    do {
      if ((e = dd_exchange(ctx, dd, (double*)r, 1, 4))) break;
      dd_stencil_launch<MODE_P>(skind, sh, tp, q, ctx->num_sms);
      ctx->launches++;
      if ((e = dd_allsum(ctx, dd, part_a, st.sc + SC_PAP, post(POST_ALPHA), nch_s))) break;
      k_dd_update<<<egrid, 256, 0, q>>>(r, p, (double2*)x_ext, ap, st, dd->S, dd->Lext, dd->T, dd->CW,
                                        lo, hi, part_b);
      ctx->launches++;
      if ((e = dd_allsum(ctx, dd, part_b, st.sc + SC_RR, post(POST_CHECK)))) break;
      // x halos are current (x is updated on every row), so no exchange here
      dd_stencil_launch<MODE_X>(skind, sh, txx, q, ctx->num_sms);
      ctx->launches++;
      // the final control also advances the iteration and, inside the WHILE
      // graph, sets the loop condition
      if ((e = dd_allsum(ctx, dd, part_b, st.sc + SC_TN2, post(POST_FINAL, h), nch_s, st.flag)))
        break;
      cudaError_t le = cudaGetLastError();
      if (le != cudaSuccess) e = sch_fail(ctx, SCH_ERR_CUDA, "dd cg launch: %s", cudaGetErrorString(le));
    } while (0);
    ctx->stream = saved;
    return e;
  };

  if (dd->comm == nullptr && use_cg_graph() && use_cg_while()) {
    // local and p2p transports: the whole loop on the device (conditional
    // WHILE graph node, as the streaming engine in cg.cu; the p2p kernels
    // keep their sequence numbers on the device); the NCCL transport keeps
    // the host-driven loop below
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
    int e = iteration(ctx->cap_stream, handle);
    cudaGraph_t captured;
    cudaError_t ce = cudaStreamEndCapture(ctx->cap_stream, &captured);
    if (e || ce != cudaSuccess) {
      cudaGraphDestroy(graph);
      return e ? e : sch_fail(ctx, SCH_ERR_CUDA, "dd cg capture: %s", cudaGetErrorString(ce));
    }
    cudaGraphExec_t exec;
    cudaError_t ie = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ie != cudaSuccess) return sch_fail(ctx, SCH_ERR_CUDA, "dd cg instantiate: %s", cudaGetErrorString(ie));
    cudaError_t le = cudaGraphLaunch(exec, s);
    cudaGraphExecDestroy(exec);
    if (le != cudaSuccess) return sch_fail(ctx, SCH_ERR_CUDA, "dd cg graph launch: %s", cudaGetErrorString(le));
  } else {
    int it = 1, chunk = 4;
    while (it <= maxiter) {
      const int n = std::min(chunk, maxiter - it + 1);
      for (int j = 0; j < n; ++j, ++it)
        if ((rc = iteration(s, 0))) return rc;
      SCH_CUDA(ctx, cudaMemcpyAsync(ctx->h_flag, st.ctl, sizeof(int), cudaMemcpyDeviceToHost, s));
      SCH_CUDA(ctx, cudaStreamSynchronize(s));
      if (*ctx->h_flag) break;
      chunk = std::min(chunk * 2, 32);
    }
  }
  int ctl[3];
  double relres;
  SCH_CUDA(ctx, cudaMemcpyAsync(ctl, st.ctl, sizeof(ctl), cudaMemcpyDeviceToHost, s));
  SCH_CUDA(ctx, cudaMemcpyAsync(&relres, st.sc + SC_RELRES, sizeof(double), cudaMemcpyDeviceToHost, s));
  SCH_CUDA(ctx, cudaStreamSynchronize(s));
  if (ctl[1] == 0 && ctl[0]) {   // zero rhs: x = 0
    SCH_CUDA(ctx, cudaMemsetAsync(x_ext, 0, vec, s));
  }
  if (h_iters) *h_iters = ctl[1];
  if (h_relres) *h_relres = relres;
  if (h_status) *h_status = ctl[2];
  return ctl[2] ? sch_fail(ctx, SCH_ERR_SOLVER, "CG exceeded %d iterations", maxiter) : SCH_OK;
}

}  // extern "C"
