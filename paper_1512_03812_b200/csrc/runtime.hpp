// Host-side runtime for the C-ABI: context, stream, workspace arena, error
// state and launch accounting.  Not part of the public header.
#pragma once

#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

struct sch_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;   // borrowed (torch's current stream) or 0
  std::string last_error;
  unsigned long long launches = 0; // kernels this context launched
  int num_sms = 148;
  // workspace arena: grown on demand, reused across calls, freed on destroy
  void* ws = nullptr;
  size_t ws_bytes = 0;
  // pinned host scalar for streaming-CG termination polls
  int* h_flag = nullptr;
  // private non-blocking stream for CUDA-graph capture (the caller's stream
  // may be the legacy default stream, which cannot be captured)
  cudaStream_t cap_stream = nullptr;
  // CUDA-graph cache for the streaming CG chunk
  struct GraphEntry {
    std::vector<long long> key;
    cudaGraphExec_t exec = nullptr;
  };
  std::vector<GraphEntry> graphs;
};

enum sch_status {
  SCH_OK = 0,
  SCH_ERR_ARG = 1,
  SCH_ERR_CUDA = 2,
  SCH_ERR_SOLVER = 3,
};

inline int sch_fail(sch_ctx* c, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  if (c) c->last_error = buf;
  return code;
}

#define SCH_CUDA(ctx, expr)                                                             \
  do {                                                                                  \
    cudaError_t _e = (expr);                                                            \
    if (_e != cudaSuccess)                                                              \
      return sch_fail((ctx), SCH_ERR_CUDA, "%s:%d %s: %s", __FILE__, __LINE__, #expr,   \
                      cudaGetErrorString(_e));                                          \
  } while (0)

#define SCH_LAUNCHED(ctx)                                                               \
  do {                                                                                  \
    cudaError_t _e = cudaGetLastError();                                                \
    if (_e != cudaSuccess)                                                              \
      return sch_fail((ctx), SCH_ERR_CUDA, "%s:%d launch: %s", __FILE__, __LINE__,      \
                      cudaGetErrorString(_e));                                          \
    (ctx)->launches++;                                                                  \
  } while (0)

#define SCH_CHECK_ARG(ctx, cond, msg)                                                   \
  do {                                                                                  \
    if (!(cond)) return sch_fail((ctx), SCH_ERR_ARG, "%s", msg);                         \
  } while (0)

// Grab `bytes` of device workspace (256-B aligned), growing the arena if needed.
inline int sch_workspace(sch_ctx* c, size_t bytes, void** out) {
  bytes = (bytes + 255) & ~size_t(255);
  if (bytes > c->ws_bytes) {
    if (c->ws) {
      cudaError_t e = cudaStreamSynchronize(c->stream);
      if (e != cudaSuccess) return sch_fail(c, SCH_ERR_CUDA, "ws sync: %s", cudaGetErrorString(e));
      cudaFree(c->ws);
      c->ws = nullptr;
      c->ws_bytes = 0;
      for (auto& g : c->graphs) cudaGraphExecDestroy(g.exec);
      c->graphs.clear();
    }
    cudaError_t e = cudaMalloc(&c->ws, bytes);
    if (e != cudaSuccess)
      return sch_fail(c, SCH_ERR_CUDA, "workspace alloc %zu B: %s", bytes, cudaGetErrorString(e));
    c->ws_bytes = bytes;
  }
  *out = c->ws;
  return SCH_OK;
}

inline unsigned blocks_for(long n, int nt) { return (unsigned)((n + nt - 1) / nt); }

// Streaming-CG kernels are launched with programmatic stream serialization
// (common.cuh pdl_enter) so each one's launch overlaps its predecessor's
// tail; SCH_NO_PDL=1 launches them plainly.
inline bool use_pdl() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SCH_NO_PDL");
    v = (e && e[0] == '1') ? 0 : 1;
  }
  return v == 1;
}

template <typename... KArgs, typename... Args>
inline void launch_k(bool pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                     cudaStream_t st, Args... args) {
  if (!pdl) {
    kern<<<grid, block, smem, st>>>(args...);
    return;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, args...);   // errors surface through cudaGetLastError
}

// The TMA-pipelined stencil is the default where its tile shapes apply;
// SCH_NO_TMA=1 selects the plain per-tile kernels (A/B measurements).
inline bool use_tma() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SCH_NO_TMA");
    v = (e && e[0] == '1') ? 0 : 1;
  }
  return v == 1;
}

// The streaming CG replays captured chunks of iterations as a CUDA graph;
// SCH_NO_CG_GRAPH=1 launches every kernel from the host instead.
inline bool use_cg_graph() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SCH_NO_CG_GRAPH");
    v = (e && e[0] == '1') ? 0 : 1;
  }
  return v == 1;
}

// The streaming CG runs its loop on the device through a conditional WHILE
// graph node; SCH_CG_WHILE=0 replays fixed chunks with host polling instead.
inline bool use_cg_while() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SCH_CG_WHILE");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

