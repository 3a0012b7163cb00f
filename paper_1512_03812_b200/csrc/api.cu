// Context management for the C-ABI (include/schwinger_sm100.h).
#include "runtime.hpp"
#include "../../include/schwinger_sm100.h"

extern "C" {

int sch_ctx_create(int device, sch_ctx** out) {
  if (!out) return SCH_ERR_ARG;
  *out = nullptr;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) return SCH_ERR_CUDA;
  if (device < 0 || device >= n) return SCH_ERR_ARG;
  if (cudaSetDevice(device) != cudaSuccess) return SCH_ERR_CUDA;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return SCH_ERR_CUDA;
  if (prop.major != 10) return SCH_ERR_CUDA;   // built for sm_100a only
  sch_ctx* c = new sch_ctx();
  c->device = device;
  c->num_sms = prop.multiProcessorCount;
  if (cudaMallocHost(&c->h_flag, sizeof(int)) != cudaSuccess) {
    delete c;
    return SCH_ERR_CUDA;
  }
  *out = c;
  return SCH_OK;
}

int sch_ctx_destroy(sch_ctx* c) {
  if (!c) return SCH_OK;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  else cudaDeviceSynchronize();
  for (auto& g : c->graphs) cudaGraphExecDestroy(g.exec);
  if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
  if (c->ws) cudaFree(c->ws);
  if (c->h_flag) cudaFreeHost(c->h_flag);
  delete c;
  return SCH_OK;
}

int sch_set_stream(sch_ctx* c, void* stream) {
  if (!c) return SCH_ERR_ARG;
  c->stream = (cudaStream_t)stream;
  return SCH_OK;
}

const char* sch_last_error(const sch_ctx* c) { return c ? c->last_error.c_str() : "null context"; }

unsigned long long sch_launch_count(const sch_ctx* c) { return c ? c->launches : 0ULL; }

#define SCH_STR2(x) #x
#define SCH_STR(x) SCH_STR2(x)
const char* sch_build_info(void) {
  return "schwinger_sm100 sm_100a fp64 nvcc " SCH_STR(__CUDACC_VER_MAJOR__) "." SCH_STR(
      __CUDACC_VER_MINOR__);
}

}  // extern "C"
