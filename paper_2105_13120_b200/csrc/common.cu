// Host plumbing: error reporting, TMA descriptor encoding, device queries.
#include <cudaTypedefs.h>

#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>

#include "common.h"

namespace rsa {

static thread_local char g_err[512] = "";

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(RSA_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return RSA_OK;
}

static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
static std::once_flag g_encode_once;

static void load_encode() {
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
      q == cudaDriverEntryPointSuccess)
    g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
}

bool encode_tmap(CUtensorMap* out, CUtensorMapDataType dtype, int rank, const void* base, const uint64_t* dims,
                 const uint64_t* strides_bytes, const uint32_t* box, CUtensorMapSwizzle swizzle) {
  std::call_once(g_encode_once, load_encode);
  if (!g_encode) {
    fail(RSA_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
    return false;
  }
  cuuint64_t gdim[5];
  cuuint64_t gstr[4];
  cuuint32_t bdim[5];
  cuuint32_t estr[5];
  for (int i = 0; i < rank; ++i) {
    gdim[i] = dims[i];
    bdim[i] = box[i];
    estr[i] = 1;
    if (i + 1 < rank) gstr[i] = strides_bytes[i];
  }
  CUresult r = g_encode(out, dtype, rank, const_cast<void*>(base), gdim, gstr, bdim, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    char buf[256];
    int n = snprintf(buf, sizeof(buf), "cuTensorMapEncodeTiled failed (%d): rank %d dims", int(r), rank);
    for (int i = 0; i < rank && n < 200; ++i) n += snprintf(buf + n, sizeof(buf) - n, " %llu", (unsigned long long)dims[i]);
    fail(RSA_ERR_UNSUPPORTED, "%s", buf);
    return false;
  }
  return true;
}

int num_sms() {
  static int cached = 0;
  if (!cached) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev);
  }
  return cached;
}

static int g_max_ctas = 0;  // 0: one CTA per SM (rsa_set_max_ctas)

int persistent_grid(int64_t items) {
  int64_t grid = num_sms();
  if (g_max_ctas > 0 && g_max_ctas < grid) grid = g_max_ctas;
  return int(items < grid ? items : grid);
}

}  // namespace rsa

extern "C" {

int rsa_abi_version(void) { return RSA_ABI_VERSION; }
const char* rsa_last_error(void) { return rsa::g_err; }
int rsa_num_sms(void) { return rsa::num_sms(); }

int rsa_set_max_ctas(int max_ctas) {
  const int prev = rsa::g_max_ctas;
  rsa::g_max_ctas = max_ctas > 0 ? max_ctas : 0;
  return prev;
}

int rsa_ipc_alloc(size_t bytes, void** ptr, void* handle) {
  if (!ptr || !handle || !bytes) return rsa::fail(RSA_ERR_INVALID, "rsa_ipc_alloc: null argument or zero size");
  *ptr = nullptr;
  cudaError_t e = cudaMalloc(ptr, bytes);
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(reinterpret_cast<cudaIpcMemHandle_t*>(handle), *ptr);
  if (e != cudaSuccess) {
    if (*ptr) cudaFree(*ptr), *ptr = nullptr;
    return rsa::fail(RSA_ERR_CUDA, "rsa_ipc_alloc: %s", cudaGetErrorString(e));
  }
  return RSA_OK;
}

int rsa_ipc_open(const void* handle, void** ptr) {
  if (!ptr || !handle) return rsa::fail(RSA_ERR_INVALID, "rsa_ipc_open: null argument");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  const cudaError_t e = cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess);
  return e == cudaSuccess ? RSA_OK : rsa::fail(RSA_ERR_CUDA, "rsa_ipc_open: %s", cudaGetErrorString(e));
}

int rsa_ipc_close(void* ptr) {
  const cudaError_t e = cudaIpcCloseMemHandle(ptr);
  return e == cudaSuccess ? RSA_OK : rsa::fail(RSA_ERR_CUDA, "rsa_ipc_close: %s", cudaGetErrorString(e));
}

int rsa_ipc_free(void* ptr) {
  const cudaError_t e = cudaFree(ptr);
  return e == cudaSuccess ? RSA_OK : rsa::fail(RSA_ERR_CUDA, "rsa_ipc_free: %s", cudaGetErrorString(e));
}

}  // extern "C"
