// Runtime entry points of the C ABI: device queries, wave accounting, the
// green-context SM partition manager and the per-CTA probe kernel.
#include "common.cuh"
#include "runtime.h"
#include "../../include/hp.h"

#include <cstring>
#include <new>
#include <string>

using namespace hp;

extern "C" int hp_abi_version(void) { return HP_ABI_VERSION; }

extern "C" const char* hp_last_error(void) { return hp::last_error(); }

extern "C" int hp_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

extern "C" int hp_device_sms(int device, int* sms) {
  HP_CHECK_ARG(sms != nullptr, "hp_device_sms: null output");
  if (hp_device_count() <= device || device < 0)
    return set_error(HP_ERR_NO_DEVICE, "hp_device_sms: no such CUDA device");
  HP_CUDA_TRY(cudaDeviceGetAttribute(sms, cudaDevAttrMultiProcessorCount, device));
  return HP_OK;
}

// perf_model.py:157-169 -- identical integer arithmetic (ceil division on
// exact ints) and the same single IEEE double division for the idle ratio.
extern "C" int hp_wave_stats(int64_t g, int64_t b, int64_t n, int64_t* waves, int64_t* tail_sms,
                             double* idle_ratio) {
  if (g < 1 || b < 1 || n < 1)
    return set_error(HP_ERR_INVALID, "wave_stats requires positive g, b, N (got " +
                                         std::to_string(g) + ", " + std::to_string(b) + ", " +
                                         std::to_string(n) + ")");
  HP_CHECK_ARG(waves && tail_sms && idle_ratio, "hp_wave_stats: null output");
  const int64_t w = (g + b * n - 1) / (b * n);
  const int64_t rem = g - b * n * (w - 1);
  const int64_t tail = (rem + b - 1) / b;
  *waves = w;
  *tail_sms = tail;
  *idle_ratio = double(n - tail) / double(n * w);
  return HP_OK;
}

// ------------------------------------------------------------------ probe
__global__ void k_probe(uint64_t* out, int64_t spin_ns) {
  __shared__ uint64_t t0;
  if (threadIdx.x == 0) {
    t0 = globaltimer();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t now = t0;
    while (int64_t(now - t0) < spin_ns) now = globaltimer();
    out[blockIdx.x * 3 + 0] = smid();
    out[blockIdx.x * 3 + 1] = t0;
    out[blockIdx.x * 3 + 2] = now;
  }
}

extern "C" int hp_probe(int ctas, int threads, int64_t spin_ns, uint64_t* out, void* stream) {
  HP_CHECK_ARG(out != nullptr && ctas >= 1 && threads >= 1 && threads <= 1024, "hp_probe: bad arguments");
  k_probe<<<ctas, threads, 0, static_cast<cudaStream_t>(stream)>>>(out, spin_ns);
  HP_LAUNCH_CHECK("k_probe");
  return HP_OK;
}

// ------------------------------------------------------------- partitions
struct hp_partition {
  CUgreenCtx ctx[2] = {nullptr, nullptr};
  CUstream stream[2] = {nullptr, nullptr};
  int sms[2] = {0, 0};
};

static int destroy_partition(hp_partition* p) {
  const Driver* d = driver();
  if (!p) return HP_OK;
  if (d) {
    for (int i = 0; i < 2; ++i) {
      if (p->stream[i]) d->streamDestroy(p->stream[i]);
      if (p->ctx[i]) d->greenCtxDestroy(p->ctx[i]);
    }
  }
  delete p;
  return HP_OK;
}

extern "C" int hp_partition_create(int device, int decode_sms, hp_partition** out) {
  HP_CHECK_ARG(out != nullptr, "hp_partition_create: null output");
  *out = nullptr;
  const Driver* d = driver();
  if (!d) return HP_ERR_NO_DEVICE;
  if (hp_device_count() <= device || device < 0)
    return set_error(HP_ERR_NO_DEVICE, "hp_partition_create: no such CUDA device");
  HP_CUDA_TRY(cudaSetDevice(device));
  HP_CUDA_TRY(cudaFree(nullptr));  // make sure the primary context exists
  int total = 0;
  HP_CUDA_TRY(cudaDeviceGetAttribute(&total, cudaDevAttrMultiProcessorCount, device));
  HP_CHECK_ARG(decode_sms >= 8 && decode_sms % 8 == 0 && decode_sms < total,
               "hp_partition_create: decode_sms must be a multiple of 8 in [8, N)");
  CUdevice dev;
  CUresult r = d->deviceGet(&dev, device);
  if (r != CUDA_SUCCESS) return set_error(HP_ERR_CUDA, "cuDeviceGet: " + cu_error_string(r));
  CUdevResource all{};
  r = d->deviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM);
  if (r != CUDA_SUCCESS) return set_error(HP_ERR_CUDA, "cuDeviceGetDevResource: " + cu_error_string(r));
  CUdevResource grp{}, rem{};
  unsigned int ngroups = 1;
  r = d->devSmResourceSplitByCount(&grp, &ngroups, &all, &rem, 0, unsigned(decode_sms));
  if (r != CUDA_SUCCESS || ngroups != 1)
    return set_error(HP_ERR_CUDA, "cuDevSmResourceSplitByCount: " + cu_error_string(r));
  auto* p = new (std::nothrow) hp_partition();
  if (!p) return set_error(HP_ERR_CUDA, "hp_partition_create: out of host memory");
  CUdevResource* res[2] = {&rem, &grp};  // phase 0 = prefill (remainder), 1 = decode
  for (int i = 0; i < 2; ++i) {
    CUdevResourceDesc desc;
    r = d->devResourceGenerateDesc(&desc, res[i], 1);
    if (r != CUDA_SUCCESS) {
      destroy_partition(p);
      return set_error(HP_ERR_CUDA, "cuDevResourceGenerateDesc: " + cu_error_string(r));
    }
    r = d->greenCtxCreate(&p->ctx[i], desc, dev, CU_GREEN_CTX_DEFAULT_STREAM);
    if (r != CUDA_SUCCESS) {
      destroy_partition(p);
      return set_error(HP_ERR_CUDA, "cuGreenCtxCreate: " + cu_error_string(r));
    }
    r = d->greenCtxStreamCreate(&p->stream[i], p->ctx[i], CU_STREAM_NON_BLOCKING, 0);
    if (r != CUDA_SUCCESS) {
      destroy_partition(p);
      return set_error(HP_ERR_CUDA, "cuGreenCtxStreamCreate: " + cu_error_string(r));
    }
    p->sms[i] = int(res[i]->sm.smCount);
  }
  *out = p;
  return HP_OK;
}

extern "C" int hp_partition_stream(hp_partition* part, int phase, void** stream) {
  HP_CHECK_ARG(part && stream && (phase == 0 || phase == 1), "hp_partition_stream: bad arguments");
  *stream = part->stream[phase];
  return HP_OK;
}

extern "C" int hp_partition_sms(hp_partition* part, int phase, int* sms) {
  HP_CHECK_ARG(part && sms && (phase == 0 || phase == 1), "hp_partition_sms: bad arguments");
  *sms = part->sms[phase];
  return HP_OK;
}

extern "C" int hp_partition_destroy(hp_partition* part) { return destroy_partition(part); }

// CUDA IPC for the fused tensor-parallel all-reduce's symmetric buffers.
static_assert(sizeof(cudaIpcMemHandle_t) <= HP_IPC_HANDLE_BYTES, "IPC handle size");

// The handle names the whole cudaMalloc block; a caching allocator hands out
// sub-ranges, so the pointer's offset inside its block travels with it.
extern "C" int hp_ipc_handle(void* dev_ptr, void* handle_out, size_t* offset_out) {
  HP_CHECK_ARG(dev_ptr && handle_out && offset_out, "hp_ipc_handle: null pointer");
  const Driver* d = driver();
  if (!d) return HP_ERR_NO_DEVICE;
  CUdeviceptr base = 0;
  size_t size = 0;
  CUresult r = d->memGetAddressRange(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr));
  if (r != CUDA_SUCCESS) return set_error(HP_ERR_CUDA, "cuMemGetAddressRange: " + cu_error_string(r));
  cudaIpcMemHandle_t h;
  HP_CUDA_TRY(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  std::memset(handle_out, 0, HP_IPC_HANDLE_BYTES);
  std::memcpy(handle_out, &h, sizeof(h));
  *offset_out = size_t(reinterpret_cast<CUdeviceptr>(dev_ptr) - base);
  return HP_OK;
}

extern "C" int hp_ipc_open(const void* handle, void** base_out) {
  HP_CHECK_ARG(handle && base_out, "hp_ipc_open: null pointer");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  HP_CUDA_TRY(cudaIpcOpenMemHandle(base_out, h, cudaIpcMemLazyEnablePeerAccess));
  return HP_OK;
}

extern "C" int hp_ipc_close(void* dev_ptr) {
  HP_CHECK_ARG(dev_ptr, "hp_ipc_close: null pointer");
  HP_CUDA_TRY(cudaIpcCloseMemHandle(dev_ptr));
  return HP_OK;
}
