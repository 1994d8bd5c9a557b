#include "runtime.h"

#include <cstdlib>

#include <cstring>
#include <map>
#include <mutex>
#include <unordered_map>

namespace hp {

static thread_local std::string g_last_error;

int set_error(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

const char* last_error() { return g_last_error.c_str(); }

static Driver g_driver;
static std::once_flag g_driver_once;
static std::string g_driver_error;

template <typename F>
static bool resolve(const char* name, F& fn) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaError_t e = cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q);
  if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || p == nullptr) {
    g_driver_error = std::string("driver entry point unavailable: ") + name;
    cudaGetLastError();
    return false;
  }
  fn = reinterpret_cast<F>(p);
  return true;
}

const Driver* driver() {
  std::call_once(g_driver_once, [] {
    bool ok = true;
    ok &= resolve("cuTensorMapEncodeTiled", g_driver.tensorMapEncodeTiled);
    ok &= resolve("cuDeviceGetDevResource", g_driver.deviceGetDevResource);
    ok &= resolve("cuDevSmResourceSplitByCount", g_driver.devSmResourceSplitByCount);
    ok &= resolve("cuDevResourceGenerateDesc", g_driver.devResourceGenerateDesc);
    ok &= resolve("cuGreenCtxCreate", g_driver.greenCtxCreate);
    ok &= resolve("cuGreenCtxDestroy", g_driver.greenCtxDestroy);
    ok &= resolve("cuGreenCtxStreamCreate", g_driver.greenCtxStreamCreate);
    ok &= resolve("cuStreamDestroy", g_driver.streamDestroy);
    ok &= resolve("cuDeviceGet", g_driver.deviceGet);
    ok &= resolve("cuGetErrorString", g_driver.getErrorString);
    ok &= resolve("cuMemGetAddressRange", g_driver.memGetAddressRange);
    g_driver.loaded = ok;
  });
  if (!g_driver.loaded) {
    set_error(HP_ERR_NO_DEVICE, g_driver_error.empty() ? "CUDA driver unavailable" : g_driver_error);
    return nullptr;
  }
  return &g_driver;
}

std::string cu_error_string(CUresult r) {
  const char* s = nullptr;
  if (g_driver.getErrorString) g_driver.getErrorString(r, &s);
  return s ? std::string(s) : ("CUresult " + std::to_string(int(r)));
}

int make_tmap_bf16(CUtensorMap* out, const void* base, uint64_t rows, uint64_t cols, uint64_t ld,
                   uint32_t box_rows, uint32_t box_cols, bool swizzle128) {
  const Driver* d = driver();
  if (!d) return HP_ERR_NO_DEVICE;
  HP_CHECK_ARG(base != nullptr, "tensor map: null base pointer");
  HP_CHECK_ARG((reinterpret_cast<uintptr_t>(base) & 15) == 0, "tensor map: base not 16B aligned");
  HP_CHECK_ARG((ld * 2) % 16 == 0, "tensor map: row pitch must be a multiple of 16 bytes");
  HP_CHECK_ARG(box_rows >= 1 && box_rows <= 256 && box_cols >= 1 && box_cols <= 256,
               "tensor map: box out of range");
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = d->tensorMapEncodeTiled(
      out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
      CU_TENSOR_MAP_INTERLEAVE_NONE,
      swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(HP_ERR_CUDA, "cuTensorMapEncodeTiled: " + cu_error_string(r));
  return HP_OK;
}

namespace {
struct TmapKey {
  const void* base;
  uint64_t rows, cols, ld;
  uint32_t box_rows, box_cols;
  bool sw;
  bool operator==(const TmapKey& o) const {
    return base == o.base && rows == o.rows && cols == o.cols && ld == o.ld &&
           box_rows == o.box_rows && box_cols == o.box_cols && sw == o.sw;
  }
};
struct TmapKeyHash {
  size_t operator()(const TmapKey& k) const {
    size_t h = std::hash<const void*>()(k.base);
    h ^= std::hash<uint64_t>()(k.rows * 1000003u + k.cols) + 0x9e3779b9 + (h << 6) + (h >> 2);
    h ^= std::hash<uint64_t>()(k.ld * 131u + k.box_rows * 7u + k.box_cols + (k.sw ? 1 : 0)) +
         0x9e3779b9 + (h << 6) + (h >> 2);
    return h;
  }
};
std::mutex g_tmap_mu;
std::unordered_map<TmapKey, CUtensorMap, TmapKeyHash> g_tmap_cache;
}  // namespace

int cached_tmap_bf16(CUtensorMap* out, const void* base, uint64_t rows, uint64_t cols,
                     uint64_t ld, uint32_t box_rows, uint32_t box_cols, bool swizzle128) {
  TmapKey key{base, rows, cols, ld, box_rows, box_cols, swizzle128};
  {
    std::lock_guard<std::mutex> lk(g_tmap_mu);
    auto it = g_tmap_cache.find(key);
    if (it != g_tmap_cache.end()) {
      *out = it->second;
      return HP_OK;
    }
  }
  int rc = make_tmap_bf16(out, base, rows, cols, ld, box_rows, box_cols, swizzle128);
  if (rc != HP_OK) return rc;
  std::lock_guard<std::mutex> lk(g_tmap_mu);
  if (g_tmap_cache.size() > 4096) g_tmap_cache.clear();
  g_tmap_cache.emplace(key, *out);
  return HP_OK;
}

static void* g_trace[TRACE_KINDS] = {nullptr, nullptr, nullptr};
static int g_gemm_tail = -1;  // -1: HP_GEMM_TAIL environment default
void* trace_buf(int kind) { return g_trace[kind]; }
uint64_t* take_cta_trace() {
  void* b = g_trace[TRACE_CTAS];
  g_trace[TRACE_CTAS] = nullptr;
  return static_cast<uint64_t*>(b);
}

}  // namespace hp

extern "C" int hp_set_trace(int kind, void* buf) {
  HP_CHECK_ARG(kind >= 0 && kind < hp::TRACE_KINDS, "hp_set_trace: unknown kind");
  hp::g_trace[kind] = buf;
  return HP_OK;
}

namespace hp {

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("HP_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

int device_sm_count() {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
  return n;
}

int gemm_tail_mode() {
  static const int env = [] {
    const char* e = std::getenv("HP_GEMM_TAIL");
    return (e && e[0] == '0') ? 0 : 1;
  }();
  return g_gemm_tail < 0 ? env : g_gemm_tail;
}

// One stream-K workspace per stream: launches on one stream are ordered, so
// they may share it; two streams running prefill GEMMs at once must not.
// Never freed (a captured graph may hold the pointers).
static std::mutex g_sk_mu;
static std::map<cudaStream_t, SkWorkspace> g_sk;

int sk_workspace(cudaStream_t st, SkWorkspace* out) {
  std::lock_guard<std::mutex> lk(g_sk_mu);
  auto it = g_sk.find(st);
  if (it != g_sk.end()) {
    *out = it->second;
    return HP_OK;
  }
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone)
    return set_error(HP_ERR_CUDA, "stream-K workspace: first use may not be inside a capture");
  SkWorkspace w{};
  HP_CUDA_TRY(cudaMalloc(&w.ws, size_t(SK_MAX_PAIRS) * SK_SLOT_FLOATS * sizeof(float)));
  HP_CUDA_TRY(cudaMalloc(&w.cnt, size_t(SK_MAX_PAIRS) * 4 * sizeof(int)));
  HP_CUDA_TRY(cudaMemsetAsync(w.cnt, 0, size_t(SK_MAX_PAIRS) * 4 * sizeof(int), st));  // ordered before use
  g_sk.emplace(st, w);
  *out = w;
  return HP_OK;
}

}  // namespace hp

extern "C" int hp_gemm_tail_reserve(void* stream) {
  hp::SkWorkspace w{};
  return hp::sk_workspace(static_cast<cudaStream_t>(stream), &w);
}

extern "C" int hp_set_gemm_tail(int mode) {
  HP_CHECK_ARG(mode >= -1 && mode <= 1, "hp_set_gemm_tail: mode must be -1, 0 or 1");
  hp::g_gemm_tail = mode;
  return HP_OK;
}
