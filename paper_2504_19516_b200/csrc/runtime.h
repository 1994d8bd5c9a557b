// Host-side runtime support shared by the C-ABI entry points: error state,
// driver entry points resolved at run time (so the .so has no libcuda link
// dependency and loads on a GPU-less host), and a tensor-map cache.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <utility>

#include "../../include/hp.h"

namespace hp {

// ---- error handling: every C entry point returns 0 or a negative code and
// leaves a message retrievable with hp_last_error().

int set_error(int code, const std::string& msg);
const char* last_error();

#define HP_CHECK_ARG(cond, msg)                                  \
  do {                                                           \
    if (!(cond)) return ::hp::set_error(HP_ERR_INVALID, msg); \
  } while (0)

#define HP_CUDA_TRY(expr)                                                            \
  do {                                                                               \
    cudaError_t _e = (expr);                                                         \
    if (_e != cudaSuccess)                                                           \
      return ::hp::set_error(HP_ERR_CUDA, std::string(#expr ": ") + cudaGetErrorString(_e)); \
  } while (0)

#define HP_LAUNCH_CHECK(name)                                                        \
  do {                                                                               \
    cudaError_t _e = cudaGetLastError();                                             \
    if (_e != cudaSuccess)                                                           \
      return ::hp::set_error(HP_ERR_CUDA, std::string(name ": ") + cudaGetErrorString(_e)); \
  } while (0)

// ---- driver API (resolved lazily through cudaGetDriverEntryPoint)
struct Driver {
  bool loaded = false;
  decltype(&::cuTensorMapEncodeTiled) tensorMapEncodeTiled = nullptr;
  decltype(&::cuDeviceGetDevResource) deviceGetDevResource = nullptr;
  decltype(&::cuDevSmResourceSplitByCount) devSmResourceSplitByCount = nullptr;
  decltype(&::cuDevResourceGenerateDesc) devResourceGenerateDesc = nullptr;
  decltype(&::cuGreenCtxCreate) greenCtxCreate = nullptr;
  decltype(&::cuGreenCtxDestroy) greenCtxDestroy = nullptr;
  decltype(&::cuGreenCtxStreamCreate) greenCtxStreamCreate = nullptr;
  decltype(&::cuStreamDestroy) streamDestroy = nullptr;
  decltype(&::cuDeviceGet) deviceGet = nullptr;
  decltype(&::cuGetErrorString) getErrorString = nullptr;
  decltype(&::cuMemGetAddressRange) memGetAddressRange = nullptr;
};

// Returns nullptr (with hp_last_error set) when the driver is unavailable.
const Driver* driver();
std::string cu_error_string(CUresult r);

// 2-D bf16 row-major tensor map: rows x cols, row pitch `ld` elements,
// box = box_rows x box_cols (box_cols * 2 bytes must be 128 for SW128).
int make_tmap_bf16(CUtensorMap* out, const void* base, uint64_t rows, uint64_t cols, uint64_t ld,
                   uint32_t box_rows, uint32_t box_cols, bool swizzle128);

// Cached variant keyed on all arguments (pointers and shapes are stable
// across steps for weights and persistent activation buffers).
int cached_tmap_bf16(CUtensorMap* out, const void* base, uint64_t rows, uint64_t cols,
                     uint64_t ld, uint32_t box_rows, uint32_t box_cols, bool swizzle128);

int device_sm_count();

// Development aid: per-kernel trace buffers (hp_set_trace); nullptr = off.
enum { TRACE_FA = 0, TRACE_SWAP = 1, TRACE_CTAS = 2, TRACE_KINDS = 3 };
void* trace_buf(int kind);
// TRACE_CTAS is one-shot: the next prefill GEMM / attention launch takes
// the armed buffer (per-CTA {smid, start_ns, end_ns}) and disarms it.
uint64_t* take_cta_trace();

// Stream-K tail of the prefill CTA-pair GEMM (hp_set_gemm_tail; default
// on unless HP_GEMM_TAIL=0): 1 = split the last partial wave of tiles along
// K over all pairs, 0 = plain persistent rounds (wave_stats rounds).
int gemm_tail_mode();
// Per-stream workspace: SK_MAX_PAIRS partial-tile slots of SK_SLOT_FLOATS
// fp32 (a 256 x 256 accumulator, both CTAs' halves) + [pairs][2] arrival
// counters for up to 2 * SK_MAX_PAIRS tail tiles (zero between launches:
// the finishing CTA resets its counter).
constexpr int SK_MAX_PAIRS = 80;
constexpr int SK_SLOT_FLOATS = 256 * 256;
struct SkWorkspace {
  float* ws;
  int* cnt;
};
int sk_workspace(cudaStream_t st, SkWorkspace* out);

// PDL on unless the environment sets HP_PDL=0 (A/B measurement).
bool pdl_enabled();

// Launch with programmatic dependent launch (PDL) enabled: the kernel may
// start while its stream predecessor is still finishing; it must call
// pdl_wait() (griddepcontrol.wait) before touching any memory the
// predecessor chain produces or consumes.  Hides the launch latency and the
// prologue (barrier init, TMEM alloc, descriptor prefetch, weight prefetch)
// of every layer kernel behind the previous kernel's tail.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

#define HP_LAUNCH_PDL(name, ...)                                                     \
  do {                                                                               \
    cudaError_t _e = ::hp::launch_pdl(__VA_ARGS__);                                  \
    if (_e != cudaSuccess)                                                           \
      return ::hp::set_error(HP_ERR_CUDA, std::string(name ": ") + cudaGetErrorString(_e)); \
  } while (0)

}  // namespace hp
