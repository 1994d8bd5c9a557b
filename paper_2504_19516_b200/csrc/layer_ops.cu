// Memory-bound layer glue: RMSNorm and RoPE + paged KV-cache write.
// Both are single-pass, 16-byte vectorised and grid-strided over a persistent
// grid sized to the partition (HBM-bound; no shared-memory staging needed).
#include "common.cuh"
#include "runtime.h"
#include "../../include/hp.h"

#include <algorithm>

namespace hp {

// One warp per row; cols % 256 == 0.  Two passes over the row (the second is
// an L1 hit): sum of squares, then scale and write.
__global__ void k_rmsnorm(const __nv_bfloat16* __restrict__ x, int ldx,
                          const __nv_bfloat16* __restrict__ w, __nv_bfloat16* __restrict__ out,
                          int ldo, int rows, int cols, float eps) {
  pdl_trigger();
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  for (int r = blockIdx.x * wpb + (threadIdx.x >> 5); r < rows; r += gridDim.x * wpb) {
    const uint4* xr = reinterpret_cast<const uint4*>(x + size_t(r) * ldx);
    float ss = 0.f;
    for (int c = lane; c < cols / 8; c += 32) {
      uint4 v = xr[c];
      const uint32_t* u = reinterpret_cast<const uint32_t*>(&v);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float a = bf16lo(u[k]), b = bf16hi(u[k]);
        ss += a * a + b * b;
      }
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
    const float inv = rsqrtf(ss / float(cols) + eps);
    const uint4* wr = reinterpret_cast<const uint4*>(w);
    uint4* orow = reinterpret_cast<uint4*>(out + size_t(r) * ldo);
    for (int c = lane; c < cols / 8; c += 32) {
      uint4 v = xr[c], g = wr[c], o;
      const uint32_t* u = reinterpret_cast<const uint32_t*>(&v);
      const uint32_t* gg = reinterpret_cast<const uint32_t*>(&g);
      uint32_t* oo = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
      for (int k = 0; k < 4; ++k)
        oo[k] = pack_bf16(bf16lo(u[k]) * inv * bf16lo(gg[k]), bf16hi(u[k]) * inv * bf16hi(gg[k]));
      orow[c] = o;
    }
  }
}

// Thread per (token, head, 2 rotary pairs).  q heads: rotate in place.
// k heads: rotate in place and write to the paged cache.  v heads: copy.
// Rotary convention (Llama / rotate_half): for i < d/2,
//   y[i] = x[i] cos - x[i+d/2] sin,  y[i+d/2] = x[i+d/2] cos + x[i] sin.
__global__ void k_rope_kv_write(__nv_bfloat16* __restrict__ qkv, int ld, int T, int Hq, int Hkv,
                                int d, const int* __restrict__ pos, const float* __restrict__ cs,
                                const int* __restrict__ slots, __nv_bfloat16* __restrict__ kc,
                                __nv_bfloat16* __restrict__ vc, int page) {
  pdl_trigger();
  pdl_wait();
  const int half = d / 2;
  const int pairs = half / 2;             // threads per head (2 rotary dims each)
  const int per_tok = (Hq + 2 * Hkv) * pairs;
  const long total = long(T) * per_tok;
  for (long idx = blockIdx.x * long(blockDim.x) + threadIdx.x; idx < total;
       idx += long(gridDim.x) * blockDim.x) {
    const int t = int(idx / per_tok);
    const int rem = int(idx % per_tok);
    const int head = rem / pairs;          // 0..Hq+2Hkv-1 across q | k | v blocks
    const int i = (rem % pairs) * 2;       // rotary dim pair start (< d/2)
    __nv_bfloat16* row = qkv + size_t(t) * ld + size_t(head) * d;
    const int slot = (head >= Hq) ? slots[t] : 0;
    const int blk = slot / page, off = slot % page;
    // cache page layout [page/64][d/64][64][64]: each 64-token tile of one
    // kv head is a contiguous 64*d run, 16B chunks swizzled by (token & 7)
    auto cidx = [&](int kvh, int j) -> size_t { return kv_cache_index(blk, Hkv, kvh, page, off, d, j); };
    if (head < Hq + Hkv) {
      const float* c = cs + size_t(pos[t]) * d;
      const float c0 = c[i], c1 = c[i + 1], s0 = c[half + i], s1 = c[half + i + 1];
      const uint32_t lo = *reinterpret_cast<const uint32_t*>(row + i);
      const uint32_t hi = *reinterpret_cast<const uint32_t*>(row + half + i);
      const float x0 = bf16lo(lo), x1 = bf16hi(lo), y0 = bf16lo(hi), y1 = bf16hi(hi);
      float a0, b0, a1, b1;
      rope_rotate(x0, y0, c0, s0, a0, b0);
      rope_rotate(x1, y1, c1, s1, a1, b1);
      const uint32_t nlo = pack_bf16(a0, a1);
      const uint32_t nhi = pack_bf16(b0, b1);
      *reinterpret_cast<uint32_t*>(row + i) = nlo;
      *reinterpret_cast<uint32_t*>(row + half + i) = nhi;
      if (head >= Hq) {
        const int kh = head - Hq;
        *reinterpret_cast<uint32_t*>(kc + cidx(kh, i)) = nlo;
        *reinterpret_cast<uint32_t*>(kc + cidx(kh, half + i)) = nhi;
      }
    } else {
      const int vh = head - Hq - Hkv;
      *reinterpret_cast<uint32_t*>(vc + cidx(vh, i)) = *reinterpret_cast<const uint32_t*>(row + i);
      *reinterpret_cast<uint32_t*>(vc + cidx(vh, half + i)) =
          *reinterpret_cast<const uint32_t*>(row + half + i);
    }
  }
}

// Row-major W [N, K] (row pitch ldw) -> tiled [N/128][K/128][2][128][64] with
// the SWIZZLE_128B chunk permutation; one thread per 16-byte chunk.
__global__ void k_tile_weight(const __nv_bfloat16* __restrict__ w, int ldw,
                              __nv_bfloat16* __restrict__ out, int N, int K) {
  const long chunks = long(N) * (K / 8);
  for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < chunks; i += long(gridDim.x) * blockDim.x) {
    const int r = int(i / (K / 8));
    const int c = int(i % (K / 8));
    const int kb = c >> 3, cc = c & 7, mb = r >> 7, rr = r & 127;
    const size_t dst = (((size_t(mb) * (K >> 7) + (kb >> 1)) * 2 + (kb & 1)) * 128 + rr) * 64 +
                       (size_t(cc ^ (rr & 7)) << 3);
    *reinterpret_cast<uint4*>(out + dst) = *reinterpret_cast<const uint4*>(w + size_t(r) * ldw + c * 8);
  }
}

// Strided row copy, 16-byte chunks, 4 independent chunks in flight per
// thread.  Either side may be pinned host memory (UVA-mapped): a decode
// step's B x hidden input / output cross PCIe through the decode
// partition's own SMs, inside its CUDA graph, instead of queueing on a copy
// engine behind the prefill side's multi-MB transfers.
__global__ void k_copy_rows(const uint8_t* __restrict__ src, long lds, uint8_t* __restrict__ dst, long ldd,
                            int rows, int row_bytes) {
  pdl_trigger();
  pdl_wait();
  const int per_row = row_bytes >> 4;
  const long total = long(rows) * per_row;
  const long stride = long(gridDim.x) * blockDim.x;
  for (long i0 = blockIdx.x * long(blockDim.x) + threadIdx.x; i0 < total; i0 += 4 * stride) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const long i = i0 + u * stride;
      if (i < total) v[u] = *reinterpret_cast<const uint4*>(src + (i / per_row) * lds + (i % per_row) * 16);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const long i = i0 + u * stride;
      if (i < total) *reinterpret_cast<uint4*>(dst + (i / per_row) * ldd + (i % per_row) * 16) = v[u];
    }
  }
}

}  // namespace hp

using namespace hp;

extern "C" int hp_copy_rows(const void* src, long lds_bytes, void* dst, long ldd_bytes, int rows, int row_bytes,
                            int max_ctas, void* stream) {
  HP_CHECK_ARG(src && dst, "hp_copy_rows: null pointer");
  HP_CHECK_ARG(rows >= 1 && row_bytes >= 16 && row_bytes % 16 == 0, "hp_copy_rows: row_bytes % 16");
  HP_CHECK_ARG(lds_bytes % 16 == 0 && ldd_bytes % 16 == 0 && lds_bytes >= row_bytes && ldd_bytes >= row_bytes,
               "hp_copy_rows: row pitches must be >= row_bytes and multiples of 16");
  HP_CHECK_ARG((reinterpret_cast<uintptr_t>(src) & 15) == 0 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0,
               "hp_copy_rows: pointers must be 16B aligned");
  HP_CHECK_ARG(max_ctas >= 1, "hp_copy_rows: max_ctas must be >= 1");
  const long total = long(rows) * (row_bytes / 16);
  const int threads = 256;
  const int grid = int(std::min<long>((total + 4 * threads - 1) / (4 * threads), long(max_ctas) * 4));
  HP_LAUNCH_PDL("k_copy_rows", k_copy_rows, dim3(grid), dim3(threads), 0, static_cast<cudaStream_t>(stream),
                static_cast<const uint8_t*>(src), lds_bytes, static_cast<uint8_t*>(dst), ldd_bytes, rows, row_bytes);
  return HP_OK;
}

extern "C" int hp_tile_weight(const void* w, int ldw, void* out, int N, int K, void* stream) {
  HP_CHECK_ARG(w && out && w != out, "hp_tile_weight: bad pointers (in place not supported)");
  HP_CHECK_ARG(N % 128 == 0 && K % 128 == 0 && ldw >= K && ldw % 8 == 0, "hp_tile_weight: N % 128, K % 128");
  const long chunks = long(N) * (K / 8);
  const int grid = int(std::min<long>((chunks + 255) / 256, 148L * 16));
  k_tile_weight<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const __nv_bfloat16*>(w), ldw, static_cast<__nv_bfloat16*>(out), N, K);
  HP_LAUNCH_CHECK("k_tile_weight");
  return HP_OK;
}

extern "C" int hp_rmsnorm(const void* x, int ldx, const void* weight, void* out, int ldo, int rows,
                          int cols, float eps, int max_ctas, void* stream) {
  HP_CHECK_ARG(x && weight && out, "hp_rmsnorm: null pointer");
  HP_CHECK_ARG(rows >= 1 && cols >= 8 && cols % 8 == 0, "hp_rmsnorm: cols must be a multiple of 8");
  HP_CHECK_ARG(ldx % 8 == 0 && ldo % 8 == 0, "hp_rmsnorm: row pitch must be a multiple of 8");
  HP_CHECK_ARG(max_ctas >= 1, "hp_rmsnorm: max_ctas must be >= 1");
  const int wpb = 8;
  const int grid = std::min((rows + wpb - 1) / wpb, max_ctas * 4);
  HP_LAUNCH_PDL("k_rmsnorm", k_rmsnorm, dim3(grid), dim3(wpb * 32), 0, static_cast<cudaStream_t>(stream),
                static_cast<const __nv_bfloat16*>(x), ldx, static_cast<const __nv_bfloat16*>(weight),
                static_cast<__nv_bfloat16*>(out), ldo, rows, cols, eps);
  return HP_OK;
}

extern "C" int hp_rope_kv_write(void* qkv, int ldqkv, int T, int Hq, int Hkv, int d,
                                const int* positions, const float* cos_sin, const int* slot_mapping,
                                void* kcache, void* vcache, int page, int max_ctas, void* stream) {
  HP_CHECK_ARG(qkv && positions && cos_sin && slot_mapping && kcache && vcache, "hp_rope_kv_write: null pointer");
  HP_CHECK_ARG(T >= 1 && Hq >= 1 && Hkv >= 1 && d % 4 == 0, "hp_rope_kv_write: bad shape");
  HP_CHECK_ARG(ldqkv >= (Hq + 2 * Hkv) * d && ldqkv % 2 == 0, "hp_rope_kv_write: bad row pitch");
  HP_CHECK_ARG(page >= 64 && page % 64 == 0 && max_ctas >= 1, "hp_rope_kv_write: page must be a multiple of 64");
  HP_CHECK_ARG(d % 64 == 0, "hp_rope_kv_write: head_dim must be a multiple of 64");
  const long total = long(T) * (Hq + 2 * Hkv) * (d / 4);
  const int threads = 256;
  const long want = (total + threads - 1) / threads;
  const int grid = int(std::min<long>(want, long(max_ctas) * 8));
  HP_LAUNCH_PDL("k_rope_kv_write", k_rope_kv_write, dim3(grid), dim3(threads), 0,
                static_cast<cudaStream_t>(stream), static_cast<__nv_bfloat16*>(qkv), ldqkv, T, Hq, Hkv, d,
                positions, cos_sin, slot_mapping, static_cast<__nv_bfloat16*>(kcache),
                static_cast<__nv_bfloat16*>(vcache), page);
  return HP_OK;
}
