// Paged-KV decode attention (reference kernel group "attn", phase decode,
// workload.py:184-188): one query token per sequence attends over its
// ctx_lens[b] cached positions.  HBM-bound: every cached K/V byte is read
// once per step.
//
// Layout: kcache/vcache [num_blocks, Hkv, page, d] bf16 (page = 64, d = 128),
// so one (block, kv head) page is a contiguous 16 KB run.  The cache is viewed
// as a 2-D tensor [num_blocks*Hkv*page, d] and streamed with TMA in tiles of
// 32 tokens (half a page, 128B-swizzled) into a 12-stage shared-memory ring
// filled by a dedicated producer warp -- ~190 KB in flight per SM.
//
// Work unit = (sequence b, kv head, split of `tps` 32-token tiles).  Four
// consumer warps take the unit's tiles round-robin; each computes the GQA
// group's scores with tensor cores in "swap" orientation
//     S^T[32 tok, 8 heads] = K[32, 128] . Q^T[128, 8]     (mma.m16n8k16)
//     O^T[128, 8]         += V^T[128, 32] . P^T[32, 8]
// so the tiny query group (<= 8 heads) sits in the MMA's N=8 dimension,
// keeps an online softmax (warp-shuffle max/sum), and the warps merge their
// (m, l, O) at the unit end.  Multi-split sequences write fp32 partials that
// k_decode_combine merges by log-sum-exp.
#include "common.cuh"
#include "runtime.h"
#include "../../include/hp.h"

#include <algorithm>
#include <cmath>

namespace hp {

constexpr int DA_D = 128;
constexpr int DA_TILE = 32;
constexpr int DA_STAGES = 12;
constexpr int DA_CONSUMERS = 4;
constexpr int DA_THREADS = (DA_CONSUMERS + 1) * 32;
constexpr uint32_t DA_BOX_BYTES = DA_TILE * 64 * 2;           // 32 rows x 128 B
constexpr uint32_t DA_STAGE_BYTES = 4 * DA_BOX_BYTES;          // K lo/hi + V lo/hi
constexpr int DA_PROW = 40;                                    // padded P^T row (bf16)
constexpr size_t DA_SMEM = 1024 + size_t(DA_STAGES) * DA_STAGE_BYTES +
                           DA_CONSUMERS * (8 * 128 + 16) * sizeof(float) +
                           DA_CONSUMERS * 8 * DA_PROW * 2 + 2 * DA_STAGES * 8 + 64;

struct DecodeParams {
  const __nv_bfloat16* q;
  int ldq;
  const int* block_table;
  int max_pages;
  const int* ctx_lens;
  __nv_bfloat16* out;
  int ldo;
  int B, Hq, Hkv, G, page;
  int tps;          // tiles per split
  int max_splits;
  float scale_log2;
  float* ws_o;      // [B, Hq, max_splits, d]
  float* ws_ml;     // [B, Hq, max_splits, 2]
};

__global__ void __launch_bounds__(DA_THREADS, 1)
    k_decode_attn(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                  const DecodeParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* ring = smem;
  float* cbuf = reinterpret_cast<float*>(ring + DA_STAGES * DA_STAGE_BYTES);  // [4][8*128 + 16]
  __nv_bfloat16* pbuf = reinterpret_cast<__nv_bfloat16*>(cbuf + DA_CONSUMERS * (8 * 128 + 16));
  uint64_t* full = reinterpret_cast<uint64_t*>(pbuf + DA_CONSUMERS * 8 * DA_PROW);
  uint64_t* empty = full + DA_STAGES;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    for (int s = 0; s < DA_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();

  const int total = p.B * p.Hkv * p.max_splits;
  const int page_tiles = p.page / DA_TILE;
  uint32_t gtile = 0;  // running tile counter across this CTA's units (ring position)

  for (int u = blockIdx.x; u < total; u += gridDim.x) {
    const int s = u % p.max_splits;
    const int bh = u / p.max_splits;
    const int kvh = bh % p.Hkv;
    const int b = bh / p.Hkv;
    const int ctx = p.ctx_lens[b];
    const int ntiles = (ctx + DA_TILE - 1) / DA_TILE;
    const int t0 = s * p.tps;
    const int t1 = min(ntiles, t0 + p.tps);
    if (t0 >= t1) continue;  // empty split (uniform across the CTA)
    const int nt = t1 - t0;

    if (warp == DA_CONSUMERS) {
      // ---------------------------------------------------------- producer
      if (lane == 0) {
        const int* bt = p.block_table + size_t(b) * p.max_pages;
        for (int i = 0; i < nt; ++i) {
          const uint32_t g = gtile + i;
          const int st = g % DA_STAGES;
          const uint32_t ph = (g / DA_STAGES) & 1;
          const int t = t0 + i;
          const int blk = bt[t / page_tiles];
          const int row = (blk * p.Hkv + kvh) * p.page + (t % page_tiles) * DA_TILE;
          mbar_wait(&empty[st], ph ^ 1);
          mbar_arrive_expect_tx(&full[st], DA_STAGE_BYTES);
          uint8_t* sb = ring + st * DA_STAGE_BYTES;
          tma_load_2d(sb, &tmK, &full[st], 0, row);
          tma_load_2d(sb + DA_BOX_BYTES, &tmK, &full[st], 64, row);
          tma_load_2d(sb + 2 * DA_BOX_BYTES, &tmV, &full[st], 0, row);
          tma_load_2d(sb + 3 * DA_BOX_BYTES, &tmV, &full[st], 64, row);
        }
      }
    } else {
      // ---------------------------------------------------------- consumers
      const int g8 = lane >> 2;  // MMA group id
      const int t4 = lane & 3;   // thread in group
      // Q^T fragments (B operand): n = head g8 of this kv group, k = d
      uint32_t qf[8][2];
      {
        const bool hv = g8 < p.G;
        const __nv_bfloat16* qrow = p.q + size_t(b) * p.ldq + size_t(kvh * p.G + (hv ? g8 : 0)) * DA_D;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          uint32_t lo = *reinterpret_cast<const uint32_t*>(qrow + kk * 16 + 2 * t4);
          uint32_t hi = *reinterpret_cast<const uint32_t*>(qrow + kk * 16 + 2 * t4 + 8);
          qf[kk][0] = hv ? lo : 0u;
          qf[kk][1] = hv ? hi : 0u;
        }
      }
      float o[8][4];
#pragma unroll
      for (int i = 0; i < 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
      float m0 = -INFINITY, m1 = -INFINITY;  // running max for heads 2t4, 2t4+1
      float l0 = 0.f, l1 = 0.f;              // per-lane partial sums
      __nv_bfloat16* pw = pbuf + warp * 8 * DA_PROW;

      for (int i = warp; i < nt; i += DA_CONSUMERS) {
        const uint32_t g = gtile + i;
        const int st = g % DA_STAGES;
        const uint32_t ph = (g / DA_STAGES) & 1;
        mbar_wait(&full[st], ph);
        const uint32_t kb = smem_u32(ring + st * DA_STAGE_BYTES);
        const uint32_t vb = kb + 2 * DA_BOX_BYTES;
        // ---- S^T = K . Q^T  (two 16-token m tiles)
        float sc[2][4];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          sc[mt][0] = sc[mt][1] = sc[mt][2] = sc[mt][3] = 0.f;
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const int mat = lane >> 3;
            const uint32_t r = mt * 16 + (mat & 1) * 8 + (lane & 7);
            const uint32_t c = (kk & 3) * 2 + (mat >> 1);
            uint32_t a[4];
            ldmatrix_x4(kb + (kk >> 2) * DA_BOX_BYTES + sw128(r, c), a[0], a[1], a[2], a[3]);
            mma_bf16_16816(sc[mt], a, qf[kk]);
          }
        }
        // ---- mask, scale, online softmax
        const int tokbase = (t0 + i) * DA_TILE;
        float tm0 = -INFINITY, tm1 = -INFINITY;
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int tok = tokbase + mt * 16 + g8 + h * 8;
            const bool valid = tok < ctx;
            sc[mt][2 * h] = valid ? sc[mt][2 * h] * p.scale_log2 : -INFINITY;
            sc[mt][2 * h + 1] = valid ? sc[mt][2 * h + 1] * p.scale_log2 : -INFINITY;
            tm0 = fmaxf(tm0, sc[mt][2 * h]);
            tm1 = fmaxf(tm1, sc[mt][2 * h + 1]);
          }
        }
#pragma unroll
        for (int off = 4; off < 32; off <<= 1) {
          tm0 = fmaxf(tm0, __shfl_xor_sync(0xffffffffu, tm0, off));
          tm1 = fmaxf(tm1, __shfl_xor_sync(0xffffffffu, tm1, off));
        }
        const float n0 = fmaxf(m0, tm0), n1 = fmaxf(m1, tm1);
        const float a0 = exp2f(m0 - n0), a1 = exp2f(m1 - n1);
        m0 = n0;
        m1 = n1;
        l0 *= a0;
        l1 *= a1;
#pragma unroll
        for (int dm = 0; dm < 8; ++dm) {
          o[dm][0] *= a0;
          o[dm][2] *= a0;
          o[dm][1] *= a1;
          o[dm][3] *= a1;
        }
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const float p0 = exp2f(sc[mt][2 * h] - n0);
            const float p1 = exp2f(sc[mt][2 * h + 1] - n1);
            l0 += p0;
            l1 += p1;
            const int tok = mt * 16 + g8 + h * 8;
            pw[(2 * t4) * DA_PROW + tok] = __float2bfloat16(p0);
            pw[(2 * t4 + 1) * DA_PROW + tok] = __float2bfloat16(p1);
          }
        }
        __syncwarp();
        // ---- O^T += V^T . P^T
        uint32_t pf[2][2];
#pragma unroll
        for (int kt = 0; kt < 2; ++kt) {
          pf[kt][0] = *reinterpret_cast<const uint32_t*>(pw + g8 * DA_PROW + kt * 16 + 2 * t4);
          pf[kt][1] = *reinterpret_cast<const uint32_t*>(pw + g8 * DA_PROW + kt * 16 + 2 * t4 + 8);
        }
#pragma unroll
        for (int dm = 0; dm < 8; ++dm) {
#pragma unroll
          for (int kt = 0; kt < 2; ++kt) {
            const int mat = lane >> 3;
            const uint32_t r = kt * 16 + (mat >> 1) * 8 + (lane & 7);
            const uint32_t c = (dm & 3) * 2 + (mat & 1);
            uint32_t a[4];
            ldmatrix_x4_trans(vb + (dm >> 2) * DA_BOX_BYTES + sw128(r, c), a[0], a[1], a[2], a[3]);
            mma_bf16_16816(o[dm], a, pf[kt]);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
      }
      // ---- merge the four warps' (m, l, O)
#pragma unroll
      for (int off = 4; off < 32; off <<= 1) {
        l0 += __shfl_xor_sync(0xffffffffu, l0, off);
        l1 += __shfl_xor_sync(0xffffffffu, l1, off);
      }
      float* cw = cbuf + warp * (8 * 128 + 16);
#pragma unroll
      for (int dm = 0; dm < 8; ++dm) {
        cw[(2 * t4) * 128 + dm * 16 + g8] = o[dm][0];
        cw[(2 * t4 + 1) * 128 + dm * 16 + g8] = o[dm][1];
        cw[(2 * t4) * 128 + dm * 16 + g8 + 8] = o[dm][2];
        cw[(2 * t4 + 1) * 128 + dm * 16 + g8 + 8] = o[dm][3];
      }
      if (g8 == 0) {
        cw[8 * 128 + 2 * t4] = m0;
        cw[8 * 128 + 2 * t4 + 1] = m1;
        cw[8 * 128 + 8 + 2 * t4] = l0;
        cw[8 * 128 + 8 + 2 * t4 + 1] = l1;
      }
      named_bar_sync(1, DA_CONSUMERS * 32);
      const int nsplit = (ntiles + p.tps - 1) / p.tps;
      for (int e = threadIdx.x; e < p.G * 32; e += DA_CONSUMERS * 32) {
        const int h = e >> 5;
        const int d4 = (e & 31) * 4;
        float M = -INFINITY;
#pragma unroll
        for (int w = 0; w < DA_CONSUMERS; ++w) M = fmaxf(M, cbuf[w * (8 * 128 + 16) + 8 * 128 + h]);
        float L = 0.f, acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int w = 0; w < DA_CONSUMERS; ++w) {
          const float* c = cbuf + w * (8 * 128 + 16);
          const float mw = c[8 * 128 + h];
          const float f = (mw == -INFINITY) ? 0.f : exp2f(mw - M);
          L += f * c[8 * 128 + 8 + h];
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[j] += f * c[h * 128 + d4 + j];
        }
        const int head = kvh * p.G + h;
        if (nsplit == 1) {
          const float inv = 1.f / L;
          uint2 w;
          w.x = pack_bf16(acc[0] * inv, acc[1] * inv);
          w.y = pack_bf16(acc[2] * inv, acc[3] * inv);
          *reinterpret_cast<uint2*>(p.out + size_t(b) * p.ldo + size_t(head) * DA_D + d4) = w;
        } else {
          const size_t slot = (size_t(b) * p.Hq + head) * p.max_splits + s;
          float4 w = make_float4(acc[0], acc[1], acc[2], acc[3]);
          *reinterpret_cast<float4*>(p.ws_o + slot * DA_D + d4) = w;
          if ((e & 31) == 0) {
            p.ws_ml[slot * 2] = M;
            p.ws_ml[slot * 2 + 1] = L;
          }
        }
      }
      named_bar_sync(1, DA_CONSUMERS * 32);
    }
    gtile += nt;
  }
}

// One warp per (sequence, head): log-sum-exp merge of the split partials.
__global__ void k_decode_combine(const DecodeParams p) {
  const int warp_global = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp_global >= p.B * p.Hq) return;
  const int b = warp_global / p.Hq;
  const int head = warp_global % p.Hq;
  const int ntiles = (p.ctx_lens[b] + DA_TILE - 1) / DA_TILE;
  const int nsplit = (ntiles + p.tps - 1) / p.tps;
  if (nsplit <= 1) return;  // written directly by the main kernel
  const size_t base = (size_t(b) * p.Hq + head) * p.max_splits;
  float M = -INFINITY;
  for (int s = 0; s < nsplit; ++s) M = fmaxf(M, p.ws_ml[(base + s) * 2]);
  float L = 0.f, acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int s = 0; s < nsplit; ++s) {
    const float f = exp2f(p.ws_ml[(base + s) * 2] - M);
    L += f * p.ws_ml[(base + s) * 2 + 1];
    const float4 v = *reinterpret_cast<const float4*>(p.ws_o + (base + s) * DA_D + lane * 4);
    acc[0] += f * v.x;
    acc[1] += f * v.y;
    acc[2] += f * v.z;
    acc[3] += f * v.w;
  }
  const float inv = 1.f / L;
  uint2 w;
  w.x = pack_bf16(acc[0] * inv, acc[1] * inv);
  w.y = pack_bf16(acc[2] * inv, acc[3] * inv);
  *reinterpret_cast<uint2*>(p.out + size_t(b) * p.ldo + size_t(head) * DA_D + lane * 4) = w;
}

}  // namespace hp

using namespace hp;

extern "C" size_t hp_decode_attn_ws_bytes(int B, int Hq, int d, int max_splits) {
  return size_t(B) * Hq * max_splits * (d + 2) * sizeof(float);
}

extern "C" int hp_decode_attn(const void* q, int ldq, const void* kcache, const void* vcache,
                              const int* block_table, int max_pages, const int* ctx_lens, void* out,
                              int ldo, int B, int Hq, int Hkv, int d, int page, int num_blocks,
                              float scale, void* workspace, size_t ws_bytes, int max_ctas,
                              void* stream) {
  HP_CHECK_ARG(q && kcache && vcache && block_table && ctx_lens && out, "hp_decode_attn: null pointer");
  HP_CHECK_ARG(d == DA_D, "hp_decode_attn: head_dim must be 128");
  HP_CHECK_ARG(page % DA_TILE == 0 && page >= DA_TILE, "hp_decode_attn: page must be a multiple of 32");
  HP_CHECK_ARG(Hkv >= 1 && Hq % Hkv == 0 && Hq / Hkv <= 8, "hp_decode_attn: GQA group must be <= 8");
  HP_CHECK_ARG(B >= 1 && max_pages >= 1 && num_blocks >= 1, "hp_decode_attn: empty batch/cache");
  HP_CHECK_ARG(max_ctas >= 1, "hp_decode_attn: max_ctas must be >= 1");
  HP_CHECK_ARG(ldq % 8 == 0 && ldo % 4 == 0, "hp_decode_attn: misaligned strides");
  DecodeParams p{};
  p.q = static_cast<const __nv_bfloat16*>(q);
  p.ldq = ldq;
  p.block_table = block_table;
  p.max_pages = max_pages;
  p.ctx_lens = ctx_lens;
  p.out = static_cast<__nv_bfloat16*>(out);
  p.ldo = ldo;
  p.B = B;
  p.Hq = Hq;
  p.Hkv = Hkv;
  p.G = Hq / Hkv;
  p.page = page;
  p.scale_log2 = scale * 1.4426950408889634f;
  // split so that the unit count covers the grid ~4x, at least 4 tiles/unit
  const int max_tiles = max_pages * (page / DA_TILE);
  const int pairs = B * Hkv;
  int tps = max_tiles;
  while (tps > 4 && pairs * ((max_tiles + tps - 1) / tps) < 4 * max_ctas) tps = (tps + 1) / 2;
  p.tps = std::max(1, tps);
  p.max_splits = (max_tiles + p.tps - 1) / p.tps;
  if (p.max_splits > 1) {
    HP_CHECK_ARG(workspace != nullptr, "hp_decode_attn: workspace required for split contexts");
    if (ws_bytes < hp_decode_attn_ws_bytes(B, Hq, d, p.max_splits)) {
      // not enough scratch for this split: fall back to fewer, longer splits
      int ms = int(ws_bytes / (size_t(B) * Hq * (d + 2) * sizeof(float)));
      HP_CHECK_ARG(ms >= 1, "hp_decode_attn: workspace too small");
      p.tps = (max_tiles + ms - 1) / ms;
      p.max_splits = (max_tiles + p.tps - 1) / p.tps;
    }
    p.ws_o = static_cast<float*>(workspace);
    p.ws_ml = p.ws_o + size_t(B) * Hq * p.max_splits * d;
  }
  CUtensorMap tk, tv;
  const uint64_t rows = uint64_t(num_blocks) * Hkv * page;
  int rc = cached_tmap_bf16(&tk, kcache, rows, d, d, DA_TILE, 64, true);
  if (rc) return rc;
  rc = cached_tmap_bf16(&tv, vcache, rows, d, d, DA_TILE, 64, true);
  if (rc) return rc;
  static bool attr = false;
  if (!attr) {
    HP_CUDA_TRY(cudaFuncSetAttribute(k_decode_attn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(DA_SMEM)));
    attr = true;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int units = B * Hkv * p.max_splits;
  k_decode_attn<<<std::min(units, max_ctas), DA_THREADS, DA_SMEM, st>>>(tk, tv, p);
  HP_LAUNCH_CHECK("k_decode_attn");
  if (p.max_splits > 1) {
    const int warps = B * Hq;
    k_decode_combine<<<(warps + 7) / 8, 256, 0, st>>>(p);
    HP_LAUNCH_CHECK("k_decode_combine");
  }
  return HP_OK;
}
