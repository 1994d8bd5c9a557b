// Paged-KV decode attention (reference kernel group "attn", phase decode,
// workload.py:184-188): one query token per sequence attends over its
// ctx_lens[b] cached positions.  HBM-bound: every cached K/V byte is read
// once per step.
//
// Cache layout (written by hp_rope_kv_write): per (block, kv head) a page is
// [D/64][page][64] bf16 with the 16-byte chunks of token row r permuted by
// (r & 7) -- the SWIZZLE_128B pattern.  A 64-token tile of one 64-dim half is
// therefore one contiguous 8 KB run: the producer warp streams K and V with
// 1-D bulk copies (one request per 8 KB rather than one per 128-byte row) into
// a 5-stage ring (160 KB in flight per SM at D = 128), and consumers read it
// with conflict-free ldmatrix exactly as if TMA had swizzled it.
//
// Work unit = (sequence b, kv head, split of `tps` 64-token tiles).  Eight
// consumer warps take the unit's tiles round-robin; each computes the GQA
// group's scores with tensor cores in "swap" orientation
//     S^T[64 tok, 8 heads] = K[64, D] . Q^T[D, 8]        (mma.m16n8k16)
//     O^T[D, 8]           += V^T[D, 64] . P^T[64, 8]
// so the query group (<= 8 heads) sits in the MMA's N=8 dimension, with an
// exp2 online softmax and warp-shuffle max/sum; the warps merge (m, l, O) at
// the unit end and multi-split sequences are merged by log-sum-exp in
// k_decode_combine.
//
// Caches must not hold NaN/Inf in unused slots of partially filled pages
// (allocate them zeroed): masked probabilities are exactly 0, but 0 * NaN is
// NaN inside the MMA.
#include "common.cuh"
#include "runtime.h"
#include "../../include/hp.h"

#include <algorithm>
#include <cmath>

namespace hp {

constexpr int DA_TILE = 64;
constexpr int DA_CONSUMERS = 8;
constexpr int DA_THREADS = (DA_CONSUMERS + 1) * 32;
constexpr uint32_t DA_BOX_BYTES = DA_TILE * 64 * 2;  // 64 rows x 128 B
constexpr int DA_PROW = 72;                          // padded P^T row (bf16)
constexpr int DA_WIN = 256;                          // block-table window (pages per unit)

template <int D>
struct DaCfg {
  static constexpr int NBOX = D / 64;                           // 128B boxes per row
  static constexpr uint32_t STAGE_BYTES = 2 * NBOX * DA_BOX_BYTES;
  static constexpr int STAGES = int((160u * 1024u) / STAGE_BYTES);
  static constexpr int CB = 8 * D + 16;                         // per-warp merge buffer (floats)
  static constexpr size_t SMEM = 1024 + size_t(STAGES) * STAGE_BYTES +
                                 DA_CONSUMERS * CB * sizeof(float) +
                                 DA_CONSUMERS * 8 * DA_PROW * 2 + 2 * STAGES * 8 + 64 + 64 +
                                 2 * DA_WIN * sizeof(int);
};

struct DecodeParams {
  const __nv_bfloat16* q;
  int ldq;
  const uint8_t* kc;
  const uint8_t* vc;
  const int* block_table;
  int max_pages;
  const int* ctx_lens;
  __nv_bfloat16* out;
  int ldo;
  int B, Hq, Hkv, G, page;
  int tps;          // tiles per split
  int max_splits;
  float scale_log2;
  float* ws_o;      // [B, Hq, max_splits, D]
  float* ws_ml;     // [B, Hq, max_splits, 2]
};

struct UnitId {
  int b, kvh, s;
};

__device__ __forceinline__ UnitId unit_of(const DecodeParams& p, int u) {
  UnitId id;
  id.s = u % p.max_splits;
  const int bh = u / p.max_splits;
  id.kvh = bh % p.Hkv;
  id.b = bh / p.Hkv;
  return id;
}

template <int D>
__global__ void __launch_bounds__(DA_THREADS, 1) k_decode_attn(const DecodeParams p) {
  using C = DaCfg<D>;
  constexpr int KK = D / 16;
  constexpr int STAGES = C::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* ring = smem;
  float* cbuf = reinterpret_cast<float*>(ring + STAGES * C::STAGE_BYTES);
  __nv_bfloat16* pbuf = reinterpret_cast<__nv_bfloat16*>(cbuf + DA_CONSUMERS * C::CB);
  uint64_t* full = reinterpret_cast<uint64_t*>(pbuf + DA_CONSUMERS * 8 * DA_PROW);
  uint64_t* empty = full + STAGES;
  // Tiles are consumed round-robin by 8 warps from a ring of STAGES slots, so
  // a warp can reach a slot more than one phase ahead of the producer, where
  // a parity wait would be ambiguous.  Consumers first wait until the slot's
  // tag names their tile (set once the producer passed the slot's empty
  // barrier for it, i.e. the previous occupant was released), then wait on
  // the slot's parity.
  volatile uint32_t* tag = reinterpret_cast<volatile uint32_t*>(empty + STAGES);
  int* win = reinterpret_cast<int*>(const_cast<uint32_t*>(tag) + 16);  // [2][DA_WIN] page ids

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 2 * C::NBOX);  // one arrive per K/V box (issued by separate lanes)
      mbar_init(&empty[s], 1);
      tag[s] = 0xffffffffu;
    }
    fence_barrier_init();
  }
  __syncthreads();

  const int total = p.B * p.Hkv * p.max_splits;
  const int page_tiles = p.page / DA_TILE;
  const size_t page_elems = size_t(p.page) * 64;  // one 64-dim half of one page

  if (warp == DA_CONSUMERS) {
    // ------------------------------------------------------------ producer
    // One thread's async-copy stream is serialised at ~one DRAM latency per
    // copy, so every 8 KB box of a tile is issued by its own lane: lane =
    // slot * PARTS + part, where `slot` takes every SLOTS-th tile of the
    // unit (SLOTS <= STAGES keeps every parity wait unambiguous) and `part`
    // is one K or V box.  The unit's block-table pages are staged in a
    // double-buffered smem window, loaded one unit ahead.
    constexpr int PARTS = 2 * C::NBOX;
    constexpr int SLOTS = (32 / PARTS) < STAGES ? (32 / PARTS) : STAGES;
    const int slot = lane / PARTS, part = lane % PARTS;
    const bool issuer = slot < SLOTS;
    const uint64_t pol = l2_policy_evict_first();  // KV is read once per step
    uint32_t gtile = 0;
    int wb = 0;
    auto load_window = [&](int u, int buf) -> int {  // returns ctx of unit u
      const UnitId id = unit_of(p, u);
      const int ctx = p.ctx_lens[id.b];
      const int first = (id.s * p.tps) / page_tiles;
      const int last = min(p.max_pages, ((id.s + 1) * p.tps + page_tiles - 1) / page_tiles);
      for (int j = lane; j < last - first; j += 32)
        win[buf * DA_WIN + j] = p.block_table[size_t(id.b) * p.max_pages + first + j];
      return ctx;
    };
    int u = blockIdx.x;
    int ctx_cur = u < total ? load_window(u, 0) : 0;
    for (; u < total; u += gridDim.x) {
      const UnitId id = unit_of(p, u);
      __syncwarp();
      const int ctx_nxt = (u + int(gridDim.x) < total) ? load_window(u + gridDim.x, wb ^ 1) : 0;
      const int ntiles = (ctx_cur + DA_TILE - 1) / DA_TILE;
      const int t0 = id.s * p.tps;
      const int t1 = min(ntiles, t0 + p.tps);
      if (issuer && t0 < t1) {
        const int first = t0 / page_tiles;
        for (int t = t0 + slot; t < t1; t += SLOTS) {
          const int blk = win[wb * DA_WIN + t / page_tiles - first];
          const uint32_t g = gtile + (t - t0);
          const int st = g % STAGES;
          const uint32_t ph = (g / STAGES) & 1;
          const size_t base = (size_t(blk) * p.Hkv + id.kvh) * C::NBOX * page_elems +
                              size_t(t % page_tiles) * DA_TILE * 64;
          mbar_wait(&empty[st], ph ^ 1);
          mbar_arrive_expect_tx(&full[st], DA_BOX_BYTES);
          const int bx = part % C::NBOX;
          const uint8_t* src = (part < C::NBOX ? p.kc : p.vc) + (base + bx * page_elems) * 2;
          bulk_load_hint(ring + st * C::STAGE_BYTES + part * DA_BOX_BYTES, src, DA_BOX_BYTES, &full[st], pol);
          if (part == 0) tag[st] = g;
        }
      }
      gtile += max(0, t1 - t0);
      ctx_cur = ctx_nxt;
      wb ^= 1;
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  const int g8 = lane >> 2;  // MMA group id
  const int t4 = lane & 3;   // thread in group
  const int mat = lane >> 3;
  __nv_bfloat16* pw = pbuf + warp * 8 * DA_PROW;
  float* cw = cbuf + warp * C::CB;
  uint32_t gtile = 0;

  auto load_q = [&](int u, uint32_t (&qf)[KK][2], int& ctx) {
    const UnitId id = unit_of(p, u);
    ctx = p.ctx_lens[id.b];
    const bool hv = g8 < p.G;
    const __nv_bfloat16* qrow = p.q + size_t(id.b) * p.ldq + size_t(id.kvh * p.G + (hv ? g8 : 0)) * D;
#pragma unroll
    for (int kk = 0; kk < KK; ++kk) {
      const uint32_t lo = *reinterpret_cast<const uint32_t*>(qrow + kk * 16 + 2 * t4);
      const uint32_t hi = *reinterpret_cast<const uint32_t*>(qrow + kk * 16 + 2 * t4 + 8);
      qf[kk][0] = hv ? lo : 0u;
      qf[kk][1] = hv ? hi : 0u;
    }
  };

  uint32_t qcur[KK][2];
  int ctx_cur = 0;
  if (blockIdx.x < total) load_q(blockIdx.x, qcur, ctx_cur);

  for (int u = blockIdx.x; u < total; u += gridDim.x) {
    const UnitId id = unit_of(p, u);
    uint32_t qnxt[KK][2];
    int ctx_nxt = 0;
    if (u + int(gridDim.x) < total) load_q(u + gridDim.x, qnxt, ctx_nxt);
    const int ctx = ctx_cur;
    const int ntiles = (ctx + DA_TILE - 1) / DA_TILE;
    const int t0 = id.s * p.tps;
    const int t1 = min(ntiles, t0 + p.tps);
    if (t0 < t1) {
      const int nt = t1 - t0;
      float o[KK][4];
#pragma unroll
      for (int i = 0; i < KK; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
      float m0 = -INFINITY, m1 = -INFINITY;  // running max for heads 2t4, 2t4+1
      float l0 = 0.f, l1 = 0.f;              // per-lane partial sums

      for (int i = warp; i < nt; i += DA_CONSUMERS) {
        const uint32_t g = gtile + i;
        const int st = g % STAGES;
        const uint32_t ph = (g / STAGES) & 1;
        while (tag[st] != g) __nanosleep(32);
        mbar_wait(&full[st], ph);
        const uint32_t kb = smem_u32(ring + st * C::STAGE_BYTES);
        const uint32_t vb = kb + C::NBOX * DA_BOX_BYTES;
        // ---- S^T = K . Q^T : four independent 16-token m tiles
        float sc[4][4];
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) sc[mt][0] = sc[mt][1] = sc[mt][2] = sc[mt][3] = 0.f;
#pragma unroll
        for (int kk = 0; kk < KK; ++kk) {
#pragma unroll
          for (int mt = 0; mt < 4; ++mt) {
            const uint32_t r = mt * 16 + (mat & 1) * 8 + (lane & 7);
            const uint32_t c = (kk & 3) * 2 + (mat >> 1);
            uint32_t a[4];
            ldmatrix_x4(kb + (kk >> 2) * DA_BOX_BYTES + sw128(r, c), a[0], a[1], a[2], a[3]);
            mma_bf16_16816(sc[mt], a, qcur[kk]);
          }
        }
        // ---- mask, scale, online softmax
        const int tokbase = (t0 + i) * DA_TILE;
        float tm0 = -INFINITY, tm1 = -INFINITY;
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const bool valid = tokbase + mt * 16 + g8 + h * 8 < ctx;
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
        for (int dm = 0; dm < KK; ++dm) {
          o[dm][0] *= a0;
          o[dm][2] *= a0;
          o[dm][1] *= a1;
          o[dm][3] *= a1;
        }
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) {
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
        uint32_t pf[4][2];
#pragma unroll
        for (int kt = 0; kt < 4; ++kt) {
          pf[kt][0] = *reinterpret_cast<const uint32_t*>(pw + g8 * DA_PROW + kt * 16 + 2 * t4);
          pf[kt][1] = *reinterpret_cast<const uint32_t*>(pw + g8 * DA_PROW + kt * 16 + 2 * t4 + 8);
        }
#pragma unroll
        for (int kt = 0; kt < 4; ++kt) {
#pragma unroll
          for (int dm = 0; dm < KK; ++dm) {
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
      // ---- merge the consumer warps' (m, l, O)
#pragma unroll
      for (int off = 4; off < 32; off <<= 1) {
        l0 += __shfl_xor_sync(0xffffffffu, l0, off);
        l1 += __shfl_xor_sync(0xffffffffu, l1, off);
      }
#pragma unroll
      for (int dm = 0; dm < KK; ++dm) {
        cw[(2 * t4) * D + dm * 16 + g8] = o[dm][0];
        cw[(2 * t4 + 1) * D + dm * 16 + g8] = o[dm][1];
        cw[(2 * t4) * D + dm * 16 + g8 + 8] = o[dm][2];
        cw[(2 * t4 + 1) * D + dm * 16 + g8 + 8] = o[dm][3];
      }
      if (g8 == 0) {
        cw[8 * D + 2 * t4] = m0;
        cw[8 * D + 2 * t4 + 1] = m1;
        cw[8 * D + 8 + 2 * t4] = l0;
        cw[8 * D + 8 + 2 * t4 + 1] = l1;
      }
      named_bar_sync(1, DA_CONSUMERS * 32);
      const int nsplit = (ntiles + p.tps - 1) / p.tps;
      const int nw = min(DA_CONSUMERS, nt);  // warps that saw at least one tile
      constexpr int Q4 = D / 4;              // float4 groups per head row
      for (int e = threadIdx.x; e < p.G * Q4; e += DA_CONSUMERS * 32) {
        const int h = e / Q4;
        const int d4 = (e % Q4) * 4;
        float M = -INFINITY;
        for (int w = 0; w < nw; ++w) M = fmaxf(M, cbuf[w * C::CB + 8 * D + h]);
        float L = 0.f, acc[4] = {0.f, 0.f, 0.f, 0.f};
        for (int w = 0; w < nw; ++w) {
          const float* c = cbuf + w * C::CB;
          const float f = exp2f(c[8 * D + h] - M);
          L += f * c[8 * D + 8 + h];
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[j] += f * c[h * D + d4 + j];
        }
        const int head = id.kvh * p.G + h;
        if (nsplit == 1) {
          const float inv = 1.f / L;
          uint2 w;
          w.x = pack_bf16(acc[0] * inv, acc[1] * inv);
          w.y = pack_bf16(acc[2] * inv, acc[3] * inv);
          *reinterpret_cast<uint2*>(p.out + size_t(id.b) * p.ldo + size_t(head) * D + d4) = w;
        } else {
          const size_t slot = (size_t(id.b) * p.Hq + head) * p.max_splits + id.s;
          *reinterpret_cast<float4*>(p.ws_o + slot * D + d4) = make_float4(acc[0], acc[1], acc[2], acc[3]);
          if (e % Q4 == 0) {
            p.ws_ml[slot * 2] = M;
            p.ws_ml[slot * 2 + 1] = L;
          }
        }
      }
      named_bar_sync(1, DA_CONSUMERS * 32);
      gtile += nt;
    }
#pragma unroll
    for (int kk = 0; kk < KK; ++kk) {
      qcur[kk][0] = qnxt[kk][0];
      qcur[kk][1] = qnxt[kk][1];
    }
    ctx_cur = ctx_nxt;
  }
}

// One warp per (sequence, head): log-sum-exp merge of the split partials.
template <int D>
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
  constexpr int PER = D / 32;  // dims per lane (2 or 4)
  float L = 0.f, acc[PER];
#pragma unroll
  for (int j = 0; j < PER; ++j) acc[j] = 0.f;
  for (int s = 0; s < nsplit; ++s) {
    const float f = exp2f(p.ws_ml[(base + s) * 2] - M);
    L += f * p.ws_ml[(base + s) * 2 + 1];
    const float* src = p.ws_o + (base + s) * D + lane * PER;
#pragma unroll
    for (int j = 0; j < PER; ++j) acc[j] += f * src[j];
  }
  const float inv = 1.f / L;
  __nv_bfloat16* dst = p.out + size_t(b) * p.ldo + size_t(head) * D + lane * PER;
#pragma unroll
  for (int j = 0; j < PER; j += 2)
    *reinterpret_cast<uint32_t*>(dst + j) = pack_bf16(acc[j] * inv, acc[j + 1] * inv);
}

template <int D>
static int launch_decode(const DecodeParams& p, int max_ctas, cudaStream_t st) {
  using C = DaCfg<D>;
  static bool attr = false;
  if (!attr) {
    HP_CUDA_TRY(cudaFuncSetAttribute(k_decode_attn<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM)));
    attr = true;
  }
  const int units = p.B * p.Hkv * p.max_splits;
  k_decode_attn<D><<<std::min(units, max_ctas), DA_THREADS, C::SMEM, st>>>(p);
  HP_LAUNCH_CHECK("k_decode_attn");
  if (p.max_splits > 1) {
    const int warps = p.B * p.Hq;
    k_decode_combine<D><<<(warps + 7) / 8, 256, 0, st>>>(p);
    HP_LAUNCH_CHECK("k_decode_combine");
  }
  return HP_OK;
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
  HP_CHECK_ARG(d == 64 || d == 128, "hp_decode_attn: head_dim must be 64 or 128");
  HP_CHECK_ARG(page % DA_TILE == 0 && page >= DA_TILE, "hp_decode_attn: page must be a multiple of 64");
  HP_CHECK_ARG(Hkv >= 1 && Hq % Hkv == 0 && Hq / Hkv <= 8, "hp_decode_attn: GQA group must be <= 8");
  HP_CHECK_ARG(B >= 1 && max_pages >= 1 && num_blocks >= 1, "hp_decode_attn: empty batch/cache");
  HP_CHECK_ARG(max_ctas >= 1, "hp_decode_attn: max_ctas must be >= 1");
  HP_CHECK_ARG(ldq % 8 == 0 && ldo % 4 == 0, "hp_decode_attn: misaligned strides");
  DecodeParams p{};
  p.q = static_cast<const __nv_bfloat16*>(q);
  p.ldq = ldq;
  p.kc = static_cast<const uint8_t*>(kcache);
  p.vc = static_cast<const uint8_t*>(vcache);
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
  // split so that the unit count covers the grid ~4x, at least 2 tiles/unit
  const int max_tiles = max_pages * (page / DA_TILE);
  const int pairs = B * Hkv;
  int tps = max_tiles;
  while (tps > 2 && pairs * ((max_tiles + tps - 1) / tps) < 4 * max_ctas) tps = (tps + 1) / 2;
  p.tps = std::max(1, std::min(tps, (DA_WIN - 1) * (page / DA_TILE)));  // unit pages fit the window
  p.max_splits = (max_tiles + p.tps - 1) / p.tps;
  if (p.max_splits > 1) {
    HP_CHECK_ARG(workspace != nullptr, "hp_decode_attn: workspace required for split contexts");
    if (ws_bytes < hp_decode_attn_ws_bytes(B, Hq, d, p.max_splits)) {
      // not enough scratch for this split: fall back to fewer, longer splits
      const int ms = int(ws_bytes / (size_t(B) * Hq * (d + 2) * sizeof(float)));
      p.tps = ms <= 1 ? max_tiles : (max_tiles + ms - 1) / ms;
      HP_CHECK_ARG(p.tps <= (DA_WIN - 1) * (page / DA_TILE),
                   "hp_decode_attn: workspace too small to split this context");
      p.max_splits = (max_tiles + p.tps - 1) / p.tps;
    }
    p.ws_o = static_cast<float*>(workspace);
    p.ws_ml = p.ws_o + size_t(B) * Hq * p.max_splits * d;
  }
  HP_CHECK_ARG((reinterpret_cast<uintptr_t>(kcache) & 15) == 0 && (reinterpret_cast<uintptr_t>(vcache) & 15) == 0,
               "hp_decode_attn: caches must be 16B aligned");
  (void)num_blocks;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  return d == 128 ? launch_decode<128>(p, max_ctas, st) : launch_decode<64>(p, max_ctas, st);
}
