// tcgen05 / TMEM / TMA GEMM for the four linear kernels of a Llama layer.
//
//   D = A . B^T  with A [Ma, K] and B [Nb, K] bf16, both K-major (torch
//   [out, in] weight layout), fp32 accumulation in TMEM.
//
// Token-major operand placement for prefill: A = activations X [T, K],
// B = weights W [N, K]; D tile = 128 tokens x BN features, and the epilogue
// writes Y [T, N] rows directly from TMEM.  (Decode's skinny GEMMs use the
// swap-AB stream-K kernel in gemm_swap.cu.)
//
// Epilogues (reference kernel groups, workload.py:164-209):
//   STORE  : Y = D                               (qkv projection)
//   RESID  : Y = D + R                           (o_proj / mlp_down residual)
//   SILU   : Y = silu(D_gate) * D_up             (mlp_up_gate; W rows are
//            interleaved in blocks of 64: [g0..g63, u0..u63, g64.., ...])
//
// Persistent: grid = min(work units, max_ctas) where max_ctas is the SM
// count of the partition the launch is confined to; units are walked in a
// static round-robin so the rounds equal wave_stats(units, 1, grid).
//
// Warp roles (192 threads): warp 0 = TMA producer, warp 1 = TMEM allocator +
// single-thread UMMA issuer, warps 2..5 = epilogue (TMEM lane quarter = warp%4).
#include "common.cuh"
#include "runtime.h"
#include "../../include/hp.h"

#include <algorithm>
#include <cstdlib>

namespace hp {

enum { EPI_STORE = 0, EPI_RESID = 1, EPI_SILU = 2, EPI_ROPE = 3 };

struct GemmParams {
  int Ma, Nb, K;
  int m_tiles, n_tiles, k_splits, kb_per_split, num_kb;
  int group_m;  // m-tiles per rasterization group (L2 reuse of the activation block)
  const uint8_t* w;  // weights in the tiled layout (hp_tile_weight)
  __nv_bfloat16* out;
  int ldo;
  const __nv_bfloat16* resid;
  int ldr;
  int epi;
  uint64_t* cta_times;  // optional [grid][3] = {smid, start_ns, end_ns} (wave measurement)
  // EPI_ROPE (fused QKV epilogue): rotary embedding of q/k heads, paged K/V write
  const int* pos;
  const float* cos_sin;  // fp32 [max_pos, d] = [cos(d/2) | sin(d/2)]
  const int* slots;
  __nv_bfloat16* kc;
  __nv_bfloat16* vc;
  int page, Hq, Hkv, hd;
  // Stream-K tail (CTA-pair kernel): tiles [0, sk_dp) run in persistent
  // rounds; the last sk_tail tiles' sk_tail * num_kb k-blocks are split into
  // one contiguous range per pair.  sk_tail = 0: plain rounds.
  int sk_dp, sk_tail;
  float* sk_ws;  // [pairs][2 ranks][8 col chunks][128 rows][32] fp32 partial tiles
  int* sk_cnt;   // [tail tile][rank] arrivals (the finishing CTA resets it)
};

#ifndef HP_GEMM_A_EVICT_LAST
#define HP_GEMM_A_EVICT_LAST 0
#endif

constexpr int BM = 128;
constexpr int BK = 64;

template <int BN>
struct GemmCfg {
  static constexpr uint32_t A_BYTES = BM * BK * 2;
  static constexpr uint32_t B_BYTES = BN * BK * 2;
  static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = (BN >= 256) ? 4 : (BN >= 128 ? 6 : 8);
  static constexpr uint32_t TMEM_COLS = (2 * BN <= 32) ? 32 : (2 * BN <= 64 ? 64 : (2 * BN <= 128 ? 128 : (2 * BN <= 256 ? 256 : 512)));
  static constexpr size_t SMEM = 1024 + size_t(STAGES) * STAGE_BYTES + 256;
};

// Tile index -> (m-tile, n-tile).  Tiles are walked in groups of `group_m`
// m-tiles: a wave of CTAs covers group_m x (grid / group_m) tiles, so the
// group's activation rows (group_m x 128 x K bf16) stay L2-resident while
// the weight tiles stream past once per group.  With group_m = m_tiles this
// is the plain column-major order (every weight tile read once, activations
// re-read per column -- right when all activations fit in L2).  The order
// does not change the tile count, so the rounds stay wave_stats(tiles, 1, n).
__device__ __forceinline__ void tile_coords(const GemmParams& p, int tile, int& mt, int& nt) {
  const int per_group = p.group_m * p.n_tiles;
  const int g = tile / per_group;
  const int first = g * p.group_m;
  const int gsize = min(p.m_tiles - first, p.group_m);
  const int r = tile - g * per_group;
  mt = first + r % gsize;
  nt = r / gsize;
}

__device__ __forceinline__ float silu(float x) { return x / (1.0f + __expf(-x)); }

__device__ __forceinline__ void store_row32(__nv_bfloat16* dst, const float* v) {
  uint4 w[4];
  uint32_t* u = reinterpret_cast<uint32_t*>(w);
#pragma unroll
  for (int j = 0; j < 16; ++j) u[j] = pack_bf16(v[2 * j], v[2 * j + 1]);
  uint4* d = reinterpret_cast<uint4*>(dst);
#pragma unroll
  for (int j = 0; j < 4; ++j) d[j] = w[j];
}

__device__ __forceinline__ void add_row32(float* v, const __nv_bfloat16* src) {
  const uint4* s = reinterpret_cast<const uint4*>(src);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    uint4 w = s[j];
    const uint32_t* u = reinterpret_cast<const uint32_t*>(&w);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      v[8 * j + 2 * k] += bf16lo(u[k]);
      v[8 * j + 2 * k + 1] += bf16hi(u[k]);
    }
  }
}

// ---- stream-K tail -------------------------------------------------------
// Pair i owns k-block range [start(i), start(i+1)) of the tail's flattened
// (tile, k-block) space.  A range is cut at tile boundaries into <= 3
// segments; the one ending mid-tile (at most one per pair) is a PARTIAL: its
// fp32 accumulator goes to workspace slot i and the tile's arrival counter is
// raised.  The pair whose range holds a tile's last k-block FINISHES it: it
// waits for the tile's other contributors (pairs j0..f-1), adds their slots in
// pair order to its own accumulator (a fixed order: deterministic sums) and
// runs the normal fused epilogue.  Pairs process their partial first, so no
// finisher waits on a pair that is itself waiting.
struct Seg {
  int tile, kb0, kb1, kind;  // kind: 0 whole tile, 1 finishing, 2 partial
};

__device__ __forceinline__ int sk_start(const GemmParams& p, int i, int P) {
  return int((long long)i * (long long)(p.sk_tail * p.num_kb) / P);
}

// Work item `it` of pair `pair`: its round-robin data-parallel tiles, then its
// tail segments (partial first).  Returns false past the last item.
__device__ __forceinline__ bool work_item(const GemmParams& p, int pair, int P, int it, Seg& w) {
  const int dp_end = p.sk_tail ? p.sk_dp : p.m_tiles * p.n_tiles;
  const int ndp = pair < dp_end ? (dp_end - pair + P - 1) / P : 0;
  if (it < ndp) {
    w.tile = pair + it * P;
    w.kb0 = 0;
    w.kb1 = p.num_kb;
    w.kind = 0;
    return true;
  }
  if (!p.sk_tail) return false;
  int k = it - ndp;
  const int a = sk_start(p, pair, P), b = sk_start(p, pair + 1, P);
  if (a >= b) return false;
  const int last_t = (b - 1) / p.num_kb;
  const bool has_partial = b != (last_t + 1) * p.num_kb;
  if (has_partial) {
    if (k == 0) {
      w.tile = p.sk_dp + last_t;
      w.kb0 = max(a, last_t * p.num_kb) - last_t * p.num_kb;
      w.kb1 = b - last_t * p.num_kb;
      w.kind = 2;
      return true;
    }
    --k;
  }
  // finishing segments in k order: tiles first_t .. (has_partial ? last_t-1 : last_t)
  const int first_t = a / p.num_kb;
  const int t = first_t + k;
  if (t > (has_partial ? last_t - 1 : last_t)) return false;
  w.tile = p.sk_dp + t;
  w.kb0 = max(a, t * p.num_kb) - t * p.num_kb;
  w.kb1 = p.num_kb;
  w.kind = w.kb0 == 0 ? 0 : 1;  // a whole tile inside the range needs no fix-up
  return true;
}

// The contributors of tail tile `tr` finished by pair f: pairs [j0, f).
__device__ __forceinline__ int sk_first_contributor(const GemmParams& p, int tr, int f, int P) {
  const int A = tr * p.num_kb;
  int j = f - 1;
  while (j >= 0 && sk_start(p, j + 1, P) > A) --j;
  return j + 1;
}

struct TailFix {
  const float* ws;  // nullptr: nothing to add
  int j0, j1, rank, row;
};

__device__ __forceinline__ const float* sk_slot(const float* ws, int j, int rank) {
  return ws + size_t(j) * SK_SLOT_FLOATS + size_t(rank) * (SK_SLOT_FLOATS / 2);
}

// v[0..31] (accumulator columns col..col+31 of this thread's row) += the
// contributors' partials, in pair order
__device__ __forceinline__ void fix_add(const TailFix& f, int col, float* v) {
  if (f.ws == nullptr) return;
  for (int j = f.j0; j < f.j1; ++j) {
    const float4* src = reinterpret_cast<const float4*>(sk_slot(f.ws, j, f.rank) +
                                                        (size_t(col >> 5) * 128 + f.row) * 32);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float4 a = __ldcg(src + k);
      v[4 * k] += a.x;
      v[4 * k + 1] += a.y;
      v[4 * k + 2] += a.z;
      v[4 * k + 3] += a.w;
    }
  }
}

template <int BN>
__device__ __forceinline__ void write_partial(uint32_t taddr, float* slot, int row) {
#pragma unroll 1
  for (int c = 0; c < BN / 32; ++c) {
    float v[32];
    tmem_ld32(taddr + c * 32, v);
    tmem_ld_wait();
    float4* dst = reinterpret_cast<float4*>(slot + (size_t(c) * 128 + row) * 32);
#pragma unroll
    for (int k = 0; k < 8; ++k) __stcg(dst + k, make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]));
  }
}

__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Epilogue of one output tile for the thread owning accumulator row `gm`
// (TMEM address `taddr` = its lane, column 0 of the tile's accumulator).
template <int BN>
__device__ __forceinline__ void epilogue_row(const GemmParams& p, uint32_t taddr, int gm, int nt,
                                             const TailFix& fx) {
  const bool ok = gm < p.Ma;
  if (p.epi == EPI_ROPE) {
    // the tile's BN columns are BN/hd whole heads of the q | k | v blocks
    const int half = p.hd / 2;
    const int pos = ok ? p.pos[gm] : 0;
    const float* cs = p.cos_sin + size_t(pos) * p.hd;
    int blk = 0, off = 0;
    if (ok) {
      const int sl = p.slots[gm];
      blk = sl / p.page;
      off = sl % p.page;
    }
#pragma unroll 1
    for (int hh = 0; hh < BN / p.hd; ++hh) {
      const int head = (nt * BN) / p.hd + hh;
      const bool rot = head < p.Hq + p.Hkv;
#pragma unroll 1
      for (int c = 0; c < half / 32; ++c) {
        float x[32], y[32];
        tmem_ld32(taddr + hh * p.hd + c * 32, x);
        tmem_ld32(taddr + hh * p.hd + half + c * 32, y);
        tmem_ld_wait();
        if (!ok) continue;
        fix_add(fx, hh * p.hd + c * 32, x);
        fix_add(fx, hh * p.hd + half + c * 32, y);
        if (rot) {  // y[i] = x cos - x' sin, y' = x' cos + x sin (rotate_half)
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            const float4 co = *reinterpret_cast<const float4*>(cs + c * 32 + j);
            const float4 si = *reinterpret_cast<const float4*>(cs + half + c * 32 + j);
            const float cc[4] = {co.x, co.y, co.z, co.w}, ss[4] = {si.x, si.y, si.z, si.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              // rotate the bf16-rounded projection, exactly as the
              // unfused GEMM store + hp_rope_kv_write pair does
              const float a = __bfloat162float(__float2bfloat16(x[j + k]));
              const float b = __bfloat162float(__float2bfloat16(y[j + k]));
              rope_rotate(a, b, cc[k], ss[k], x[j + k], y[j + k]);
            }
          }
        }
        __nv_bfloat16* dst = p.out + size_t(gm) * p.ldo + size_t(head) * p.hd;
        store_row32(dst + c * 32, x);
        store_row32(dst + half + c * 32, y);
        if (head >= p.Hq) {  // k or v head -> paged cache page [page/64][hd/64][64][64], swizzled
          const int kvh = rot ? head - p.Hq : head - p.Hq - p.Hkv;
          __nv_bfloat16* cache = rot ? p.kc : p.vc;
          const size_t base = ((size_t(blk) * p.Hkv + kvh) * (p.page / 64) + off / 64) * (p.hd / 64);
#pragma unroll
          for (int part = 0; part < 2; ++part) {
            const float* v = part ? y : x;
            const int j0 = (part ? half : 0) + c * 32;  // first head dim of these 32
#pragma unroll
            for (int q8 = 0; q8 < 4; ++q8) {
              const int j = j0 + q8 * 8;
              uint4 w;
              w.x = pack_bf16(v[q8 * 8 + 0], v[q8 * 8 + 1]);
              w.y = pack_bf16(v[q8 * 8 + 2], v[q8 * 8 + 3]);
              w.z = pack_bf16(v[q8 * 8 + 4], v[q8 * 8 + 5]);
              w.w = pack_bf16(v[q8 * 8 + 6], v[q8 * 8 + 7]);
              const size_t e = (base + j / 64) * 4096 + size_t(off & 63) * 64 +
                               ((((j & 63) >> 3) ^ (off & 7)) << 3);
              *reinterpret_cast<uint4*>(cache + e) = w;
            }
          }
        }
      }
    }
  } else if (p.epi == EPI_SILU) {
#pragma unroll 1
    for (int h = 0; h < BN / 128; ++h) {
#pragma unroll 1
      for (int c = 0; c < 2; ++c) {
        float g[32], v[32];
        tmem_ld32(taddr + h * 128 + c * 32, g);
        tmem_ld32(taddr + h * 128 + 64 + c * 32, v);
        tmem_ld_wait();
        fix_add(fx, h * 128 + c * 32, g);
        fix_add(fx, h * 128 + 64 + c * 32, v);
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = silu(g[j]) * v[j];
        if (ok) store_row32(p.out + size_t(gm) * p.ldo + nt * (BN / 2) + h * 64 + c * 32, v);
      }
    }
  } else {
#pragma unroll 1
    for (int c = 0; c < BN / 32; ++c) {
      float v[32];
      tmem_ld32(taddr + c * 32, v);
      tmem_ld_wait();
      fix_add(fx, c * 32, v);
      const int col = nt * BN + c * 32;
      if (ok) {
        if (p.epi == EPI_RESID) add_row32(v, p.resid + size_t(gm) * p.ldr + col);
        store_row32(p.out + size_t(gm) * p.ldo + col, v);
      }
    }
  }
}

template <int BN>
__global__ void __launch_bounds__(192, 1)
    k_gemm_tc(const __grid_constant__ CUtensorMap tmA, const GemmParams p) {
  using C = GemmCfg<BN>;
  constexpr int STAGES = C::STAGES;
  pdl_trigger();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * C::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  uint64_t* t_start = reinterpret_cast<uint64_t*>(tmem_slot + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    tmem_alloc(tmem_slot, C::TMEM_COLS);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_wait();  // activations / residual from the stream predecessor
  if (threadIdx.x == 0) *t_start = globaltimer();
  const uint32_t tmem_base = *tmem_slot;

  const int total = p.m_tiles * p.n_tiles * p.k_splits;

  if (warp == 0) {
    // One in-order issue stream (operands are mostly L2-resident here:
    // activation tiles are re-read by every N tile, weights by every M tile);
    // the warp walks the schedule converged and one elected lane issues.
    uint32_t g = 0;
    for (int u = blockIdx.x; u < total; u += gridDim.x) {
      const int tile = u / p.k_splits, ks = u % p.k_splits;
      int mt, nt;
      tile_coords(p, tile, mt, nt);
      const int kb0 = ks * p.kb_per_split;
      const int kb1 = min(p.num_kb, kb0 + p.kb_per_split);
      for (int kb = kb0; kb < kb1; ++kb, ++g) {
        const int stage = g % STAGES;
        const uint32_t phase = (g / STAGES) & 1;
        mbar_wait(&empty[stage], phase ^ 1);
        if (elect_one()) {
          mbar_arrive_expect_tx(&full[stage], C::STAGE_BYTES);
          tma_load_2d(sA + stage * C::A_BYTES, &tmA, &full[stage], kb * BK, mt * BM);
#pragma unroll
          for (int h = 0; h < BN / 128; ++h)  // BN rows = BN/128 tiled 128-row blocks
            bulk_load(sB + stage * C::B_BYTES + h * (128 * BK * 2),
                      p.w + wtile_offset(nt * BN + h * 128, kb, p.K), 128 * BK * 2, &full[stage]);
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {
    // warp-converged schedule walk (descriptors in uniform registers); one
    // elected lane issues the UMMAs
    constexpr uint32_t idesc = umma_idesc_bf16(BM, BN);
    const uint64_t adesc0 = umma_desc_sw128(smem_u32(sA));
    const uint64_t bdesc0 = umma_desc_sw128(smem_u32(sB));
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = blockIdx.x; u < total; u += gridDim.x) {
      const int ks = u % p.k_splits;
      const int kb0 = ks * p.kb_per_split;
      const int kb1 = min(p.num_kb, kb0 + p.kb_per_split);
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        const uint64_t ad = adesc0 + uint64_t((stage * C::A_BYTES) >> 4);
        const uint64_t bd = bdesc0 + uint64_t((stage * C::B_BYTES) >> 4);
        const bool first = kb == kb0;
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            umma_bf16(d_tmem, ad + 2 * k, bd + 2 * k, idesc, (!first || k > 0) ? 1u : 0u);
          umma_commit(&empty[stage]);
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      if (elect_one()) umma_commit(&tfull[acc]);
      __syncwarp();
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;              // TMEM lane quarter this warp may access
    const int row = q * 32 + lane;       // accumulator row owned by this thread
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = blockIdx.x; u < total; u += gridDim.x) {
      const int tile = u / p.k_splits;
      int mt, nt;
      tile_coords(p, tile, mt, nt);
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t taddr = tmem_base + (uint32_t(q * 32) << 16) + acc * BN;
      {
        epilogue_row<BN>(p, taddr, mt * BM + row, nt, TailFix{nullptr, 0, 0, 0, 0});
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
      }
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, C::TMEM_COLS);
  }
  if (p.cta_times != nullptr && threadIdx.x == 0) {
    p.cta_times[blockIdx.x * 3 + 0] = smid();
    p.cta_times[blockIdx.x * 3 + 1] = *t_start;
    p.cta_times[blockIdx.x * 3 + 2] = globaltimer();
  }
}

// ---------------------------------------------------------------------------
// CTA-pair GEMM: a 2-CTA cluster owns a 256 x 256 output tile; the leader
// issues tcgen05.mma.cta_group::2 (M = 256) reading each CTA's 128 activation
// rows and 128 weight rows from that CTA's own smem.  A pair MMA runs at the
// full 4096 MAC/clk/SM where the 1-CTA SS M=128 N=256 form reaches 76 %
// (profiles/r01_umma_rates.md).  Per stage each CTA stages 16 KB of A and
// 16 KB of B, so 6 stages fit.
//   warp 0       producer (own CTA's halves), signals its own `full`
//   warp 1       leader: TMEM alloc + MMA issue; peer: TMEM alloc + forwards
//                its `full` completions to the leader's `full` (count 2)
//   warps 2-5    epilogue of the CTA's 128 rows; arrive on the leader's
//                `tempty` (count 8: both CTAs' epilogue warps)
constexpr int PAIR_BN = 256;
struct GemmPairCfg {
  static constexpr uint32_t A_BYTES = BM * BK * 2;               // 16 KB: this CTA's 128 rows
  static constexpr uint32_t B_BYTES = (PAIR_BN / 2) * BK * 2;    // 16 KB: this CTA's 128 weight rows
  static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = 6;
  static constexpr uint32_t TMEM_COLS = 2 * PAIR_BN;
  static constexpr size_t SMEM = 1024 + size_t(STAGES) * STAGE_BYTES + 256;
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(192, 1)
    k_gemm_pair(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmW,
                const GemmParams p) {
  using C = GemmPairCfg;
  constexpr int STAGES = C::STAGES;
  constexpr int BN = PAIR_BN;
  pdl_trigger();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * C::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  uint64_t* t_start = reinterpret_cast<uint64_t*>(tmem_slot + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmW);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);  // leader: its producer's expect_tx for both CTAs' bytes
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 8);  // used on the leader: 4 epilogue warps per CTA
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_pair(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  pdl_wait();  // activations / residual from the stream predecessor
  if (threadIdx.x == 0) *t_start = globaltimer();
  const uint32_t tmem_base = *tmem_slot;
  const int total = p.m_tiles * p.n_tiles;

  if (warp == 0) {
    // both CTAs' loads complete on the LEADER's `full` (pair TMA); the
    // leader's producer posts the expected bytes of both halves
    uint32_t g = 0;
    const uint32_t lfull = mapa_shared(full, 0);
    Seg w;
    for (int it = 0; work_item(p, pair, npairs, it, w); ++it) {
      int mt, nt;
      tile_coords(p, w.tile, mt, nt);
      for (int kb = w.kb0; kb < w.kb1; ++kb, ++g) {
        const int stage = g % STAGES;
        const uint32_t phase = (g / STAGES) & 1;
        mbar_wait(&empty[stage], phase ^ 1);
        if (elect_one()) {
          if (leader) mbar_arrive_expect_tx(&full[stage], 2 * C::STAGE_BYTES);
          const uint32_t bar = lfull + 8u * stage;
#if HP_GEMM_A_EVICT_LAST
          // activations are re-read by every n-tile of their m-group: ask L2
          // to keep them over a co-running decode's streams
          tma_load_2d_pair_hint(sA + stage * C::A_BYTES, &tmA, bar, kb * BK, mt * 2 * BM + int(rank) * BM,
                                l2_policy_evict_last());
#else
          tma_load_2d_pair(sA + stage * C::A_BYTES, &tmA, bar, kb * BK, mt * 2 * BM + int(rank) * BM);
#endif
          // weight rows of this CTA's half: one pre-swizzled [128][64] sub-tile
          // of the tiled layout, addressed as rows of a [*, 64] tensor
          const int wrow = int(wtile_offset(nt * BN + int(rank) * (BN / 2), kb, p.K) / 128);
          tma_load_2d_pair(sB + stage * C::B_BYTES, &tmW, bar, 0, wrow);
        }
        __syncwarp();
      }
    }
  } else if (warp == 1 && !leader) {
    // peer: nothing to issue (the leader drives the pair's tensor core)
  } else if (warp == 1) {
    // leader: MMA issue for the pair (converged walk, one elected lane)
    constexpr uint32_t idesc = umma_idesc_bf16(2 * BM, BN);
    const uint64_t adesc0 = umma_desc_sw128(smem_u32(sA));
    const uint64_t bdesc0 = umma_desc_sw128(smem_u32(sB));
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    Seg w;
    for (int it = 0; work_item(p, pair, npairs, it, w); ++it) {
      mbar_wait_cluster(&tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;
      for (int kb = w.kb0; kb < w.kb1; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        const uint64_t ad = adesc0 + uint64_t((stage * C::A_BYTES) >> 4);
        const uint64_t bd = bdesc0 + uint64_t((stage * C::B_BYTES) >> 4);
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            umma_bf16_pair(d_tmem, ad + 2 * k, bd + 2 * k, idesc, (kb > w.kb0 || k > 0) ? 1u : 0u);
          umma_commit_pair(&empty[stage]);
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      if (elect_one()) umma_commit_pair(&tfull[acc]);
      __syncwarp();
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  } else {
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const uint32_t ltempty = mapa_shared(tempty, 0);
    int acc = 0;
    uint32_t acc_phase = 0;
    Seg w;
    for (int it = 0; work_item(p, pair, npairs, it, w); ++it) {
      int mt, nt;
      tile_coords(p, w.tile, mt, nt);
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t taddr = tmem_base + (uint32_t(q * 32) << 16) + acc * BN;
      if (w.kind == 2) {
        // partial: raw fp32 accumulator to this pair's slot, then one arrival
        // per CTA on the tile's counter (every thread's stores fenced first)
        write_partial<BN>(taddr, p.sk_ws + size_t(pair) * SK_SLOT_FLOATS + size_t(rank) * (SK_SLOT_FLOATS / 2),
                          row);
        __threadfence();
        named_bar_sync(1, 128);
        if (threadIdx.x == 64) atomicAdd(p.sk_cnt + (w.tile - p.sk_dp) * 2 + int(rank), 1);
      } else {
        TailFix fx{nullptr, 0, 0, int(rank), row};
        if (w.kind == 1) {
          const int tr = w.tile - p.sk_dp;
          const int j0 = sk_first_contributor(p, tr, pair, npairs);
          if (threadIdx.x == 64) {
            int* c = p.sk_cnt + tr * 2 + int(rank);
            while (ld_acquire_gpu(c) < pair - j0) __nanosleep(32);
            *c = 0;  // every contributor has arrived: ready for the next launch
          }
          named_bar_sync(1, 128);
          __threadfence();
          fx = TailFix{p.sk_ws, j0, pair, int(rank), row};
        }
        epilogue_row<BN>(p, taddr, mt * 2 * BM + int(rank) * BM + row, nt, fx);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster_relaxed(ltempty + 8u * acc);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, C::TMEM_COLS);
  }
  if (p.cta_times != nullptr && threadIdx.x == 0) {
    p.cta_times[blockIdx.x * 3 + 0] = smid();
    p.cta_times[blockIdx.x * 3 + 1] = *t_start;
    p.cta_times[blockIdx.x * 3 + 2] = globaltimer();
  }
}

static int launch_pair(const CUtensorMap& ta, const GemmParams& p, int grid, cudaStream_t st) {
  static bool attr_set = false;
  if (!attr_set) {
    HP_CUDA_TRY(cudaFuncSetAttribute(k_gemm_pair, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(GemmPairCfg::SMEM)));
    attr_set = true;
  }
  // the tiled weights viewed as a [N*K/64, 64] bf16 tensor: one 128-row box is
  // one pre-swizzled [128][64] sub-tile, copied verbatim (no TMA swizzle)
  CUtensorMap tw;
  int rc = cached_tmap_bf16(&tw, p.w, uint64_t(p.Nb) * p.K / 64, 64, 64, 128, 64, false);
  if (rc) return rc;
  HP_LAUNCH_PDL("k_gemm_pair", k_gemm_pair, dim3(grid), dim3(192), GemmPairCfg::SMEM, st, ta, tw, p);
  return HP_OK;
}

template <int BN>
static int launch(const CUtensorMap& ta, const GemmParams& p, int grid, cudaStream_t st) {
  using C = GemmCfg<BN>;
  static bool attr_set = false;
  if (!attr_set) {
    HP_CUDA_TRY(cudaFuncSetAttribute(k_gemm_tc<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(C::SMEM)));
    attr_set = true;
  }
  HP_LAUNCH_PDL("k_gemm_tc", k_gemm_tc<BN>, dim3(grid), dim3(192), C::SMEM, st, ta, p);
  return HP_OK;
}

static int ceil_div(int a, int b) { return (a + b - 1) / b; }

}  // namespace hp

using namespace hp;

extern "C" int hp_gemm_traced(const void* X, int ldx, const void* W, int ldw, void* Y, int ldy,
                              const void* R, int ldr, int T, int N, int K, int epilogue, int max_ctas,
                              uint64_t* cta_times, void* stream);

// Pair mode (CTA-pair 256 x 256 tiles) unless HP_GEMM_PAIR=0, the tile
// width is 128, or the partition has a single SM.
static bool use_pair(int BN, int max_ctas) {
  static const bool on = [] {
    const char* e = std::getenv("HP_GEMM_PAIR");
    return !(e && e[0] == '0');
  }();
  return on && BN == PAIR_BN && max_ctas >= 2;
}

// Stream-K tail policy.  Measured (tools/tail_layer_ab.py,
// profiles/r02_gemm_tail_ab.jsonl): a last round with fewer busy pairs runs
// its tiles faster than the wave model's equal-tile assumption (less HBM /
// power contention), and the fix-up costs a few microseconds per finishing
// tile (latency-bound partial reads in the epilogue), so splitting pays only
// for long-K GEMMs (>= 128 k-blocks: the down projection) whose last round
// would leave at least half of the pairs idle.  Then the last full round +
// the partial one are split (units > P), or every tile (units < P).
static bool tail_plan(int units, int P, int num_kb, int* dp, int* tail) {
  *dp = units;
  *tail = 0;
  if (!gemm_tail_mode() || P < 2 || P > SK_MAX_PAIRS || num_kb < 128) return false;
  if (units > P) {
    const int R = units % P;
    if (R == 0 || 2 * R > P) return false;
    *dp = (units / P - 1) * P;
  } else {
    if (2 * units > P) return false;
    *dp = 0;
  }
  *tail = units - *dp;
  return long(*tail) * num_kb >= 8l * P;
}

static bool use_pair(int BN, int max_ctas);

// Fill the tile geometry of `p` (T x N output, K reduction) and launch the
// 1-CTA kernel or the CTA-pair kernel on at most `max_ctas` SMs.
static int plan_and_launch(const CUtensorMap& ta, GemmParams& p, int T, int N, int K, int BN, int max_ctas,
                           cudaStream_t st) {
  const bool pair = use_pair(BN, max_ctas);
  const int rows = pair ? 2 * BM : BM;
  p.Ma = T;
  p.Nb = N;
  p.K = K;
  p.m_tiles = ceil_div(T, rows);
  p.n_tiles = N / BN;
  p.k_splits = 1;
  p.num_kb = K / BK;
  p.kb_per_split = p.num_kb;
  // rasterization group: keep the activation block of a group within ~32 MB
  // of the 126 MB L2 (decode traffic shares it during co-execution)
  const long a_tile_bytes = long(rows) * K * 2;
  const long budget = 32l << 20;
  p.group_m = a_tile_bytes * p.m_tiles <= 2 * budget ? p.m_tiles
                                                     : int(std::max<long>(pair ? 4 : 8, budget / a_tile_bytes));
  const int units = p.m_tiles * p.n_tiles;
  p.sk_dp = units;
  p.sk_tail = 0;
  if (pair) {
    int P = std::min(units, max_ctas / 2);
    int dp = 0, tail = 0;
    SkWorkspace ws{};
    if (tail_plan(units, max_ctas / 2, p.num_kb, &dp, &tail) && sk_workspace(st, &ws) == HP_OK) {
      P = max_ctas / 2;
      p.sk_dp = dp;
      p.sk_tail = tail;
      p.sk_ws = ws.ws;
      p.sk_cnt = ws.cnt;
    }
    return launch_pair(ta, p, 2 * P, st);
  }
  const int grid = std::min(units, max_ctas);
  return BN == 128 ? launch<128>(ta, p, grid, st) : launch<256>(ta, p, grid, st);
}

static int gemm_bn(int T, int N, int K, int ctas);

extern "C" int hp_gemm_qkv_rope(const void* X, int ldx, const void* W, int ldw, void* Y, int ldy, int T,
                                int Hq, int Hkv, int d, int K, const int* positions, const float* cos_sin,
                                const int* slot_mapping, void* kcache, void* vcache, int page, int max_ctas,
                                void* stream) {
  HP_CHECK_ARG(X && W && Y && positions && cos_sin && slot_mapping && kcache && vcache,
               "hp_gemm_qkv_rope: null pointer");
  HP_CHECK_ARG(T >= 1 && K % 128 == 0 && ldw == K, "hp_gemm_qkv_rope: K must be a multiple of 128 (tiled W)");
  HP_CHECK_ARG(d == 64 || d == 128, "hp_gemm_qkv_rope: head_dim must be 64 or 128");
  HP_CHECK_ARG(Hq >= 1 && Hkv >= 1 && Hq % Hkv == 0, "hp_gemm_qkv_rope: bad head counts");
  HP_CHECK_ARG(page >= 64 && page % 64 == 0 && max_ctas >= 1, "hp_gemm_qkv_rope: page must be a multiple of 64");
  const int N = (Hq + 2 * Hkv) * d;
  HP_CHECK_ARG(N % 128 == 0 && ldy >= N && ldy % 8 == 0, "hp_gemm_qkv_rope: (Hq+2Hkv)*d must be a multiple of 128");
  const int BN = gemm_bn(T, N, K, max_ctas);
  CUtensorMap ta;
  int rc = cached_tmap_bf16(&ta, X, T, K, ldx, BM, BK, true);
  if (rc) return rc;
  GemmParams p{};
  p.w = static_cast<const uint8_t*>(W);
  p.out = static_cast<__nv_bfloat16*>(Y);
  p.ldo = ldy;
  p.epi = EPI_ROPE;
  p.pos = positions;
  p.cos_sin = cos_sin;
  p.slots = slot_mapping;
  p.kc = static_cast<__nv_bfloat16*>(kcache);
  p.vc = static_cast<__nv_bfloat16*>(vcache);
  p.page = page;
  p.Hq = Hq;
  p.Hkv = Hkv;
  p.hd = d;
  p.cta_times = take_cta_trace();
  return plan_and_launch(ta, p, T, N, K, BN, max_ctas, static_cast<cudaStream_t>(stream));
}

extern "C" int hp_gemm(const void* X, int ldx, const void* W, int ldw, void* Y, int ldy,
                       const void* R, int ldr, int T, int N, int K, int epilogue, int max_ctas,
                       void* stream) {
  return hp_gemm_traced(X, ldx, W, ldw, Y, ldy, R, ldr, T, N, K, epilogue, max_ctas, take_cta_trace(), stream);
}

// Tile-width choice for a partition of `ctas` SMs.  A persistent grid over
// `tiles` runs ceil(tiles / ctas) rounds (wave_stats, perf_model.py:157-169);
// halving BN doubles the tile count, which can cut the rounds' total width
// when few tiles are left for the last wave (T = 1024 qkv on 148 SMs: 192
// tiles of 256 = 2 rounds x 256 cols vs 384 tiles of 128 = 3 x 128).  A
// 128-wide tile is 15-30 % slower per FLOP on B200 (tools/gemm_bn_sweep.py:
// the activation tile is re-streamed per 128 columns and the MMA is half
// as wide), folded in as 1.25.
// HP_GEMM_BN=128|256 forces a width (measurement).
static int gemm_bn(int T, int N, int K, int ctas) {
  static const int forced = [] {
    const char* e = std::getenv("HP_GEMM_BN");
    return e ? std::atoi(e) : 0;
  }();
  if (forced == 128 || (forced == 256 && N % 256 == 0)) return forced;
  if (N % 256 != 0) return 128;
  const int m = (T + BM - 1) / BM;
  const long t256 = long(m) * (N / 256), t128 = long(m) * (N / 128);
  double c256 = double((t256 + ctas - 1) / ctas) * 256.0;
  if (ctas >= 4 && use_pair(256, ctas)) {  // pair tiles: 256-row units over ctas / 2 pairs
    const int units = ((T + 2 * BM - 1) / (2 * BM)) * (N / 256);
    int dp = 0, tail = 0;
    if (tail_plan(units, ctas / 2, K / BK, &dp, &tail))
      c256 = (double(units) / (ctas / 2) + 0.1) * 256.0;  // rounds spread evenly, + fix-up
    else
      c256 = double((units + ctas / 2 - 1) / (ctas / 2)) * 256.0;
  }
  const double c128 = double((t128 + ctas - 1) / ctas) * 128.0 * 1.25;
  return c128 < c256 ? 128 : 256;
}

extern "C" int hp_gemm_tiles(int T, int N) { return ((T + BM - 1) / BM) * (N / 256); }

extern "C" int hp_gemm_plan(int T, int N, int K, int max_ctas, int* bn, int* tiles, int* ctas_per_tile,
                            int* tail_tiles) {
  HP_CHECK_ARG(T >= 1 && N % 128 == 0 && K % 128 == 0 && max_ctas >= 1, "hp_gemm_plan: bad shape");
  const int b = gemm_bn(T, N, K, max_ctas);
  const bool pair = use_pair(b, max_ctas);
  const int rows = pair ? 2 * BM : BM;
  const int t = ((T + rows - 1) / rows) * (N / b);
  int dp = 0, tail = 0;
  if (!pair || !tail_plan(t, max_ctas / 2, K / BK, &dp, &tail)) tail = 0;
  if (bn) *bn = b;
  if (tiles) *tiles = t;
  if (ctas_per_tile) *ctas_per_tile = pair ? 2 : 1;
  if (tail_tiles) *tail_tiles = tail;
  return HP_OK;
}

extern "C" int hp_gemm_traced(const void* X, int ldx, const void* W, int ldw, void* Y, int ldy,
                              const void* R, int ldr, int T, int N, int K, int epilogue, int max_ctas,
                              uint64_t* cta_times, void* stream) {
  HP_CHECK_ARG(X && W && Y, "hp_gemm: null pointer");
  HP_CHECK_ARG(T >= 1 && N >= 1 && K >= 1, "hp_gemm: empty problem");
  HP_CHECK_ARG(K % 128 == 0, "hp_gemm: K must be a multiple of 128 (tiled weight layout)");
  HP_CHECK_ARG(epilogue >= EPI_STORE && epilogue <= EPI_SILU, "hp_gemm: bad epilogue");
  HP_CHECK_ARG(epilogue != EPI_RESID || R != nullptr, "hp_gemm: residual epilogue needs R");
  HP_CHECK_ARG(max_ctas >= 1, "hp_gemm: max_ctas must be >= 1");
  HP_CHECK_ARG(N % 128 == 0, "hp_gemm: N must be a multiple of 128 (tiled weight layout)");
  HP_CHECK_ARG(ldw == K, "hp_gemm: W must be in the tiled layout (ldw == K)");
  const int BN = gemm_bn(T, N, K, max_ctas);
  CUtensorMap ta;
  int rc = cached_tmap_bf16(&ta, X, T, K, ldx, BM, BK, true);
  if (rc) return rc;
  GemmParams p{};
  p.w = static_cast<const uint8_t*>(W);
  p.out = static_cast<__nv_bfloat16*>(Y);
  p.ldo = ldy;
  p.resid = static_cast<const __nv_bfloat16*>(R);
  p.ldr = ldr;
  p.epi = epilogue;
  p.cta_times = cta_times;
  return plan_and_launch(ta, p, T, N, K, BN, max_ctas, static_cast<cudaStream_t>(stream));
}

