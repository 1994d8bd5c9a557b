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
// k_decode_combine.  A group of 16 heads at d = 64 (the moe-a22b preset's
// 64 q / 4 kv heads) uses two N=8 column blocks per K/V fragment (NB = 2:
// every K and V ldmatrix feeds two MMAs); other groups above 8 run as
// Gb-head blocks of
// one unit each, sibling units adjacent in the unit order so the later
// blocks' K/V reads are L2 hits of the first's (no evict-first hint then).
//
// Caches must not hold NaN/Inf in unused slots of partially filled pages
// (allocate them zeroed): masked probabilities are exactly 0, but 0 * NaN is
// NaN inside the MMA.
#include "common.cuh"
#include "runtime.h"
#include "../../include/hp.h"

#include <algorithm>
#include <cstdlib>
#include <cmath>

namespace hp {

constexpr int DA_TILE = 64;
constexpr int DA_CONSUMERS = 8;
#ifndef HP_DA_PRODUCERS
#define HP_DA_PRODUCERS 4
#endif
constexpr int DA_PRODUCERS = HP_DA_PRODUCERS;         // issuing warps (one copy stream each)
constexpr int DA_THREADS = (DA_CONSUMERS + DA_PRODUCERS) * 32;
constexpr uint32_t DA_BOX_BYTES = DA_TILE * 64 * 2;   // 64 rows x 128 B
constexpr int DA_WREG = 8;                            // block-table window regs per lane
constexpr int DA_WIN = 32 * DA_WREG;                  // window: pages per unit
constexpr int DA_MAX_RS = 32;                         // ring slots (tags array size)
constexpr size_t DA_SMEM_MAX = 227 * 1024;

// Shared-memory plan, computed on the host (ring depth depends on the GQA
// group through the merge buffer) and recomputed identically on the device.
struct DaPlan {
  int rs;               // ring slots (half-tiles), multiple of DA_PRODUCERS
  uint32_t hs;          // bytes per slot = one 64-token K or V tile
  int cb;               // per-warp merge buffer (floats)
  size_t smem;
};

// G = heads per unit (Gb), NB = 8-head column blocks (1 or 2)
inline size_t da_fixed_bytes(int D, int G, int NB) {
  const int cb = G * D + 16 * NB;
  return 1024 + size_t(DA_CONSUMERS) * cb * 4 +
         2 * DA_MAX_RS * 8 + DA_MAX_RS * 4 + 64;
}

inline DaPlan da_plan(int D, int G, int NB) {
  DaPlan pl;
  pl.hs = uint32_t(DA_TILE) * D * 2;
  pl.cb = G * D + 16 * NB;
  const size_t fixed = da_fixed_bytes(D, G, NB);
  int rs = int((DA_SMEM_MAX - fixed) / pl.hs);
  rs = std::min(rs, DA_MAX_RS);
  rs -= rs % DA_PRODUCERS;
  pl.rs = rs;
  pl.smem = fixed + size_t(rs) * pl.hs;
  return pl;
}

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
  int HB, Gb;       // head blocks per kv head, heads per block (min(G, 8))
  int tps;          // tiles per split
  int max_splits;
  int rs;           // ring slots
  float scale_log2;
  float* ws_o;      // [B, Hq, max_splits, D]
  float* ws_ml;     // [B, Hq, max_splits, 2]
};

// Context length of sequence b, clamped to what its block-table row can
// address (max_pages * page): a longer ctx_lens[b] (a caller bug, see hp.h)
// must not index split slots past max_splits or pages past the row.
__device__ __forceinline__ int da_ctx(const DecodeParams& p, int b) {
  return max(0, min(p.ctx_lens[b], p.max_pages * p.page));
}

#ifdef HP_DA_TRACE
// development aid: clock64 stamps of CTA 0 (consumers: 6 per tile for their
// first 16 tiles; producers: empty-wait start/end per half-tile, first 64)
__device__ long long g_da_trace[12][64][6];
__device__ long long g_da_utrace[64][4];  // consumer warp 0: unit start, tiles done, merged, end
#endif

struct UnitId {
  int b, kvh, s, hb;
};

__device__ __forceinline__ UnitId unit_of(const DecodeParams& p, int u) {
  UnitId id;
  id.hb = u % p.HB;
  u /= p.HB;
  id.s = u % p.max_splits;
  const int bh = u / p.max_splits;
  id.kvh = bh % p.Hkv;
  id.b = bh / p.Hkv;
  return id;
}

// Work unit = (sequence b, kv head, split s of `tps` 64-token tiles).  The
// CTA streams its units' tiles through a ring of `rs` slots, each holding
// one 64-token K or V tile (16 KB at D = 128, one contiguous run of the page
// layout [page/64][D/64][64][64]): half-slot h = 2 * tile + (0: K, 1: V).
//
// Producers: DA_PRODUCERS warps; warp w owns every slot s with s % P == w
// and issues the half-tiles h with h % P == w (rs % P == 0), so each slot is
// refilled by one thread in order and its empty-barrier waits are
// unambiguous.  One bulk copy per half-tile.  Each producer keeps the unit's
// block-table pages in registers (DA_WREG per lane, fetched one unit ahead)
// and resolves 32 of its positions at a time, one per lane (tile, K/V, page
// by warp shuffle); the serial part per copy is then one empty-barrier wait
// and one issue.  Resolving each position just before its copy (~420 of the
// ~800 cycles per copy, clock64 trace tools/da_trace.py) capped the ring at
// 124 GB/s per SM even without the math; batched, 142 (HP_DA_NOCOMPUTE) and
// 109.5 with it at 8 SMs (was 98).
//
// Consumers: DA_CONSUMERS warps take the unit's tiles round-robin.  The K
// slot is released as soon as the scores are in registers, the V slot after
// the P.V product, so a slot is held for one MMA chain, not a whole tile.
template <int D, int NB>
__global__ void __launch_bounds__(DA_THREADS, 1) k_decode_attn(const DecodeParams p) {
  pdl_trigger();
  constexpr int KK = D / 16;
  constexpr uint32_t HS = uint32_t(DA_TILE) * D * 2;
  constexpr int SO = 8 * NB;  // offset of the l (sum) stats after the m stats
  const int RS = p.rs;
  const int CB = p.Gb * D + 2 * SO;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* cbuf = reinterpret_cast<float*>(ring + size_t(RS) * HS);
  uint64_t* full = reinterpret_cast<uint64_t*>(cbuf + DA_CONSUMERS * CB);
  uint64_t* empty = full + DA_MAX_RS;
  // Consumers can reach a slot more than one phase ahead of its producer
  // (8 warps round-robin over the ring), where a parity wait would be
  // ambiguous: they first wait until the slot's tag names their half-tile
  // (written once the producer passed the slot's empty barrier for it).
  const uint32_t tag = smem_u32(empty + DA_MAX_RS);  // u32 [DA_MAX_RS], volatile shared accesses

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < RS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      st_volatile_shared(tag + 4u * s, 0xffffffffu);
    }
    fence_barrier_init();
  }
  __syncthreads();
  pdl_wait();  // q, K/V (incl. the token rope_kv_write just stored), block table

  const int total = p.B * p.Hkv * p.HB * p.max_splits;
  const int page_tiles = p.page / DA_TILE;

  if (warp >= DA_CONSUMERS) {
    // ------------------------------------------------------------ producers
    const int pw = warp - DA_CONSUMERS;
    // KV is read once per step -- unless sibling head blocks re-read it from L2
    const uint64_t pol = p.HB > 1 ? l2_policy_evict_last() : l2_policy_evict_first();
    int win[DA_WREG], winn[DA_WREG];
    auto fetch = [&](int u, int (&w)[DA_WREG]) -> int {  // returns ctx of unit u
      const UnitId id = unit_of(p, u);
      const int first = (id.s * p.tps) / page_tiles;
      const int last = min(p.max_pages, ((id.s + 1) * p.tps + page_tiles - 1) / page_tiles);
      const int* row = p.block_table + size_t(id.b) * p.max_pages;
#pragma unroll
      for (int r = 0; r < DA_WREG; ++r) {
        const int j = first + r * 32 + lane;
        w[r] = j < last ? row[j] : 0;
      }
      return da_ctx(p, id.b);
    };
    uint32_t hbase = 0;
    int u = blockIdx.x;
    int ctx_cur = u < total ? fetch(u, win) : 0;
    for (; u < total; u += gridDim.x) {
      const UnitId id = unit_of(p, u);
      const int ctx_nxt = (u + int(gridDim.x) < total) ? fetch(u + gridDim.x, winn) : 0;
      const int ntiles = (ctx_cur + DA_TILE - 1) / DA_TILE;
      const int t0 = id.s * p.tps;
      const int t1 = min(ntiles, t0 + p.tps);
      const int nh = 2 * max(0, t1 - t0);
      const int first = t0 / page_tiles;
      // Positions hh = pw', pw' + P, ... of this unit (pw' = this warp's
      // residue), 32 at a time: lane j resolves position hb + P*j (tile,
      // K/V, page via the lane-distributed window) up front, then the warp
      // walks the batch -- wait for the slot, lane j issues its copy -- so
      // the serial part per copy is one barrier wait and one issue.
      for (int hb = (pw - int(hbase % DA_PRODUCERS) + DA_PRODUCERS) % DA_PRODUCERS; hb < nh;
           hb += 32 * DA_PRODUCERS) {
        const int hh_l = hb + DA_PRODUCERS * lane;
        int kv_l = 0, t_l = t0, pr_l = 0;
        if (hh_l < nh) {
          t_l = t0 + (hh_l >> 1);  // half-tile 2t: K of tile t, 2t + 1: its V
          kv_l = hh_l & 1;
          pr_l = t_l / page_tiles - first;
        }
        int blk_l = 0;
#pragma unroll
        for (int r = 0; r < DA_WREG; ++r) {
          const int v = __shfl_sync(0xffffffffu, win[r], pr_l & 31);
          if ((pr_l >> 5) == r) blk_l = v;
        }
        const uint8_t* src_l = (kv_l ? p.vc : p.kc) +
                               ((size_t(blk_l) * p.Hkv + id.kvh) * page_tiles + (t_l % page_tiles)) * HS;
        const int cnt = min(32, (nh - hb + DA_PRODUCERS - 1) / DA_PRODUCERS);
        for (int j = 0; j < cnt; ++j) {
          const uint32_t h = hbase + hb + DA_PRODUCERS * j;
          const int st = int(h % RS);
#ifdef HP_DA_TRACE
          const long long tw0 = clock64();
#endif
          mbar_wait(&empty[st], ((h / RS) & 1) ^ 1);
#ifdef HP_DA_TRACE
          if (blockIdx.x == 0 && lane == 0 && j < 64 && hb < DA_PRODUCERS && u == int(blockIdx.x + 2 * gridDim.x)) {
            g_da_trace[8 + pw][j][0] = tw0;
            g_da_trace[8 + pw][j][1] = clock64();
          }
#endif
          if (lane == j) {
            mbar_arrive_expect_tx(&full[st], HS);
            bulk_load_hint(ring + size_t(st) * HS, src_l, HS, &full[st], pol);
            st_volatile_shared(tag + 4u * st, h);
          }
          __syncwarp();
        }
      }
      hbase += nh;
      ctx_cur = ctx_nxt;
#pragma unroll
      for (int r = 0; r < DA_WREG; ++r) win[r] = winn[r];
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  const int g8 = lane >> 2;  // MMA group id
  const int t4 = lane & 3;   // thread in group
  const int mat = lane >> 3;
  float* cw = cbuf + warp * CB;
  uint32_t hbase = 0;

  auto load_q = [&](int u, uint32_t (&qf)[NB][KK][2], int& ctx) {
    const UnitId id = unit_of(p, u);
    ctx = da_ctx(p, id.b);
#pragma unroll
    for (int nb = 0; nb < NB; ++nb) {
      const int hl = nb * 8 + g8;  // head within the unit
      const bool hv = hl < p.Gb;
      const __nv_bfloat16* qrow =
          p.q + size_t(id.b) * p.ldq + size_t(id.kvh * p.G + id.hb * p.Gb + (hv ? hl : 0)) * D;
#pragma unroll
      for (int kk = 0; kk < KK; ++kk) {
        const uint32_t lo = *reinterpret_cast<const uint32_t*>(qrow + kk * 16 + 2 * t4);
        const uint32_t hi = *reinterpret_cast<const uint32_t*>(qrow + kk * 16 + 2 * t4 + 8);
        qf[nb][kk][0] = hv ? lo : 0u;
        qf[nb][kk][1] = hv ? hi : 0u;
      }
    }
  };
  auto acquire = [&](uint32_t h) -> uint32_t {
    const int st = int(h % RS);
    while (ld_volatile_shared(tag + 4u * st) != h) __nanosleep(20);
    mbar_wait(&full[st], (h / RS) & 1);
    return uint32_t(st);
  };

  uint32_t qcur[NB][KK][2];
  int ctx_cur = 0;
  if (blockIdx.x < total) load_q(blockIdx.x, qcur, ctx_cur);

  for (int u = blockIdx.x; u < total; u += gridDim.x) {
    const UnitId id = unit_of(p, u);
    uint32_t qnxt[NB][KK][2];
    int ctx_nxt = 0;
    if (u + int(gridDim.x) < total) load_q(u + gridDim.x, qnxt, ctx_nxt);
    const int ctx = ctx_cur;
    const int ntiles = (ctx + DA_TILE - 1) / DA_TILE;
    const int t0 = id.s * p.tps;
    const int t1 = min(ntiles, t0 + p.tps);
#ifdef HP_DA_TRACE
    const int uix = (u - int(blockIdx.x)) / int(gridDim.x);
    const bool utr = blockIdx.x == 0 && threadIdx.x == 0 && uix < 64;
    if (utr) g_da_utrace[uix][0] = clock64();
#endif
    if (t0 < t1) {
      const int nt = t1 - t0;
      float o[NB][KK][4];
      float m0[NB], m1[NB], l0[NB], l1[NB];  // per block: heads 2t4, 2t4+1
#pragma unroll
      for (int nb = 0; nb < NB; ++nb) {
#pragma unroll
        for (int i = 0; i < KK; ++i) o[nb][i][0] = o[nb][i][1] = o[nb][i][2] = o[nb][i][3] = 0.f;
        m0[nb] = m1[nb] = -INFINITY;
        l0[nb] = l1[nb] = 0.f;
      }

      for (int i = warp; i < nt; i += DA_CONSUMERS) {
        uint32_t pf[NB][4][2];  // P^T B fragments of the PV MMA (per 16-token k-step)
        const uint32_t hk = hbase + 2 * i;
        const uint32_t hv = hk + 1;
#ifdef HP_DA_NOCOMPUTE  // experiment: stream the ring without the math
        {
          const uint32_t a = acquire(hk);
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[a]);
          const uint32_t b = acquire(hv);
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[b]);
          continue;
        }
#endif
        // ---- S^T = K . Q^T : four independent 16-token m tiles per column block
#ifdef HP_DA_TRACE
        const bool trc = blockIdx.x == 0 && lane == 0 && i / DA_CONSUMERS < 64 && u == int(blockIdx.x + 2 * gridDim.x);
        long long* tr = g_da_trace[warp][min(63, i / DA_CONSUMERS)];
        if (trc) tr[0] = clock64();
#endif
        const uint32_t sk = acquire(hk);
#ifdef HP_DA_TRACE
        if (trc) tr[1] = clock64();
#endif
        const uint32_t kb = smem_u32(ring + size_t(sk) * HS);
        float sc[NB][4][4];
#pragma unroll
        for (int nb = 0; nb < NB; ++nb)
#pragma unroll
          for (int mt = 0; mt < 4; ++mt) sc[nb][mt][0] = sc[nb][mt][1] = sc[nb][mt][2] = sc[nb][mt][3] = 0.f;
#pragma unroll
        for (int kk = 0; kk < KK; ++kk) {
#pragma unroll
          for (int mt = 0; mt < 4; ++mt) {
            const uint32_t r = mt * 16 + (mat & 1) * 8 + (lane & 7);
            const uint32_t c = (kk & 3) * 2 + (mat >> 1);
            uint32_t a[4];
            ldmatrix_x4(kb + (kk >> 2) * DA_BOX_BYTES + sw128(r, c), a[0], a[1], a[2], a[3]);
#pragma unroll
            for (int nb = 0; nb < NB; ++nb) mma_bf16_16816(sc[nb][mt], a, qcur[nb][kk]);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[sk]);  // K tile consumed
#ifdef HP_DA_TRACE
        if (trc) tr[2] = clock64();
#endif
        // ---- mask, scale, online softmax
        const int tokbase = (t0 + i) * DA_TILE;
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) {
          float tm0 = -INFINITY, tm1 = -INFINITY;
#pragma unroll
          for (int mt = 0; mt < 4; ++mt) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const bool valid = tokbase + mt * 16 + g8 + h * 8 < ctx;
              sc[nb][mt][2 * h] = valid ? sc[nb][mt][2 * h] * p.scale_log2 : -INFINITY;
              sc[nb][mt][2 * h + 1] = valid ? sc[nb][mt][2 * h + 1] * p.scale_log2 : -INFINITY;
              tm0 = fmaxf(tm0, sc[nb][mt][2 * h]);
              tm1 = fmaxf(tm1, sc[nb][mt][2 * h + 1]);
            }
          }
#pragma unroll
          for (int off = 4; off < 32; off <<= 1) {
            tm0 = fmaxf(tm0, __shfl_xor_sync(0xffffffffu, tm0, off));
            tm1 = fmaxf(tm1, __shfl_xor_sync(0xffffffffu, tm1, off));
          }
          const float n0 = fmaxf(m0[nb], tm0), n1 = fmaxf(m1[nb], tm1);
          const float a0 = exp2f(m0[nb] - n0), a1 = exp2f(m1[nb] - n1);
          m0[nb] = n0;
          m1[nb] = n1;
          l0[nb] *= a0;
          l1[nb] *= a1;
          // most tiles leave every row max unchanged (a == 1 exactly): skip
          if (__any_sync(0xffffffffu, (a0 != 1.f) || (a1 != 1.f))) {
#pragma unroll
            for (int dm = 0; dm < KK; ++dm) {
              o[nb][dm][0] *= a0;
              o[nb][dm][2] *= a0;
              o[nb][dm][1] *= a1;
              o[nb][dm][3] *= a1;
            }
          }
          // P^T as the PV MMA's B fragments, transposed in registers: the
          // lane's packed (token g8 [+8], heads 2t4, 2t4+1) pair is its
          // fragment of the 8x8 matrix [token][head]; movmatrix.trans hands
          // it (head g8, tokens 2t4, 2t4+1) -- b0 (tokens 0-7) / b1 (8-15)
#pragma unroll
          for (int mt = 0; mt < 4; ++mt) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const float p0 = exp2f(sc[nb][mt][2 * h] - n0);
              const float p1 = exp2f(sc[nb][mt][2 * h + 1] - n1);
              l0[nb] += p0;
              l1[nb] += p1;
              pf[nb][mt][h] = movmatrix_trans(pack_bf16(p0, p1));
            }
          }
        }
        // ---- O^T += V^T . P^T
#ifdef HP_DA_TRACE
        if (trc) tr[3] = clock64();
#endif
        const uint32_t sv = acquire(hv);
#ifdef HP_DA_TRACE
        if (trc) tr[4] = clock64();
#endif
        const uint32_t vb = smem_u32(ring + size_t(sv) * HS);
#pragma unroll
        for (int kt = 0; kt < 4; ++kt) {
#pragma unroll
          for (int dm = 0; dm < KK; ++dm) {
            const uint32_t r = kt * 16 + (mat >> 1) * 8 + (lane & 7);
            const uint32_t c = (dm & 3) * 2 + (mat & 1);
            uint32_t a[4];
            ldmatrix_x4_trans(vb + (dm >> 2) * DA_BOX_BYTES + sw128(r, c), a[0], a[1], a[2], a[3]);
#pragma unroll
            for (int nb = 0; nb < NB; ++nb) mma_bf16_16816(o[nb][dm], a, pf[nb][kt]);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[sv]);  // V tile consumed
#ifdef HP_DA_TRACE
        if (trc) tr[5] = clock64();
#endif
      }
      // ---- merge the consumer warps' (m, l, O) for the Gb live heads
      const int G = p.Gb;
#pragma unroll
      for (int nb = 0; nb < NB; ++nb) {
#pragma unroll
        for (int off = 4; off < 32; off <<= 1) {
          l0[nb] += __shfl_xor_sync(0xffffffffu, l0[nb], off);
          l1[nb] += __shfl_xor_sync(0xffffffffu, l1[nb], off);
        }
        const int ha = nb * 8 + 2 * t4, hb2 = ha + 1;
        const bool h0 = ha < G, h1 = hb2 < G;
#pragma unroll
        for (int dm = 0; dm < KK; ++dm) {
          if (h0) {
            cw[ha * D + dm * 16 + g8] = o[nb][dm][0];
            cw[ha * D + dm * 16 + g8 + 8] = o[nb][dm][2];
          }
          if (h1) {
            cw[hb2 * D + dm * 16 + g8] = o[nb][dm][1];
            cw[hb2 * D + dm * 16 + g8 + 8] = o[nb][dm][3];
          }
        }
        if (g8 == 0) {
          if (h0) {
            cw[G * D + ha] = m0[nb];
            cw[G * D + SO + ha] = l0[nb];
          }
          if (h1) {
            cw[G * D + hb2] = m1[nb];
            cw[G * D + SO + hb2] = l1[nb];
          }
        }
      }
#ifdef HP_DA_TRACE
      if (utr) g_da_utrace[uix][1] = clock64();
#endif
      named_bar_sync(1, DA_CONSUMERS * 32);
      const int nsplit = (ntiles + p.tps - 1) / p.tps;
      const int nw = min(DA_CONSUMERS, nt);  // warps that saw at least one tile
      constexpr int Q4 = D / 4;              // float4 groups per head row
      for (int e = threadIdx.x; e < G * Q4; e += DA_CONSUMERS * 32) {
        const int h = e / Q4;
        const int d4 = (e % Q4) * 4;
        float M = -INFINITY;
        for (int w = 0; w < nw; ++w) M = fmaxf(M, cbuf[w * CB + G * D + h]);
        float L = 0.f, acc[4] = {0.f, 0.f, 0.f, 0.f};
        for (int w = 0; w < nw; ++w) {
          const float* c = cbuf + w * CB;
          const float f = exp2f(c[G * D + h] - M);
          L += f * c[G * D + SO + h];
          const float4 v = *reinterpret_cast<const float4*>(c + h * D + d4);
          acc[0] += f * v.x;
          acc[1] += f * v.y;
          acc[2] += f * v.z;
          acc[3] += f * v.w;
        }
        const int head = id.kvh * p.G + id.hb * G + h;
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
#ifdef HP_DA_TRACE
      if (utr) g_da_utrace[uix][2] = clock64();
#endif
      named_bar_sync(1, DA_CONSUMERS * 32);
#ifdef HP_DA_TRACE
      if (utr) g_da_utrace[uix][3] = clock64();
#endif
      hbase += 2 * nt;
    }
#pragma unroll
    for (int nb = 0; nb < NB; ++nb)
#pragma unroll
      for (int kk = 0; kk < KK; ++kk) {
        qcur[nb][kk][0] = qnxt[nb][kk][0];
        qcur[nb][kk][1] = qnxt[nb][kk][1];
      }
    ctx_cur = ctx_nxt;
  }
}

// One warp per (sequence, head): log-sum-exp merge of the split partials.
template <int D>
__global__ void k_decode_combine(const DecodeParams p) {
  pdl_trigger();
  pdl_wait();
  const int warp_global = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp_global >= p.B * p.Hq) return;
  const int b = warp_global / p.Hq;
  const int head = warp_global % p.Hq;
  const int ntiles = (da_ctx(p, b) + DA_TILE - 1) / DA_TILE;
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

template <int D, int NB>
static int launch_decode(DecodeParams& p, int max_ctas, cudaStream_t st) {
  const DaPlan pl = da_plan(D, p.Gb, NB);
  p.rs = pl.rs;
  static bool attr = false;
  if (!attr) {
    HP_CUDA_TRY(cudaFuncSetAttribute(k_decode_attn<D, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(DA_SMEM_MAX)));
    attr = true;
  }
  const int units = p.B * p.Hkv * p.HB * p.max_splits;
  HP_LAUNCH_PDL("k_decode_attn", k_decode_attn<D, NB>, dim3(std::min(units, max_ctas)), dim3(DA_THREADS),
                pl.smem, st, p);
  if (p.max_splits > 1) {
    const int warps = p.B * p.Hq;
    HP_LAUNCH_PDL("k_decode_combine", k_decode_combine<D>, dim3((warps + 7) / 8), dim3(256), 0, st, p);
  }
  return HP_OK;
}

}  // namespace hp

using namespace hp;

#ifdef HP_DA_TRACE
extern "C" int hp_da_trace_read(long long* host) {
  if (cudaMemcpyFromSymbol(host + sizeof(g_da_trace) / 8, g_da_utrace, sizeof(g_da_utrace)) != cudaSuccess) return -1;
  return cudaMemcpyFromSymbol(host, g_da_trace, sizeof(g_da_trace)) == cudaSuccess ? 0 : -1;
}
#endif

extern "C" size_t hp_decode_attn_ws_bytes(int B, int Hq, int d, int max_splits) {
  return size_t(B) * Hq * max_splits * (d + 2) * sizeof(float);
}

// 8-head column blocks per unit: two for 16-head groups at d = 64 (at d = 128
// the doubled O accumulators would spill; those run as 8-head units).
static int da_nb(int G, int d) { return (G % 16 == 0 && d == 64) ? 2 : 1; }

// Tiles per split the launch below picks.  Every unit costs ~2 us of
// fixed work (merge, drain, the combine pass when split), and a lone SM
// streams ~100 GB/s, so: as few splits as keep >= max_ctas / 2 units
// (enough streaming SMs to saturate HBM), never below 2 (d = 128) / 4
// (d = 64) tiles per unit.  Measured (profiles/r01_decode_attn_tps.txt):
// B=32 ctx 2048 on 148 SMs, no split 44.8 us vs 52.6 at 8 tiles per unit.
static int decode_tps(int B, int Hq, int Hkv, int d, int max_pages, int page, int max_ctas) {
  const int max_tiles = max_pages * (page / DA_TILE);
  const int G = Hq / Hkv;
  const int units_per_split = B * Hkv * (G / std::min(G, 8 * da_nb(G, d)));  // x head blocks
  const int min_tps = d == 64 ? 4 : 2;
  static const int forced = [] {  // HP_DA_TPS=n: fixed tiles per split (measurement)
    const char* e = std::getenv("HP_DA_TPS");
    return e ? std::atoi(e) : 0;
  }();
  if (forced > 0) return std::max(1, std::min({forced, max_tiles, (DA_WIN - 1) * (page / DA_TILE)}));
  int splits = 1;
  while (long(units_per_split) * splits < max_ctas / 2 && (max_tiles + 2 * splits - 1) / (2 * splits) >= min_tps)
    splits *= 2;
  const int tps = (max_tiles + splits - 1) / splits;
  return std::max(1, std::min(tps, (DA_WIN - 1) * (page / DA_TILE)));  // unit pages fit the window
}

extern "C" int hp_decode_attn_launches(int B, int Hq, int Hkv, int d, int max_pages, int page, int max_ctas) {
  if (B < 1 || Hkv < 1 || Hq % Hkv || max_pages < 1 || page < DA_TILE || max_ctas < 1) return 0;
  const int max_tiles = max_pages * (page / DA_TILE);
  const int tps = decode_tps(B, Hq, Hkv, d, max_pages, page, max_ctas);
  return (max_tiles + tps - 1) / tps > 1 ? 2 : 1;
}

extern "C" int hp_decode_attn(const void* q, int ldq, const void* kcache, const void* vcache,
                              const int* block_table, int max_pages, const int* ctx_lens, void* out,
                              int ldo, int B, int Hq, int Hkv, int d, int page, int num_blocks,
                              float scale, void* workspace, size_t ws_bytes, int max_ctas,
                              void* stream) {
  HP_CHECK_ARG(q && kcache && vcache && block_table && ctx_lens && out, "hp_decode_attn: null pointer");
  HP_CHECK_ARG(d == 64 || d == 128, "hp_decode_attn: head_dim must be 64 or 128");
  HP_CHECK_ARG(page % DA_TILE == 0 && page >= DA_TILE, "hp_decode_attn: page must be a multiple of 64");
  HP_CHECK_ARG(Hkv >= 1 && Hq % Hkv == 0 && (Hq / Hkv <= 8 || (Hq / Hkv) % 8 == 0),
               "hp_decode_attn: GQA group must be <= 8 or a multiple of 8");
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
  const int NB = da_nb(p.G, d);
  p.Gb = std::min(p.G, 8 * NB);
  p.HB = p.G / p.Gb;
  p.page = page;
  p.scale_log2 = scale * 1.4426950408889634f;
  // split so that the unit count covers the grid ~4x, at least 2 tiles/unit
  const int max_tiles = max_pages * (page / DA_TILE);
  p.tps = decode_tps(B, Hq, Hkv, d, max_pages, page, max_ctas);
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
  if (NB == 2) return launch_decode<64, 2>(p, max_ctas, st);
  return d == 128 ? launch_decode<128, 1>(p, max_ctas, st) : launch_decode<64, 1>(p, max_ctas, st);
}
