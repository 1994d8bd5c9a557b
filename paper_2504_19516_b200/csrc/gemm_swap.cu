// Decode-side GEMMs (reference kernel groups qkv / o_proj / mlp_up_gate /
// mlp_down at phase "decode", workload.py:153-210): Y[T, N] = epi(X . W^T)
// with T <= 256 tokens.  The work is a pure weight stream (AI ~ 31), so the
// kernel is built to keep HBM busy from any partition size:
//
//   * swap-AB: W [N, K] is the UMMA A operand (M = 128 output features per
//     tile), X [T, K] the B operand (UMMA N = BN >= T), accumulator in TMEM;
//   * stream-K: the (tile, k-block) iteration space is cut into equal
//     contiguous ranges, one per CTA of the persistent grid, so every SM
//     streams the same number of weight bytes regardless of how many output
//     tiles exist (no wave quantization on the decode partition);
//   * tiles split across CTAs leave fp32 partials in a workspace; the last
//     contributor (arrival counter, self-resetting) sums them and runs the
//     epilogue.  Tiles owned by one CTA go straight from TMEM to the output.
//
// Epilogues: STORE, RESID (+R), SILU (W rows interleaved in 64-row gate/up
// blocks, so a 128-row tile yields 64 outputs).  Outputs are written through
// a padded shared-memory transpose so stores along the feature dim coalesce.
//
// Warp roles (288 threads): warps 0..3 copy producers (each owns every 4th
// pipeline stage: one thread's async-copy stream is serialised at roughly one
// memory latency per copy), warp 4 TMEM alloc + UMMA issuer, warps 5..8
// epilogue (TMEM lane quarter = warp % 4).
#include "common.cuh"
#include "runtime.h"
#include "../../include/hp.h"

#include <algorithm>
#include <cstdlib>

namespace hp {

namespace {

#ifndef HP_SWAP_W_EVICT_FIRST
#define HP_SWAP_W_EVICT_FIRST 1
#endif

constexpr int SBM = 128;
constexpr int SBK = 128;  // k per pipeline stage: one contiguous 32 KB weight tile
constexpr int VLD = 33;  // padded fp32 row of the epilogue transpose buffer
constexpr int SW_PRODUCERS = 4;
constexpr int SW_MMA = SW_PRODUCERS;
constexpr int SW_THREADS = (SW_PRODUCERS + 5) * 32;

template <int BN>
struct SwapCfg {
  static constexpr uint32_t A_BYTES = SBM * SBK * 2;
  static constexpr uint32_t B_BYTES = BN * SBK * 2;
  static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = BN >= 256 ? 2 : (BN >= 128 ? 3 : (BN >= 64 ? 4 : 5));
  static constexpr int PL = STAGES < SW_PRODUCERS ? STAGES : SW_PRODUCERS;  // issuing warps
  // independent accumulation chains: consecutive UMMAs into one TMEM
  // accumulator serialise on its latency (~150 cycles at N=32), so k-steps
  // rotate over NCH accumulators that the epilogue sums
  static constexpr int NCH = BN <= 64 ? 4 : (BN == 128 ? 2 : 1);
  static constexpr uint32_t ACC_COLS = NCH * BN;
  static constexpr uint32_t TMEM_COLS = (2 * ACC_COLS <= 64) ? 64 : (2 * ACC_COLS <= 128 ? 128 : (2 * ACC_COLS <= 256 ? 256 : 512));
  static constexpr size_t VBUF = size_t(SBM) * VLD * 4;
  static constexpr size_t SMEM = 1024 + size_t(STAGES) * STAGE_BYTES + VBUF + 256;
};

struct SwapParams {
  int N, T, K;
  int m_tiles, n_tiles, num_kb;  // m_tiles: 128-feature tiles
  int m_walk;       // feature tiles of the stream-K walk (m_tiles, or m_tiles / 2 for CTA pairs)
  int ipc;          // k-block iterations per CTA
  int total_iters;  // m_tiles * n_tiles * num_kb
  int max_contrib;
  __nv_bfloat16* out;
  int ldo;
  const __nv_bfloat16* resid;
  int ldr;
  float* ws;        // [tiles][max_contrib][128][BN]
  int* counters;    // [tiles], zero on entry and exit
  const uint8_t* w;  // weights in the tiled layout (hp_tile_weight)
  int epi;
  unsigned long long* trace;  // optional [grid][10] globaltimer stamps (hp_set_trace; development aid)
  // HP_EPI_PEER (row-parallel layers under tensor parallelism): the partial
  // tile goes to slot `rank` of every rank's receive buffer [world][T][N]
  // over peer memory, then flag [rank][tile] := epoch is raised on every rank.
  // Buffers are double: half (epoch & 1) at base + half * half_{out,flags};
  // epoch = *epoch_dev + 1 when epoch_dev is set (graph-replayable), else `epoch`.
  __nv_bfloat16* peer_out[HP_MAX_PEERS];
  int* peer_flags[HP_MAX_PEERS];
  size_t half_out, half_flags;
  const int* epoch_dev;
  int world, rank, epoch;
  int two_shot;     // 1: a tile goes only to its owner rank (feature tile mt % world)
  // SW_EPI_ROPE (decode QKV, hp_gemm_swap_qkv_rope): rotary embedding of the
  // q / k heads and the paged K / V write of the new tokens, fused
  const int* pos;
  const float* cos_sin;  // fp32 [max_pos, hd] = [cos(hd/2) | sin(hd/2)]
  const int* slots;
  __nv_bfloat16* kc;
  __nv_bfloat16* vc;
  int page, Hq, Hkv, hd;
};

constexpr int SW_EPI_ROPE = 4;  // internal epilogue id (after HP_EPI_PEER)

struct Seg {
  int tile, kb0, kb1;
};

__device__ __forceinline__ bool next_seg(const SwapParams& p, int& it, int end, Seg& s) {
  if (it >= end) return false;
  s.tile = it / p.num_kb;
  s.kb0 = it - s.tile * p.num_kb;
  s.kb1 = min(p.num_kb, s.kb0 + (end - it));
  it += s.kb1 - s.kb0;
  return true;
}

__device__ __forceinline__ float silu_f(float x) { return x / (1.0f + __expf(-x)); }

// Sum of the NCH accumulation chains (columns ch*BN apart) for 32 columns.
template <int BN, int NCH>
__device__ __forceinline__ void load_acc(uint32_t taddr, float* v) {
  tmem_ld32(taddr, v);
  if constexpr (NCH > 1) {
    float w[32];
#pragma unroll
    for (int ch = 1; ch < NCH; ++ch) {
      tmem_ld_wait();
      tmem_ld32(taddr + ch * BN, w);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] += w[j];
    }
  }
  tmem_ld_wait();
}

// Epilogue-warp barrier (128 threads, named barrier 1).
__device__ __forceinline__ void epi_sync() { named_bar_sync(1, 128); }

// Write a 128 x 32 fp32 chunk held in smem V (row = feature, col = token
// offset c0..c0+31) to the output.  et: 0..127 epilogue thread index.
template <int BN>
__device__ __forceinline__ void emit_chunk(const SwapParams& p, const float* V, int mt, int nt,
                                           int c0, int et, int ep) {
  const int lane = et & 31, w = et >> 5;
  if (p.epi == HP_EPI_SILU) {
    // 64 outputs per tile: feature r (gate) pairs with r + 64 (up)
    for (int j = w; j < 32; j += 4) {
      const int t = nt * BN + c0 + j;
      if (t >= p.T) break;
      const int r = 2 * lane;
      const float g0 = V[r * VLD + j], g1 = V[(r + 1) * VLD + j];
      const float u0 = V[(r + 64) * VLD + j], u1 = V[(r + 65) * VLD + j];
      *reinterpret_cast<uint32_t*>(p.out + size_t(t) * p.ldo + mt * 64 + r) =
          pack_bf16(silu_f(g0) * u0, silu_f(g1) * u1);
    }
  } else if (p.epi == SW_EPI_ROPE) {
    // the tile's 128 features are 128 / hd whole heads of the q | k | v
    // blocks; lane -> rotary pair (i, i + hd/2) at i = 2 lane mod hd/2, so the
    // warp covers all 64 pairs of the tile for token j.  Same arithmetic as
    // hp_rope_kv_write on the bf16 projection the unfused GEMM stores.
    const int half = p.hd / 2;
    const int pi = 2 * lane;
    const int hl = pi / half, i = pi % half;
    const int rlo = hl * p.hd + i, rhi = rlo + half;
    const int head = (mt * SBM) / p.hd + hl;
    const bool rot = head < p.Hq + p.Hkv;
    for (int j = w; j < 32; j += 4) {
      const int t = nt * BN + c0 + j;
      if (t >= p.T) break;
      uint32_t lo = pack_bf16(V[rlo * VLD + j], V[(rlo + 1) * VLD + j]);
      uint32_t hi = pack_bf16(V[rhi * VLD + j], V[(rhi + 1) * VLD + j]);
      if (rot) {
        const float* cs = p.cos_sin + size_t(p.pos[t]) * p.hd;
        float a0, b0, a1, b1;
        rope_rotate(bf16lo(lo), bf16lo(hi), cs[i], cs[half + i], a0, b0);
        rope_rotate(bf16hi(lo), bf16hi(hi), cs[i + 1], cs[half + i + 1], a1, b1);
        lo = pack_bf16(a0, a1);
        hi = pack_bf16(b0, b1);
      }
      __nv_bfloat16* row = p.out + size_t(t) * p.ldo + size_t(head) * p.hd;
      *reinterpret_cast<uint32_t*>(row + i) = lo;
      *reinterpret_cast<uint32_t*>(row + half + i) = hi;
      if (head >= p.Hq) {
        const int slot = p.slots[t];
        const int blk = slot / p.page, off = slot % p.page;
        const int kvh = rot ? head - p.Hq : head - p.Hq - p.Hkv;
        __nv_bfloat16* cache = rot ? p.kc : p.vc;
        *reinterpret_cast<uint32_t*>(cache + kv_cache_index(blk, p.Hkv, kvh, p.page, off, p.hd, i)) = lo;
        *reinterpret_cast<uint32_t*>(cache + kv_cache_index(blk, p.Hkv, kvh, p.page, off, p.hd, half + i)) = hi;
      }
    }
  } else if (p.epi == HP_EPI_PEER) {
    // 16-byte stores: thread -> (token j, 8 consecutive features g*8..g*8+7)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int f = i * 128 + et, j = f >> 4, g = f & 15;
      const int t = nt * BN + c0 + j;
      if (t < p.T) {
        const float* c = V + (g * 8) * VLD + j;
        const uint4 v = make_uint4(pack_bf16(c[0], c[VLD]), pack_bf16(c[2 * VLD], c[3 * VLD]),
                                   pack_bf16(c[4 * VLD], c[5 * VLD]), pack_bf16(c[6 * VLD], c[7 * VLD]));
        const size_t off = (ep & 1) * p.half_out + (size_t(p.rank) * p.T + t) * p.N + mt * SBM + g * 8;
        if (p.two_shot)
          *reinterpret_cast<uint4*>(p.peer_out[mt % p.world] + off) = v;
        else
          for (int q = 0; q < p.world; ++q) *reinterpret_cast<uint4*>(p.peer_out[q] + off) = v;
      }
    }
  } else {
    for (int j = w; j < 32; j += 4) {
      const int t = nt * BN + c0 + j;
      if (t >= p.T) break;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = h * 64 + 2 * lane;
        float v0 = V[r * VLD + j], v1 = V[(r + 1) * VLD + j];
        const int o = mt * SBM + r;
        if (p.epi == HP_EPI_RESID) {
          const uint32_t rr = *reinterpret_cast<const uint32_t*>(p.resid + size_t(t) * p.ldr + o);
          v0 += bf16lo(rr);
          v1 += bf16hi(rr);
        }
        *reinterpret_cast<uint32_t*>(p.out + size_t(t) * p.ldo + o) = pack_bf16(v0, v1);
      }
    }
  }
}

// Epilogue warps of the decode GEMM (both kernels): per stream-K segment,
// whole tiles go TMEM -> smem transpose -> output; split tiles leave fp32
// partials and the last contributor sums them.  cid: this CTA's (or pair's)
// contributor index in the walk; PAIR: rank = CTA in the pair, TMEM release
// goes to the leader's `tempty` (both CTAs' epilogue warps arrive).
template <int BN, int NCH, bool PAIR>
__device__ __forceinline__ void swap_epilogue(const SwapParams& p, float* V, uint64_t* tfull, uint64_t* tempty,
                                              int* last_flag, uint32_t tmem_base, int begin, int end, int cid,
                                              uint32_t rank) {
  const uint32_t ltempty = PAIR ? mapa_shared(tempty, 0) : 0u;
  auto release = [&](int acc) {
    if (PAIR)
      mbar_arrive_cluster_relaxed(ltempty + 8u * acc);
    else
      mbar_arrive(&tempty[acc]);
  };
pdl_wait();  // residual, workspace and output are shared with the stream predecessor
const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
const int q = warp & 3;
  const int row = q * 32 + lane;
  const int et = (warp - SW_MMA - 1) * 32 + lane;
  // HP_EPI_PEER: this call's epoch (after pdl_wait: the previous reduce
  // advanced *epoch_dev); once the whole tile sits in every rank's receive
  // buffer, publish it with a system-scope release on every rank's flags
  const int ep = p.epi != HP_EPI_PEER ? 0 : (p.epoch_dev ? *p.epoch_dev + 1 : p.epoch);
  auto publish = [&](int tile) {
    if (p.epi != HP_EPI_PEER) return;
    epi_sync();
    if (et == 0) {
      __threadfence_system();
      const size_t f = (ep & 1) * p.half_flags + size_t(p.rank) * (p.m_tiles * p.n_tiles) + tile;
      if (p.two_shot)
        st_relaxed_sys(p.peer_flags[(tile % p.m_tiles) % p.world] + f, ep);
      else
        for (int r = 0; r < p.world; ++r) st_relaxed_sys(p.peer_flags[r] + f, ep);  // fenced above
    }
  };
  int acc = 0;
  uint32_t acc_phase = 0;
  int it = begin;
  Seg s;
  while (next_seg(p, it, end, s)) {
    const int mw = s.tile % p.m_walk, nt = s.tile / p.m_walk;
    const int mt = PAIR ? 2 * mw + int(rank) : mw;  // this CTA's 128-feature tile
    const int t128 = nt * p.m_tiles + mt;           // its workspace / counter / flag slot
    const int first = (s.tile * p.num_kb) / p.ipc;
    const int last = ((s.tile + 1) * p.num_kb - 1) / p.ipc;
    const bool single = first == last;
    mbar_wait(&tfull[acc], acc_phase);
    tc_fence_after();
    const uint32_t taddr = tmem_base + (uint32_t(q * 32) << 16) + acc * (NCH * BN);
    if (single) {
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        float v[32];
        load_acc<BN, NCH>(taddr + c * 32, v);
        if (c == BN / 32 - 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) release(acc);
        }
        epi_sync();  // previous chunk's readers are done with V
#pragma unroll
        for (int j = 0; j < 32; ++j) V[row * VLD + j] = v[j];
        epi_sync();
        emit_chunk<BN>(p, V, mt, nt, c * 32, et, ep);
      }
      publish(t128);
    } else {
      float* mine = p.ws + (size_t(t128) * p.max_contrib + (cid - first)) * (SBM * BN) +
                    size_t(row) * BN;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        float v[32];
        load_acc<BN, NCH>(taddr + c * 32, v);
#pragma unroll
        for (int j = 0; j < 32; j += 4)
          *reinterpret_cast<float4*>(mine + c * 32 + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) release(acc);
      __threadfence();
      epi_sync();
      unsigned long long* etr = (p.trace && et == 0) ? p.trace + blockIdx.x * 10 : nullptr;
      if (etr) etr[6] = globaltimer();  // partial written
      if (et == 0) {
        const int prev = atomicAdd(p.counters + t128, 1);
        *last_flag = (prev == last - first) ? 1 : 0;
      }
      epi_sync();
      if (etr) etr[7] = globaltimer();  // arrival counted
      if (*last_flag) {
        __threadfence();
        const int ncontrib = last - first + 1;
        const float* base = p.ws + size_t(t128) * p.max_contrib * (SBM * BN);
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          // 128 rows x 32 cols chunk: 1024 float4, 8 per thread
          float4 a[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) a[i] = make_float4(0.f, 0.f, 0.f, 0.f);
          // two contributors per round with all 16 loads in flight (the
          // partials are L2 hits; a one-at-a-time loop paid one L2 round
          // trip per contributor on the GEMM's critical tail)
          auto ld = [&](int k, int i) {
            const int f = i * 128 + et;            // float4 index within the chunk
            const int r = f >> 3, cc = (f & 7) * 4;
            return __ldcg(reinterpret_cast<const float4*>(base + size_t(k) * (SBM * BN) + size_t(r) * BN +
                                                          c * 32 + cc));
          };
          int k = 0;
          for (; k + 1 < ncontrib; k += 2) {
            float4 x0[8], x1[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              x0[i] = ld(k, i);
              x1[i] = ld(k + 1, i);
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              a[i].x += x0[i].x; a[i].y += x0[i].y; a[i].z += x0[i].z; a[i].w += x0[i].w;
              a[i].x += x1[i].x; a[i].y += x1[i].y; a[i].z += x1[i].z; a[i].w += x1[i].w;
            }
          }
          if (k < ncontrib) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const float4 x = ld(k, i);
              a[i].x += x.x; a[i].y += x.y; a[i].z += x.z; a[i].w += x.w;
            }
          }
          epi_sync();
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int f = i * 128 + et;
            const int r = f >> 3, cc = (f & 7) * 4;
            V[r * VLD + cc] = a[i].x;
            V[r * VLD + cc + 1] = a[i].y;
            V[r * VLD + cc + 2] = a[i].z;
            V[r * VLD + cc + 3] = a[i].w;
          }
          epi_sync();
          if (etr) etr[8] = globaltimer();  // partials summed
          emit_chunk<BN>(p, V, mt, nt, c * 32, et, ep);
        }
        if (etr) etr[9] = globaltimer();  // tile emitted
        if (et == 0) p.counters[t128] = 0;
        publish(t128);
      }
    }
    acc ^= 1;
    if (acc == 0) acc_phase ^= 1;
  }
}

}  // namespace

template <int BN>
__global__ void __launch_bounds__(SW_THREADS, 1)
    k_gemm_swap_sk(const __grid_constant__ CUtensorMap tmX,
                   const SwapParams p) {
  using C = SwapCfg<BN>;
  constexpr int STAGES = C::STAGES;
  pdl_trigger();
  if (p.trace && threadIdx.x == 0) p.trace[blockIdx.x * 10] = globaltimer();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * C::A_BYTES;
  float* V = reinterpret_cast<float*>(smem + STAGES * C::STAGE_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(V) + C::VBUF);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  int* last_flag = reinterpret_cast<int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmX);
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
  if (warp == SW_MMA) {
    tmem_alloc(tmem_slot, C::TMEM_COLS);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  unsigned long long* tr = p.trace ? p.trace + blockIdx.x * 10 : nullptr;
  if (tr && threadIdx.x == 0) tr[1] = globaltimer();

  const int begin = blockIdx.x * p.ipc;
  const int end = min(begin + p.ipc, p.total_iters);

  if (warp < SW_PRODUCERS) {
    constexpr int PL = C::PL;  // <= STAGES keeps parity waits unambiguous; extra warps idle
    // warp-converged walk (uniform registers), one elected lane issues
    {
      const uint64_t w_policy = l2_policy_evict_first();  // weights: read once per step
      // Weights are constant across the layer chain, so the first ring's worth
      // of weight tiles is fetched BEFORE the programmatic-dependency wait,
      // overlapping the predecessor kernel's tail; activation tiles follow it.
      for (int pass = 0; pass < 2; ++pass) {
        uint32_t g = 0;
        int it = begin;
        Seg s;
        while (next_seg(p, it, end, s)) {
          const int mt = s.tile % p.m_tiles, nt = s.tile / p.m_tiles;
          for (int kb = s.kb0; kb < s.kb1; ++kb, ++g) {
            const bool pre = g < uint32_t(STAGES);  // stage issued in pass 0 (weights only)
            if (int(g % PL) != warp || (pass == 0 && !pre)) continue;
            const int stage = g % STAGES;
            const uint32_t phase = (g / STAGES) & 1;
            if (pass == 0 || !pre) {
              mbar_wait(&empty[stage], phase ^ 1);
              if (elect_one()) {
                mbar_arrive_expect_tx(&full[stage], C::STAGE_BYTES);
                // 128 rows x 128 k of W: one contiguous 32 KB run (two swizzled 64-k halves)
                bulk_load_hint(sA + stage * C::A_BYTES, p.w + wtile_offset(mt * SBM, 2 * kb, p.K), C::A_BYTES,
                               &full[stage], w_policy);
              }
            }
            if (pass == 1 && elect_one()) {
              tma_load_2d(sB + stage * C::B_BYTES, &tmX, &full[stage], kb * SBK, nt * BN);
              tma_load_2d(sB + stage * C::B_BYTES + BN * 128, &tmX, &full[stage], kb * SBK + 64, nt * BN);
            }
            __syncwarp();
          }
          if (pass == 0 && g >= uint32_t(STAGES)) break;
        }
        if (pass == 0) pdl_wait();  // X is produced by the stream predecessor
      }
      if (tr && warp == 0 && lane == 0) tr[2] = globaltimer();
    }
  } else if (warp == SW_MMA) {
    // The whole warp walks the (warp-uniform) schedule so descriptors live in
    // uniform registers; one elected lane issues.  A divergent single-lane
    // issuer paid ~150 cycles of register shuffling per tcgen05.mma, which
    // capped a 16 KB stage of four N=32 MMAs at ~55 GB/s per SM.
    constexpr uint32_t idesc = umma_idesc_bf16(SBM, BN);
    const uint64_t adesc0 = umma_desc_sw128(smem_u32(sA));
    const uint64_t bdesc0 = umma_desc_sw128(smem_u32(sB));
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    int it = begin;
    Seg s;
    while (next_seg(p, it, end, s)) {
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * C::ACC_COLS;
      for (int kb = s.kb0; kb < s.kb1; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        const uint64_t ad = adesc0 + uint64_t((stage * C::A_BYTES) >> 4);
        const uint64_t bd = bdesc0 + uint64_t((stage * C::B_BYTES) >> 4);
        const bool first = kb == s.kb0;
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < SBK / 16; ++k)  // k-steps of 16: 4 per 64-k swizzled half
            umma_bf16(d_tmem + (k % C::NCH) * BN, ad + (k >> 2) * (128 * 128 >> 4) + 2 * (k & 3),
                      bd + (k >> 2) * (BN * 128 >> 4) + 2 * (k & 3), idesc,
                      (!first || k >= C::NCH) ? 1u : 0u);
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
    if (tr && lane == 0) tr[3] = globaltimer();
  } else {
    swap_epilogue<BN, C::NCH, false>(p, V, tfull, tempty, last_flag, tmem_base, begin, end, blockIdx.x, 0);
  }
  if (tr && threadIdx.x == (SW_MMA + 1) * 32) tr[4] = globaltimer();
  tc_fence_before();
  __syncthreads();
  if (warp == SW_MMA) {
    tc_fence_after();
    tmem_dealloc(tmem_base, C::TMEM_COLS);
  }
  if (tr && threadIdx.x == 0) tr[5] = globaltimer();
}

// ---------------------------------------------------------------------------
// CTA-pair variant: a 2-CTA cluster owns 256 output features; the leader
// issues tcgen05.mma.cta_group::2 (M = 256) with each CTA's 128 weight rows
// and half of the BN tokens in its own smem.  At N = BN = 32 one pair MMA
// runs at 41 % of the pair's MAC rate where the 1-CTA form manages 18 %
// (profiles/r01_umma_rates.md), which is what caps a small decode partition:
// 8 MMAs per 32 KB weight stage take ~710 cycles on one SM (~107 GB/s).
// Both CTAs' stage copies (TMA, .cta_group::2) complete on the leader's
// `full`; the leader's commits free both CTAs' stages (multicast).
template <int BN>
struct SwapPairCfg {
  static constexpr uint32_t A_BYTES = SBM * SBK * 2;       // this CTA's 128 weight rows
  static constexpr uint32_t B_BYTES = (BN / 2) * SBK * 2;  // this CTA's BN/2 tokens
  static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr size_t VBUF = size_t(SBM) * VLD * 4;
  static constexpr int STAGES_FIT = int((227 * 1024 - 1024 - VBUF - 256) / STAGE_BYTES);
  static constexpr int STAGES = STAGES_FIT < 6 ? STAGES_FIT : 6;
  static constexpr int PL = STAGES < SW_PRODUCERS ? STAGES : SW_PRODUCERS;
  static constexpr int NCH = SwapCfg<BN>::NCH;
  static constexpr uint32_t ACC_COLS = NCH * BN;
  static constexpr uint32_t TMEM_COLS = SwapCfg<BN>::TMEM_COLS;
  static constexpr size_t SMEM = 1024 + size_t(STAGES) * STAGE_BYTES + VBUF + 256;
};

template <int BN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(SW_THREADS, 1)
    k_gemm_swap_pair(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW,
                     const SwapParams p) {
  using C = SwapPairCfg<BN>;
  constexpr int STAGES = C::STAGES;
  pdl_trigger();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * C::A_BYTES;
  float* V = reinterpret_cast<float*>(smem + STAGES * C::STAGE_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(V) + C::VBUF);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  int* last_flag = reinterpret_cast<int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1;
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmX);
    tma_prefetch_desc(&tmW);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 8);  // on the leader: 4 epilogue warps per CTA
    }
    fence_barrier_init();
  }
  if (warp == SW_MMA) tmem_alloc_pair(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int begin = pair * p.ipc;
  const int end = min(begin + p.ipc, p.total_iters);

  if (warp < SW_PRODUCERS) {
    constexpr int PL = C::PL;
    const uint32_t lfull = mapa_shared(full, 0);
    // weights (constant across the layer chain) for the first ring before the
    // programmatic-dependency wait, activations after it
    for (int pass = 0; pass < 2; ++pass) {
      uint32_t g = 0;
      int it = begin;
      Seg s;
      while (next_seg(p, it, end, s)) {
        const int mw = s.tile % p.m_walk, nt = s.tile / p.m_walk;
        for (int kb = s.kb0; kb < s.kb1; ++kb, ++g) {
          const bool pre = g < uint32_t(STAGES);
          if (int(g % PL) != warp || (pass == 0 && !pre)) continue;
          const int stage = g % STAGES;
          const uint32_t phase = (g / STAGES) & 1;
          const uint32_t bar = lfull + 8u * stage;
          if (pass == 0 || !pre) {
            mbar_wait(&empty[stage], phase ^ 1);
            if (elect_one()) {
              if (leader) mbar_arrive_expect_tx(&full[stage], 2 * C::STAGE_BYTES);
              // this CTA's 128 x 128 weight block: one 32 KB run of the tiled layout
              const int wrow = int(wtile_offset((2 * mw + int(rank)) * SBM, 2 * kb, p.K) / 128);
#if HP_SWAP_W_EVICT_FIRST
              // weights are read once per step: keep them from displacing a
              // co-running prefill's L2 working set (as the 1-CTA kernel does)
              tma_load_2d_pair_hint(sA + stage * C::A_BYTES, &tmW, bar, 0, wrow, l2_policy_evict_first());
#else
              tma_load_2d_pair(sA + stage * C::A_BYTES, &tmW, bar, 0, wrow);
#endif
            }
          }
          if (pass == 1 && elect_one()) {
            const int t0 = nt * BN + int(rank) * (BN / 2);
            tma_load_2d_pair(sB + stage * C::B_BYTES, &tmX, bar, kb * SBK, t0);
            tma_load_2d_pair(sB + stage * C::B_BYTES + (BN / 2) * 128, &tmX, bar, kb * SBK + 64, t0);
          }
          __syncwarp();
        }
        if (pass == 0 && g >= uint32_t(STAGES)) break;
      }
      if (pass == 0) pdl_wait();
    }
  } else if (warp == SW_MMA) {
    if (leader) {
      constexpr uint32_t idesc = umma_idesc_bf16(2 * SBM, BN);
      const uint64_t adesc0 = umma_desc_sw128(smem_u32(sA));
      const uint64_t bdesc0 = umma_desc_sw128(smem_u32(sB));
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      int it = begin;
      Seg s;
      while (next_seg(p, it, end, s)) {
        mbar_wait_cluster(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * C::ACC_COLS;
        for (int kb = s.kb0; kb < s.kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t ad = adesc0 + uint64_t((stage * C::A_BYTES) >> 4);
          const uint64_t bd = bdesc0 + uint64_t((stage * C::B_BYTES) >> 4);
          const bool first = kb == s.kb0;
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < SBK / 16; ++k)
              umma_bf16_pair(d_tmem + (k % C::NCH) * BN, ad + (k >> 2) * (128 * 128 >> 4) + 2 * (k & 3),
                             bd + (k >> 2) * ((BN / 2) * 128 >> 4) + 2 * (k & 3), idesc,
                             (!first || k >= C::NCH) ? 1u : 0u);
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
    }
  } else {
    swap_epilogue<BN, C::NCH, true>(p, V, tfull, tempty, last_flag, tmem_base, begin, end, pair, rank);
  }
  tc_fence_before();
  cluster_sync();
  if (warp == SW_MMA) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, C::TMEM_COLS);
  }
}

template <int BN>
static int launch_swap_pair(const CUtensorMap& tx, const SwapParams& p, int grid, cudaStream_t st) {
  using C = SwapPairCfg<BN>;
  static bool attr_set = false;
  if (!attr_set) {
    HP_CUDA_TRY(cudaFuncSetAttribute(k_gemm_swap_pair<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(C::SMEM)));
    attr_set = true;
  }
  // the tiled weights as a [N*K/64, 64] bf16 tensor: one 256-row box is one
  // CTA's contiguous 32 KB stage (two pre-swizzled [128][64] halves, verbatim)
  CUtensorMap tw;
  int rc = cached_tmap_bf16(&tw, p.w, uint64_t(p.N) * p.K / 64, 64, 64, 256, 64, false);
  if (rc) return rc;
  HP_LAUNCH_PDL("k_gemm_swap_pair", k_gemm_swap_pair<BN>, dim3(grid), dim3(SW_THREADS), C::SMEM, st, tx, tw, p);
  HP_LAUNCH_CHECK("k_gemm_swap_pair");
  return HP_OK;
}

template <int BN>
static int launch_swap(const CUtensorMap& tx, const SwapParams& p, int grid,
                       cudaStream_t st) {
  using C = SwapCfg<BN>;
  static bool attr_set = false;
  if (!attr_set) {
    HP_CUDA_TRY(cudaFuncSetAttribute(k_gemm_swap_sk<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM)));
    attr_set = true;
  }
  HP_LAUNCH_PDL("k_gemm_swap_sk", k_gemm_swap_sk<BN>, dim3(grid), dim3(SW_THREADS), C::SMEM, st, tx, p);
  HP_LAUNCH_CHECK("k_gemm_swap_sk");
  return HP_OK;
}

static inline int swap_bn(int T) { return T <= 32 ? 32 : (T <= 64 ? 64 : (T <= 128 ? 128 : 256)); }

// Stream-K grid on a large partition: among [ceil(3 units / 4), units] CTAs,
// prefer a count whose per-CTA k range aligns with tile boundaries -- whole
// tiles per CTA (no fixup at all), or an even split of every tile (one
// segment per CTA) -- over a misaligned range whose CTAs straddle tiles and
// serialise on split-tile fixups (tools/swap_ctas.py, full GPU, T = 32:
// o_proj 14.4 -> 12.4 us at 128 CTAs, mlp_up_gate 38.9 -> 35.3 at 112,
// mlp_down 27.4 -> 23.6 at 128).  Below 64 units every SM's own streaming
// bandwidth counts (HBM is not the limit) and the walk uses all of them.
static int swap_grid(int total, int num_kb, int units) {
  const int g0 = std::max(1, std::min(units, total));
  if (units < 64) return g0;
  int best = g0;
  double best_score = 1e30;
  for (int c = g0; c >= (3 * units + 3) / 4; --c) {
    const int ipc = (total + c - 1) / c;
    const double pen = ipc % num_kb == 0 ? 0.0 : (num_kb % ipc == 0 ? 0.05 : 0.35);
    const double score = ipc * (1.0 + pen);
    if (score < best_score - 1e-9) {
      best_score = score;
      best = c;
    }
  }
  return best;
}

}  // namespace hp

using namespace hp;

extern "C" size_t hp_gemm_swap_ws_bytes(int T, int N, int K, int max_ctas) {
  const int BN = swap_bn(T);
  const int tiles = (N / SBM) * ((T + BN - 1) / BN);
  const int num_kb = K / SBK;
  const int total = tiles * num_kb;
  const int grid = std::max(1, std::min(max_ctas, total));
  const int ipc = (total + grid - 1) / grid;
  const int max_contrib = (num_kb + ipc - 1) / ipc + 1;
  return size_t(tiles) * max_contrib * SBM * BN * sizeof(float);
}

// Receive side of the fused tensor-parallel all-reduce.  Block = 16 tokens x
// one 128-feature tile column (thread: 8 features, 16-byte loads); it waits
// until every rank published the tile for this call's epoch, then writes
// out = sum over ranks (rank order, fp32) + resid.  With epoch_dev, the last
// block to finish advances *epoch_dev (every block read it before).
__global__ void __launch_bounds__(256) k_peer_reduce(const __nv_bfloat16* __restrict__ recv, size_t half_recv,
                                                     const int* flags, size_t half_flags, int world, int T, int N,
                                                     int m_tiles, int bn, int epoch, int* epoch_dev, int* done,
                                                     const __nv_bfloat16* __restrict__ resid, int ldr,
                                                     __nv_bfloat16* __restrict__ out, int ldo) {
  pdl_trigger();
  pdl_wait();
  const int ep = epoch_dev ? *reinterpret_cast<volatile int*>(epoch_dev) + 1 : epoch;
  recv += (ep & 1) * half_recv;
  flags += (ep & 1) * half_flags;
  const int mt = blockIdx.x, t0 = blockIdx.y * 16;
  const int tile = (t0 / bn) * m_tiles + mt;
  const int ntiles = m_tiles * ((T + bn - 1) / bn);
  if (threadIdx.x < world) {
    const int* f = flags + size_t(threadIdx.x) * ntiles + tile;
    while (ld_acquire_sys(f) < ep) __nanosleep(32);
  }
  __syncthreads();
  const int t = t0 + (threadIdx.x >> 4);
  if (t < T) {
    const int o = mt * SBM + (threadIdx.x & 15) * 8;
    float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    auto add = [&](uint4 v) {
      a[0] += bf16lo(v.x); a[1] += bf16hi(v.x); a[2] += bf16lo(v.y); a[3] += bf16hi(v.y);
      a[4] += bf16lo(v.z); a[5] += bf16hi(v.z); a[6] += bf16lo(v.w); a[7] += bf16hi(v.w);
    };
    uint4 v[HP_MAX_PEERS];
#pragma unroll
    for (int r = 0; r < HP_MAX_PEERS; ++r)
      if (r < world) v[r] = __ldcg(reinterpret_cast<const uint4*>(recv + (size_t(r) * T + t) * N + o));
#pragma unroll
    for (int r = 0; r < HP_MAX_PEERS; ++r)
      if (r < world) add(v[r]);
    if (resid) add(*reinterpret_cast<const uint4*>(resid + size_t(t) * ldr + o));
    *reinterpret_cast<uint4*>(out + size_t(t) * ldo + o) =
        make_uint4(pack_bf16(a[0], a[1]), pack_bf16(a[2], a[3]), pack_bf16(a[4], a[5]), pack_bf16(a[6], a[7]));
  }
  if (epoch_dev) {
    __syncthreads();
    if (threadIdx.x == 0) {
      const int nblk = int(gridDim.x * gridDim.y);
      if (atomicAdd(done, 1) == nblk - 1) {
        *done = 0;
        __threadfence();
        atomicAdd(epoch_dev, 1);
      }
    }
  }
}

// Two-shot receive side, step 1 (reduce-scatter): this rank owns the
// feature tiles mt with mt % world == rank; per owned tile and 16-token row
// block, wait for every rank's partial, sum (+ resid) and broadcast the bf16
// result into every rank's gather buffer, then raise gather flag
// [row block][mt] = epoch on every rank.
struct PeerPtrs {  // per-rank device pointers, passed by value in the kernel parameters
  __nv_bfloat16* buf[HP_MAX_PEERS];
  int* flag[HP_MAX_PEERS];
};

__global__ void __launch_bounds__(256) k_peer_rs(const __nv_bfloat16* __restrict__ recv, size_t half_recv,
                                                 const int* flags, size_t half_flags, const PeerPtrs g,
                                                 size_t half_gather, size_t half_gflags, int world, int rank,
                                                 int T, int N, int m_tiles, int bn, int epoch, const int* epoch_dev,
                                                 const __nv_bfloat16* __restrict__ resid, int ldr) {
  pdl_trigger();
  pdl_wait();
  const int ep = epoch_dev ? *reinterpret_cast<const volatile int*>(epoch_dev) + 1 : epoch;
  recv += (ep & 1) * half_recv;
  flags += (ep & 1) * half_flags;
  const int mt = rank + int(blockIdx.x) * world, t0 = blockIdx.y * 16;
  const int tile = (t0 / bn) * m_tiles + mt;
  const int ntiles = m_tiles * ((T + bn - 1) / bn);
  if (threadIdx.x < world) {
    const int* f = flags + size_t(threadIdx.x) * ntiles + tile;
    while (ld_acquire_sys(f) < ep) __nanosleep(32);
  }
  __syncthreads();
  const int t = t0 + (threadIdx.x >> 4);
  if (t < T) {
    const int o = mt * SBM + (threadIdx.x & 15) * 8;
    float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    auto add = [&](uint4 v) {
      a[0] += bf16lo(v.x); a[1] += bf16hi(v.x); a[2] += bf16lo(v.y); a[3] += bf16hi(v.y);
      a[4] += bf16lo(v.z); a[5] += bf16hi(v.z); a[6] += bf16lo(v.w); a[7] += bf16hi(v.w);
    };
    uint4 v[HP_MAX_PEERS];
#pragma unroll
    for (int r = 0; r < HP_MAX_PEERS; ++r)
      if (r < world) v[r] = __ldcg(reinterpret_cast<const uint4*>(recv + (size_t(r) * T + t) * N + o));
#pragma unroll
    for (int r = 0; r < HP_MAX_PEERS; ++r)
      if (r < world) add(v[r]);
    if (resid) add(*reinterpret_cast<const uint4*>(resid + size_t(t) * ldr + o));
    const uint4 w =
        make_uint4(pack_bf16(a[0], a[1]), pack_bf16(a[2], a[3]), pack_bf16(a[4], a[5]), pack_bf16(a[6], a[7]));
    const size_t off = (ep & 1) * half_gather + size_t(t) * N + o;
    for (int q = 0; q < world; ++q) *reinterpret_cast<uint4*>(g.buf[q] + off) = w;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    const size_t f = (ep & 1) * half_gflags + size_t(blockIdx.y) * m_tiles + mt;
    for (int q = 0; q < world; ++q) st_relaxed_sys(g.flag[q] + f, ep);  // fenced above
  }
}

// Two-shot step 2 (all-gather, local): wait for the owner's flag of every
// (row block, feature tile) and copy the reduced tile to `out`.  With
// epoch_dev, the last block advances *epoch_dev.
__global__ void __launch_bounds__(256) k_peer_ag(const __nv_bfloat16* __restrict__ gather, size_t half_gather,
                                                 const int* gflags, size_t half_gflags, int T, int N, int m_tiles,
                                                 int epoch, int* epoch_dev, int* done,
                                                 __nv_bfloat16* __restrict__ out, int ldo) {
  pdl_trigger();
  pdl_wait();
  const int ep = epoch_dev ? *reinterpret_cast<volatile int*>(epoch_dev) + 1 : epoch;
  const int mt = blockIdx.x, t0 = blockIdx.y * 16;
  if (threadIdx.x == 0) {
    const int* f = gflags + (ep & 1) * half_gflags + size_t(blockIdx.y) * m_tiles + mt;
    while (ld_acquire_sys(f) < ep) __nanosleep(32);
  }
  __syncthreads();
  const int t = t0 + (threadIdx.x >> 4);
  if (t < T) {
    const int o = mt * SBM + (threadIdx.x & 15) * 8;
    *reinterpret_cast<uint4*>(out + size_t(t) * ldo + o) =
        __ldcg(reinterpret_cast<const uint4*>(gather + (ep & 1) * half_gather + size_t(t) * N + o));
  }
  if (epoch_dev) {
    __syncthreads();
    if (threadIdx.x == 0) {
      const int nblk = int(gridDim.x * gridDim.y);
      if (atomicAdd(done, 1) == nblk - 1) {
        *done = 0;
        __threadfence();
        atomicAdd(epoch_dev, 1);
      }
    }
  }
}

struct PeerArgs {
  void* const* recv;
  size_t half_recv;
  int* const* flags;
  size_t half_flags;
  int world, rank, epoch;
  const int* epoch_dev;
  int two_shot;
};

struct RopeArgs {
  const int* pos;
  const float* cos_sin;
  const int* slots;
  void* kc;
  void* vc;
  int page, Hq, Hkv, hd;
};

static int gemm_swap_impl(const void* X, int ldx, const void* W, int ldw, void* Y, int ldy, const void* R, int ldr,
                          int T, int N, int K, int epilogue, void* workspace, size_t ws_bytes, int* counters,
                          int n_counters, int max_ctas, void* stream, const PeerArgs* peer,
                          const RopeArgs* rope = nullptr);

extern "C" int hp_gemm_swap_qkv_rope(const void* X, int ldx, const void* W, int ldw, void* Y, int ldy, int T,
                                     int Hq, int Hkv, int d, int K, const int* positions, const float* cos_sin,
                                     const int* slot_mapping, void* kcache, void* vcache, int page, void* workspace,
                                     size_t ws_bytes, int* counters, int n_counters, int max_ctas, void* stream) {
  HP_CHECK_ARG(Y && positions && cos_sin && slot_mapping && kcache && vcache, "hp_gemm_swap_qkv_rope: null pointer");
  HP_CHECK_ARG(d == 64 || d == 128, "hp_gemm_swap_qkv_rope: head_dim must be 64 or 128");
  HP_CHECK_ARG(Hq >= 1 && Hkv >= 1 && Hq % Hkv == 0, "hp_gemm_swap_qkv_rope: bad head counts");
  HP_CHECK_ARG(page >= 64 && page % 64 == 0, "hp_gemm_swap_qkv_rope: page must be a multiple of 64");
  const int N = (Hq + 2 * Hkv) * d;
  HP_CHECK_ARG(N % 128 == 0 && ldy >= N, "hp_gemm_swap_qkv_rope: (Hq+2Hkv)*d must be a multiple of 128");
  const RopeArgs ra{positions, cos_sin, slot_mapping, kcache, vcache, page, Hq, Hkv, d};
  return gemm_swap_impl(X, ldx, W, ldw, Y, ldy, nullptr, 0, T, N, K, SW_EPI_ROPE, workspace, ws_bytes, counters,
                        n_counters, max_ctas, stream, nullptr, &ra);
}

extern "C" int hp_gemm_swap(const void* X, int ldx, const void* W, int ldw, void* Y, int ldy,
                            const void* R, int ldr, int T, int N, int K, int epilogue,
                            void* workspace, size_t ws_bytes, int* counters, int n_counters,
                            int max_ctas, void* stream) {
  HP_CHECK_ARG(Y, "hp_gemm_swap: null pointer");
  HP_CHECK_ARG(epilogue >= HP_EPI_STORE && epilogue <= HP_EPI_SILU, "hp_gemm_swap: bad epilogue");
  return gemm_swap_impl(X, ldx, W, ldw, Y, ldy, R, ldr, T, N, K, epilogue, workspace, ws_bytes, counters,
                        n_counters, max_ctas, stream, nullptr);
}

extern "C" int hp_gemm_swap_peer(const void* X, int ldx, const void* W, int ldw, int T, int N, int K,
                                 void* const* peer_recv, size_t recv_half_elems, int* const* peer_flags,
                                 size_t flags_half_elems, int world, int rank, int epoch, const int* epoch_dev,
                                 int two_shot, void* workspace, size_t ws_bytes, int* counters, int n_counters,
                                 int max_ctas, void* stream) {
  HP_CHECK_ARG(peer_recv && peer_flags && world >= 1 && world <= HP_MAX_PEERS && rank >= 0 && rank < world,
               "hp_gemm_swap_peer: bad peer arguments");
  HP_CHECK_ARG(epoch_dev || epoch >= 1, "hp_gemm_swap_peer: host epochs start at 1 and increase per call");
  for (int q = 0; q < world; ++q)
    HP_CHECK_ARG(peer_recv[q] && peer_flags[q], "hp_gemm_swap_peer: null peer buffer");
  const PeerArgs pa{peer_recv, recv_half_elems, peer_flags, flags_half_elems, world, rank, epoch, epoch_dev,
                    two_shot ? 1 : 0};
  return gemm_swap_impl(X, ldx, W, ldw, nullptr, 0, nullptr, 0, T, N, K, HP_EPI_PEER, workspace, ws_bytes,
                        counters, n_counters, max_ctas, stream, &pa);
}

extern "C" int hp_peer_reduce(const void* recv, size_t recv_half_elems, const int* flags, size_t flags_half_elems,
                              int world, int T, int N, int epoch, int* epoch_dev, int* done, const void* resid,
                              int ldr, void* out, int ldo, void* stream) {
  HP_CHECK_ARG(recv && flags && out && world >= 1 && world <= HP_MAX_PEERS, "hp_peer_reduce: bad arguments");
  HP_CHECK_ARG(T >= 1 && T <= 256 && N % SBM == 0, "hp_peer_reduce: T in [1, 256], N a multiple of 128");
  HP_CHECK_ARG(ldo % 8 == 0 && (resid == nullptr || ldr % 8 == 0), "hp_peer_reduce: pitch not 16-byte aligned");
  HP_CHECK_ARG(epoch_dev ? done != nullptr : epoch >= 1, "hp_peer_reduce: device epochs need a zeroed `done` word");
  const int m_tiles = N / SBM;
  HP_LAUNCH_PDL("k_peer_reduce", k_peer_reduce, dim3(m_tiles, (T + 15) / 16), dim3(256), 0,
                static_cast<cudaStream_t>(stream), static_cast<const __nv_bfloat16*>(recv), recv_half_elems, flags,
                flags_half_elems, world, T, N, m_tiles, swap_bn(T), epoch, epoch_dev, done,
                static_cast<const __nv_bfloat16*>(resid), ldr, static_cast<__nv_bfloat16*>(out), ldo);
  HP_LAUNCH_CHECK("k_peer_reduce");
  return HP_OK;
}

extern "C" int hp_peer_rs(const void* recv, size_t recv_half_elems, const int* flags, size_t flags_half_elems,
                          void* const* peer_gather, size_t gather_half_elems, int* const* peer_gflags,
                          size_t gflags_half_elems, int world, int rank, int T, int N, int epoch,
                          const int* epoch_dev, const void* resid, int ldr, void* stream) {
  HP_CHECK_ARG(recv && flags && peer_gather && peer_gflags && world >= 1 && world <= HP_MAX_PEERS && rank >= 0 &&
                   rank < world, "hp_peer_rs: bad arguments");
  HP_CHECK_ARG(T >= 1 && T <= 256 && N % SBM == 0, "hp_peer_rs: T in [1, 256], N a multiple of 128");
  HP_CHECK_ARG(resid == nullptr || ldr % 8 == 0, "hp_peer_rs: residual pitch not 16-byte aligned");
  HP_CHECK_ARG(epoch_dev || epoch >= 1, "hp_peer_rs: host epochs start at 1");
  const int m_tiles = N / SBM;
  const int owned = (m_tiles - rank + world - 1) / world;  // feature tiles rank, rank + world, ...
  if (owned == 0) return HP_OK;
  PeerPtrs g{};
  for (int q = 0; q < world; ++q) {
    HP_CHECK_ARG(peer_gather[q] && peer_gflags[q], "hp_peer_rs: null peer buffer");
    g.buf[q] = static_cast<__nv_bfloat16*>(peer_gather[q]);
    g.flag[q] = peer_gflags[q];
  }
  HP_LAUNCH_PDL("k_peer_rs", k_peer_rs, dim3(owned, (T + 15) / 16), dim3(256), 0, static_cast<cudaStream_t>(stream),
                static_cast<const __nv_bfloat16*>(recv), recv_half_elems, flags, flags_half_elems, g,
                gather_half_elems, gflags_half_elems, world, rank, T, N, m_tiles, swap_bn(T), epoch, epoch_dev,
                static_cast<const __nv_bfloat16*>(resid), ldr);
  HP_LAUNCH_CHECK("k_peer_rs");
  return HP_OK;
}

extern "C" int hp_peer_ag(const void* gather, size_t gather_half_elems, const int* gflags, size_t gflags_half_elems,
                          int T, int N, int epoch, int* epoch_dev, int* done, void* out, int ldo, void* stream) {
  HP_CHECK_ARG(gather && gflags && out, "hp_peer_ag: null pointer");
  HP_CHECK_ARG(T >= 1 && T <= 256 && N % SBM == 0 && ldo % 8 == 0, "hp_peer_ag: bad shape");
  HP_CHECK_ARG(epoch_dev ? done != nullptr : epoch >= 1, "hp_peer_ag: device epochs need a zeroed `done` word");
  const int m_tiles = N / SBM;
  HP_LAUNCH_PDL("k_peer_ag", k_peer_ag, dim3(m_tiles, (T + 15) / 16), dim3(256), 0, static_cast<cudaStream_t>(stream),
                static_cast<const __nv_bfloat16*>(gather), gather_half_elems, gflags, gflags_half_elems, T, N,
                m_tiles, epoch, epoch_dev, done, static_cast<__nv_bfloat16*>(out), ldo);
  HP_LAUNCH_CHECK("k_peer_ag");
  return HP_OK;
}

extern "C" int hp_peer_tiles(int T, int N) {
  if (T < 1 || T > 256 || N % SBM) return HP_ERR_INVALID;
  const int BN = swap_bn(T);
  return (N / SBM) * ((T + BN - 1) / BN);
}

static int gemm_swap_impl(const void* X, int ldx, const void* W, int ldw, void* Y, int ldy, const void* R, int ldr,
                          int T, int N, int K, int epilogue, void* workspace, size_t ws_bytes, int* counters,
                          int n_counters, int max_ctas, void* stream, const PeerArgs* peer, const RopeArgs* rope) {
  HP_CHECK_ARG(X && W, "hp_gemm_swap: null pointer");
  HP_CHECK_ARG(T >= 1 && T <= 256, "hp_gemm_swap: token count must be in [1, 256]");
  HP_CHECK_ARG(N % 128 == 0, "hp_gemm_swap: N must be a multiple of 128 (tiled weight layout)");
  HP_CHECK_ARG(ldw == K, "hp_gemm_swap: W must be in the tiled layout (ldw == K)");
  HP_CHECK_ARG(K % SBK == 0, "hp_gemm_swap: K must be a multiple of 128");
  HP_CHECK_ARG(epilogue != HP_EPI_RESID || R != nullptr, "hp_gemm_swap: residual epilogue needs R");
  HP_CHECK_ARG(max_ctas >= 1, "hp_gemm_swap: max_ctas must be >= 1");
  HP_CHECK_ARG(ldy % 2 == 0 && (R == nullptr || ldr % 2 == 0), "hp_gemm_swap: odd output pitch");
  const int BN = swap_bn(T);
  SwapParams p{};
  p.N = N;
  p.T = T;
  p.K = K;
  p.m_tiles = N / SBM;
  p.n_tiles = (T + BN - 1) / BN;
  p.num_kb = K / SBK;
  // CTA pairs (M = 256 MMAs) on small partitions (2..16 SMs), where one SM's
  // MMA issue rate at N = 32 is the limit (8 SMs: 105 -> 113 GB/s per SM,
  // tools/swap_sms.py); on the full GPU the 1-CTA walk is faster (2.89 vs
  // 2.57 TB/s: half as many independent streams).  HP_SWAP_PAIR=0/1 forces.
  static const int pair_env = [] {
    const char* e = std::getenv("HP_SWAP_PAIR");
    return e ? std::atoi(e) : -1;
  }();
  const bool pair_ok = N % 256 == 0 && max_ctas >= 2;
  const bool pair = pair_ok && (pair_env >= 0 ? pair_env == 1 : max_ctas <= 16);
  p.m_walk = pair ? p.m_tiles / 2 : p.m_tiles;
  p.total_iters = p.m_walk * p.n_tiles * p.num_kb;
  const int units = pair ? max_ctas / 2 : max_ctas;
  const int grid = swap_grid(p.total_iters, p.num_kb, units);
  p.ipc = (p.total_iters + grid - 1) / grid;
  p.max_contrib = (p.num_kb + p.ipc - 1) / p.ipc + 1;
  p.out = static_cast<__nv_bfloat16*>(Y);
  p.ldo = ldy;
  p.resid = static_cast<const __nv_bfloat16*>(R);
  p.ldr = ldr;
  p.w = static_cast<const uint8_t*>(W);
  p.ws = static_cast<float*>(workspace);
  p.counters = counters;
  p.epi = epilogue;
  p.trace = static_cast<unsigned long long*>(trace_buf(TRACE_SWAP));
  if (rope) {
    p.pos = rope->pos;
    p.cos_sin = rope->cos_sin;
    p.slots = rope->slots;
    p.kc = static_cast<__nv_bfloat16*>(rope->kc);
    p.vc = static_cast<__nv_bfloat16*>(rope->vc);
    p.page = rope->page;
    p.Hq = rope->Hq;
    p.Hkv = rope->Hkv;
    p.hd = rope->hd;
  }
  if (peer) {
    for (int q = 0; q < peer->world; ++q) {
      p.peer_out[q] = static_cast<__nv_bfloat16*>(peer->recv[q]);
      p.peer_flags[q] = peer->flags[q];
    }
    p.half_out = peer->half_recv;
    p.half_flags = peer->half_flags;
    p.epoch_dev = peer->epoch_dev;
    p.world = peer->world;
    p.rank = peer->rank;
    p.epoch = peer->epoch;
    p.two_shot = peer->two_shot;
  }
  const bool any_split = p.ipc % p.num_kb != 0 || p.ipc < p.num_kb;
  if (any_split) {
    HP_CHECK_ARG(workspace && counters, "hp_gemm_swap: split tiles need workspace and counters");
    HP_CHECK_ARG(ws_bytes >= hp_gemm_swap_ws_bytes(T, N, K, max_ctas), "hp_gemm_swap: workspace too small");
    HP_CHECK_ARG(n_counters >= p.m_tiles * p.n_tiles, "hp_gemm_swap: too few counters");
  }
  CUtensorMap tx;
  // two 64-k boxes per stage; a pair CTA loads its BN/2 tokens
  int rc = cached_tmap_bf16(&tx, X, T, K, ldx, pair ? BN / 2 : BN, 64, true);
  if (rc) return rc;
  const int g = (p.total_iters + p.ipc - 1) / p.ipc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (pair) {
    switch (BN) {
      case 32: return launch_swap_pair<32>(tx, p, 2 * g, st);
      case 64: return launch_swap_pair<64>(tx, p, 2 * g, st);
      case 128: return launch_swap_pair<128>(tx, p, 2 * g, st);
      default: return launch_swap_pair<256>(tx, p, 2 * g, st);
    }
  }
  switch (BN) {
    case 32: return launch_swap<32>(tx, p, g, st);
    case 64: return launch_swap<64>(tx, p, g, st);
    case 128: return launch_swap<128>(tx, p, g, st);
    default: return launch_swap<256>(tx, p, g, st);
  }
}
