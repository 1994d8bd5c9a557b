// Causal GQA prefill attention on the 5th-gen tensor cores (reference kernel
// group "attn", phase prefill; workload.py:176-183).  Two operand sources:
//   dense   (prior_lens = 0): K/V are the new span's columns of the fused qkv
//           buffer, fetched as 128B-swizzled TMA boxes;
//   paged   (prior_lens >= 0, chunked prefill / hybrid batches, workload.py:
//           177-183, 213-257): K/V are read from the paged cache, which holds
//           the cached prefix plus the new span (hp_rope_kv_write ran first).
//           A cache page stores each 64-token tile as [d/64][64][64] with the
//           same 128B swizzle, so every (tile, 64-dim half) is ONE 8 KB bulk
//           copy landing exactly where the TMA box would have put it.
//           Query i of a sequence sits at position prior + i and attends keys
//           [0, prior + i].
//
// One CTA owns one (sequence, 128-query tile, q head) unit at a time
// (persistent grid = partition SMs, units longest-first).  Warp roles:
//   warp 0      TMA producer: Q once per unit, then K_j / V_j (128-token
//               tiles, 128B-swizzled boxes) into 2-stage rings
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer:
//                 S_j  = Q . K_j^T        (M=128, N=128, K=D; K-major A/B)
//                 O   += P_j . V_j        (M=128, N=D,   K=128; V MN-major)
//               S is double-buffered in TMEM so S_{j+1} is computed while
//               the softmax warps work on S_j; O accumulates in TMEM.
//   warps 2-5   softmax: one thread per query row (TMEM lane); tcgen05.ld of
//               the S row, causal mask, exp2 online softmax with lazy O
//               rescaling (only when a row max grows by > 2^8), P written as
//               bf16 into a 128B-swizzled K-major smem tile for the PV MMA;
//               epilogue O / l from TMEM to global.
// TMEM: S0 cols [0,128), S1 [128,256), O [256, 256+D).
#include "common.cuh"
#include "runtime.h"
#include "../../include/hp.h"

#include <algorithm>
#include <cmath>

namespace hp {

namespace {

constexpr int FQ = 128;    // query rows per unit (UMMA M)
constexpr int FK = 128;    // kv rows per tile
constexpr int KST = 2;     // K ring stages
constexpr int VST = 2;     // V ring stages
constexpr uint32_t BOX = 128 * 128;  // 128 rows x 128 B
constexpr float RESCALE_THRESHOLD = 8.0f;  // log2 units: rescale O when max grows by > 256x

template <int D>
struct FaCfg {
  static constexpr int NB = D / 64;             // 64-dim boxes per row
  static constexpr uint32_t QB = NB * BOX;      // Q tile bytes
  static constexpr uint32_t KB = NB * BOX;      // K (and V) tile bytes
  static constexpr uint32_t PB = 2 * BOX;       // P tile bytes (128 x 128 bf16)
  static constexpr size_t SMEM = 1024 + QB + KST * KB + VST * KB + PB + 512;
};

struct FaParams {
  const int* cu_seqlens;
  int nseq, n_qt, Hq, G;
  __nv_bfloat16* out;
  int ldo;
  float scale_log2;
  // paged operand source (PAGED kernels only)
  const __nv_bfloat16* kc;
  const __nv_bfloat16* vc;
  const int* block_table;
  const int* prior_lens;
  int max_pages, page, Hkv;
};

__device__ __forceinline__ uint64_t desc_mn_sw128(uint32_t addr, uint32_t lbo_bytes) {
  uint64_t d = 0;
  d |= uint64_t((addr & 0x3FFFF) >> 4);
  d |= uint64_t((lbo_bytes >> 4) & 0x3FFF) << 16;  // LBO: stride between 64-element MN blocks
  d |= uint64_t(1024 >> 4) << 32;                   // SBO: stride between 8-row K groups
  d |= uint64_t(1) << 46;
  d |= uint64_t(2) << 61;
  return d;
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float* v) {
  const uint32_t* r = reinterpret_cast<const uint32_t*>(v);
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]),
      "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]),
      "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}

__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

struct Unit {
  int head, seq, qt, s0, len, nkv;
  int prior, kvlen;  // cached prefix length; keys visible to the last query
};

template <bool PAGED>
__device__ __forceinline__ bool unit_of(const FaParams& p, int u, Unit& x) {
  x.head = u % p.Hq;
  const int rest = u / p.Hq;
  x.seq = rest % p.nseq;
  x.qt = p.n_qt - 1 - rest / p.nseq;
  x.s0 = p.cu_seqlens[x.seq];
  x.len = p.cu_seqlens[x.seq + 1] - x.s0;
  if (x.qt * FQ >= x.len) return false;
  x.prior = PAGED ? p.prior_lens[x.seq] : 0;
  x.kvlen = x.prior + x.len;
  const int q0 = x.qt * FQ;
  x.nkv = min((x.prior + q0 + FQ + FK - 1) / FK, (x.kvlen + FK - 1) / FK);
  return true;
}

// Address of the 64-token tile holding cache position `pos` of sequence
// `seq`, kv head `kvh` (positions past the sequence map to its first page:
// finite data whose scores the causal mask removes).
template <int D>
__device__ __forceinline__ const __nv_bfloat16* page_tile(const FaParams& p, const __nv_bfloat16* base,
                                                          int seq, int kvh, int pos, int kvlen) {
  if (pos >= kvlen) pos = 0;
  const int blk = __ldg(p.block_table + size_t(seq) * p.max_pages + pos / p.page);
  const int sub = (pos % p.page) >> 6;
  return base + (size_t(blk) * p.Hkv + kvh) * size_t(p.page) * D + size_t(sub) * 64 * D;
}

}  // namespace

template <int D, bool PAGED>
__global__ void __launch_bounds__(192, 1)
    k_fa_tc(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
            const __grid_constant__ CUtensorMap tmV, const FaParams p) {
  using C = FaCfg<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + C::QB;
  uint8_t* sV = sK + KST * C::KB;
  uint8_t* sP = sV + VST * C::KB;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + C::PB);
  uint64_t* q_full = bars + 0;
  uint64_t* q_empty = bars + 1;
  uint64_t* k_full = bars + 2;             // [KST]
  uint64_t* k_empty = k_full + KST;        // [KST]
  uint64_t* v_full = k_empty + KST;        // [VST]
  uint64_t* v_empty = v_full + VST;        // [VST]
  uint64_t* s_full = v_empty + VST;        // [2]
  uint64_t* s_free = s_full + 2;           // [2]
  uint64_t* p_full = s_free + 2;
  uint64_t* p_free = p_full + 1;
  uint64_t* o_full = p_free + 1;
  uint64_t* o_empty = o_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_empty + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int s = 0; s < KST; ++s) { mbar_init(&k_full[s], 1); mbar_init(&k_empty[s], 1); }
    for (int s = 0; s < VST; ++s) { mbar_init(&v_full[s], 1); mbar_init(&v_empty[s], 1); }
    for (int s = 0; s < 2; ++s) { mbar_init(&s_full[s], 1); mbar_init(&s_free[s], 4); }
    mbar_init(p_full, 4);
    mbar_init(p_free, 1);
    mbar_init(o_full, 1);
    mbar_init(o_empty, 4);
    fence_barrier_init();
  }
  if (warp == 1) {
    tmem_alloc(tmem_slot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int total = p.nseq * p.n_qt * p.Hq;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      uint32_t un = 0, kt = 0, vt = 0;
      for (int u = blockIdx.x; u < total; u += gridDim.x) {
        Unit x;
        if (!unit_of<PAGED>(p, u, x)) continue;
        const int kvh = x.head / p.G;
        mbar_wait(q_empty, (un & 1) ^ 1);
        mbar_arrive_expect_tx(q_full, C::QB);
        for (int b = 0; b < C::NB; ++b)
          tma_load_2d(sQ + b * BOX, &tmQ, q_full, x.head * D + b * 64, x.s0 + x.qt * FQ);
        for (int j = 0; j < x.nkv; ++j, ++kt, ++vt) {
          const int ks = kt % KST, vs = vt % VST;
          mbar_wait(&k_empty[ks], ((kt / KST) & 1) ^ 1);
          mbar_arrive_expect_tx(&k_full[ks], C::KB);
          if constexpr (PAGED) {
            // 128 keys = two 64-token cache tiles; each 64-dim half is one
            // contiguous, already-swizzled 8 KB run -> rows t*64.. of box b
#pragma unroll
            for (int t = 0; t < 2; ++t) {
              const __nv_bfloat16* src = page_tile<D>(p, p.kc, x.seq, kvh, j * FK + t * 64, x.kvlen);
#pragma unroll
              for (int b = 0; b < C::NB; ++b)
                bulk_load(sK + ks * C::KB + b * BOX + t * (BOX / 2), src + b * 64 * 64, BOX / 2, &k_full[ks]);
            }
          } else {
            for (int b = 0; b < C::NB; ++b)
              tma_load_2d(sK + ks * C::KB + b * BOX, &tmK, &k_full[ks], kvh * D + b * 64, x.s0 + j * FK);
          }
          mbar_wait(&v_empty[vs], ((vt / VST) & 1) ^ 1);
          mbar_arrive_expect_tx(&v_full[vs], C::KB);
          if constexpr (PAGED) {
#pragma unroll
            for (int t = 0; t < 2; ++t) {
              const __nv_bfloat16* src = page_tile<D>(p, p.vc, x.seq, kvh, j * FK + t * 64, x.kvlen);
#pragma unroll
              for (int b = 0; b < C::NB; ++b)
                bulk_load(sV + vs * C::KB + b * BOX + t * (BOX / 2), src + b * 64 * 64, BOX / 2, &v_full[vs]);
            }
          } else {
            for (int b = 0; b < C::NB; ++b)
              tma_load_2d(sV + vs * C::KB + b * BOX, &tmV, &v_full[vs], kvh * D + b * 64, x.s0 + j * FK);
          }
        }
        ++un;
      }
    }
  } else if (warp == 1) {
    // --------------------------------------------------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc_qk = umma_idesc_bf16(FQ, FK);
      constexpr uint32_t idesc_pv = umma_idesc_bf16(FQ, D) | (1u << 16);  // B (V) MN-major
      uint32_t un = 0, kt = 0, vt = 0, gt = 0;  // gt: global kv-tile counter (S buffer / P phases)
      auto issue_pv = [&](uint32_t tile, bool first) {
        const int vs = vt % VST;
        if (first) mbar_wait(o_empty, (un & 1) ^ 1);  // previous unit's epilogue has read O
        mbar_wait(p_full, tile & 1);
        mbar_wait(&v_full[vs], (vt / VST) & 1);
        tc_fence_after();
        const uint32_t pa = smem_u32(sP), vb = smem_u32(sV + vs * C::KB);
#pragma unroll
        for (int kk = 0; kk < FK / 16; ++kk)
          umma_bf16(tmem + 256, umma_desc_sw128(pa + (kk >> 2) * BOX + (kk & 3) * 32),
                    desc_mn_sw128(vb + kk * 2048, BOX), idesc_pv, (first && kk == 0) ? 0u : 1u);
        umma_commit(&v_empty[vs]);
        umma_commit(p_free);
        ++vt;
      };
      for (int u = blockIdx.x; u < total; u += gridDim.x) {
        Unit x;
        if (!unit_of<PAGED>(p, u, x)) continue;
        mbar_wait(q_full, un & 1);
        for (int j = 0; j < x.nkv; ++j, ++kt, ++gt) {
          const int sb = gt & 1;
          const int ks = kt % KST;
          mbar_wait(&s_free[sb], ((gt >> 1) & 1) ^ 1);
          mbar_wait(&k_full[ks], (kt / KST) & 1);
          tc_fence_after();
          const uint32_t qa = smem_u32(sQ), kb = smem_u32(sK + ks * C::KB);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk)
            umma_bf16(tmem + sb * 128, umma_desc_sw128(qa + (kk >> 2) * BOX + (kk & 3) * 32),
                      umma_desc_sw128(kb + (kk >> 2) * BOX + (kk & 3) * 32), idesc_qk, kk > 0 ? 1u : 0u);
          umma_commit(&k_empty[ks]);
          umma_commit(&s_full[sb]);
          if (j == x.nkv - 1) umma_commit(q_empty);
          if (j >= 1) issue_pv(gt - 1, j == 1);
        }
        issue_pv(gt - 1, x.nkv == 1);
        umma_commit(o_full);
        ++un;
      }
    }
  } else {
    // ------------------------------------------------------------- softmax
    const int q4 = warp & 3;
    const int row = q4 * 32 + lane;
    const uint32_t lane_base = uint32_t(q4 * 32) << 16;
    uint32_t un = 0, gt = 0;
    for (int u = blockIdx.x; u < total; u += gridDim.x) {
      Unit x;
      if (!unit_of<PAGED>(p, u, x)) continue;
      const int q0 = x.qt * FQ;
      const int qi = q0 + row;      // row of this thread within the new span
      const int qpos = x.prior + qi;  // its key-space position
      float m_run = -INFINITY, l = 0.f;
      for (int j = 0; j < x.nkv; ++j, ++gt) {
        const int sb = gt & 1;
        mbar_wait(&s_full[sb], (gt >> 1) & 1);
        tc_fence_after();
        float s[128];
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_ld32(tmem + lane_base + sb * 128 + c * 32, s + c * 32);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_free[sb]);
        const int kbase = j * FK;
        const bool need_mask = (kbase + FK - 1 > x.prior + q0) || (kbase + FK > x.kvlen);
        float mx = -INFINITY;
#pragma unroll
        for (int c = 0; c < 128; ++c) {
          float v = s[c] * p.scale_log2;
          if (need_mask && (kbase + c > qpos || kbase + c >= x.kvlen)) v = -INFINITY;
          s[c] = v;
          mx = fmaxf(mx, v);
        }
        const float m_new = fmaxf(m_run, mx);
        const bool grow = m_new > m_run + RESCALE_THRESHOLD;
        // P buffer / O are free once the previous PV completed
        mbar_wait(p_free, (gt & 1) ^ 1);
        tc_fence_after();
        if (__any_sync(0xffffffffu, grow) && j > 0) {
          const float alpha = grow ? exp2f(m_run - m_new) : 1.f;
#pragma unroll 1
          for (int c = 0; c < D / 32; ++c) {
            float o[32];
            tmem_ld32(tmem + lane_base + 256 + c * 32, o);
            tmem_ld_wait();
#pragma unroll
            for (int k = 0; k < 32; ++k) o[k] *= alpha;
            tmem_st32(tmem + lane_base + 256 + c * 32, o);
          }
          tmem_st_wait();
          if (grow) l *= alpha;
        }
        if (grow) m_run = m_new;
        const float mb = (m_run == -INFINITY) ? 0.f : m_run;
        // P row -> smem, 128B-swizzled K-major (two 64-token halves)
        uint8_t* prow = sP + row * 128;
#pragma unroll
        for (int ch = 0; ch < 16; ++ch) {
          uint32_t w[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const float a = ex2(s[ch * 8 + 2 * k] - mb), b = ex2(s[ch * 8 + 2 * k + 1] - mb);
            l += a + b;
            w[k] = pack_bf16(a, b);
          }
          const int half = ch >> 3, cc = ch & 7;
          *reinterpret_cast<uint4*>(prow + half * BOX + ((cc ^ (row & 7)) << 4)) = make_uint4(w[0], w[1], w[2], w[3]);
        }
        fence_proxy_async();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(p_full);
      }
      // epilogue: O / l -> global
      mbar_wait(o_full, un & 1);
      tc_fence_after();
      const float inv = l > 0.f ? 1.f / l : 0.f;
      const bool ok = qi < x.len;
      __nv_bfloat16* orow = p.out + size_t(x.s0 + qi) * p.ldo + size_t(x.head) * D;
#pragma unroll 1
      for (int c = 0; c < D / 32; ++c) {
        float o[32];
        tmem_ld32(tmem + lane_base + 256 + c * 32, o);
        tmem_ld_wait();
        if (ok) {
          uint4 w[4];
          uint32_t* ww = reinterpret_cast<uint32_t*>(w);
#pragma unroll
          for (int k = 0; k < 16; ++k) ww[k] = pack_bf16(o[2 * k] * inv, o[2 * k + 1] * inv);
          uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
          for (int k = 0; k < 4; ++k) dst[k] = w[k];
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(o_empty);
      ++un;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int D, bool PAGED>
static int launch_fa(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                     const FaParams& p, int grid, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    HP_CUDA_TRY(cudaFuncSetAttribute(k_fa_tc<D, PAGED>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(FaCfg<D>::SMEM)));
    attr = true;
  }
  k_fa_tc<D, PAGED><<<grid, 192, FaCfg<D>::SMEM, st>>>(tq, tk, tv, p);
  HP_LAUNCH_CHECK("k_fa_tc");
  return HP_OK;
}

}  // namespace hp

using namespace hp;

extern "C" int hp_prefill_attn(const void* q, int ldq, const void* k, int ldk, const void* v, int ldv,
                               void* o, int ldo, const int* cu_seqlens, int nseq, int total_tokens,
                               int max_seqlen, int Hq, int Hkv, int d, float scale, int max_ctas,
                               void* stream) {
  HP_CHECK_ARG(q && k && v && o && cu_seqlens, "hp_prefill_attn: null pointer");
  HP_CHECK_ARG(d == 64 || d == 128, "hp_prefill_attn: head_dim must be 64 or 128");
  HP_CHECK_ARG(Hkv >= 1 && Hq % Hkv == 0, "hp_prefill_attn: Hkv must divide Hq");
  HP_CHECK_ARG(nseq >= 1 && max_seqlen >= 1 && total_tokens >= 1, "hp_prefill_attn: empty batch");
  HP_CHECK_ARG(max_ctas >= 1, "hp_prefill_attn: max_ctas must be >= 1");
  HP_CHECK_ARG(ldo % 8 == 0, "hp_prefill_attn: output pitch must be a multiple of 8");
  const uint64_t rows = uint64_t(total_tokens);  // TMA zero-fills past the last row
  CUtensorMap tq, tk, tv;
  int rc = cached_tmap_bf16(&tq, q, rows, uint64_t(Hq) * d, ldq, 128, 64, true);
  if (rc) return rc;
  rc = cached_tmap_bf16(&tk, k, rows, uint64_t(Hkv) * d, ldk, 128, 64, true);
  if (rc) return rc;
  rc = cached_tmap_bf16(&tv, v, rows, uint64_t(Hkv) * d, ldv, 128, 64, true);
  if (rc) return rc;
  FaParams p{};
  p.cu_seqlens = cu_seqlens;
  p.nseq = nseq;
  p.n_qt = (max_seqlen + FQ - 1) / FQ;
  p.Hq = Hq;
  p.G = Hq / Hkv;
  p.out = static_cast<__nv_bfloat16*>(o);
  p.ldo = ldo;
  p.scale_log2 = scale * 1.4426950408889634f;
  const int units = nseq * p.n_qt * Hq;
  const int grid = std::min(units, max_ctas);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  return d == 128 ? launch_fa<128, false>(tq, tk, tv, p, grid, st) : launch_fa<64, false>(tq, tk, tv, p, grid, st);
}

extern "C" int hp_prefill_attn_paged(const void* q, int ldq, const void* kcache, const void* vcache,
                                     const int* block_table, int max_pages, const int* cu_seqlens,
                                     const int* prior_lens, int nseq, int total_tokens, int max_seqlen,
                                     void* o, int ldo, int Hq, int Hkv, int d, int page, int num_blocks,
                                     float scale, int max_ctas, void* stream) {
  HP_CHECK_ARG(q && kcache && vcache && block_table && cu_seqlens && prior_lens && o,
               "hp_prefill_attn_paged: null pointer");
  HP_CHECK_ARG(d == 64 || d == 128, "hp_prefill_attn_paged: head_dim must be 64 or 128");
  HP_CHECK_ARG(Hkv >= 1 && Hq % Hkv == 0, "hp_prefill_attn_paged: Hkv must divide Hq");
  HP_CHECK_ARG(page >= 64 && page % 64 == 0, "hp_prefill_attn_paged: page must be a multiple of 64");
  HP_CHECK_ARG(nseq >= 1 && max_seqlen >= 1 && total_tokens >= 1 && max_pages >= 1 && num_blocks >= 1,
               "hp_prefill_attn_paged: empty batch");
  HP_CHECK_ARG(max_ctas >= 1, "hp_prefill_attn_paged: max_ctas must be >= 1");
  HP_CHECK_ARG(ldo % 8 == 0, "hp_prefill_attn_paged: output pitch must be a multiple of 8");
  HP_CHECK_ARG((reinterpret_cast<uintptr_t>(kcache) & 15) == 0 && (reinterpret_cast<uintptr_t>(vcache) & 15) == 0,
               "hp_prefill_attn_paged: caches must be 16-byte aligned");
  CUtensorMap tq;
  int rc = cached_tmap_bf16(&tq, q, uint64_t(total_tokens), uint64_t(Hq) * d, ldq, 128, 64, true);
  if (rc) return rc;
  FaParams p{};
  p.cu_seqlens = cu_seqlens;
  p.nseq = nseq;
  p.n_qt = (max_seqlen + FQ - 1) / FQ;
  p.Hq = Hq;
  p.G = Hq / Hkv;
  p.out = static_cast<__nv_bfloat16*>(o);
  p.ldo = ldo;
  p.scale_log2 = scale * 1.4426950408889634f;
  p.kc = static_cast<const __nv_bfloat16*>(kcache);
  p.vc = static_cast<const __nv_bfloat16*>(vcache);
  p.block_table = block_table;
  p.prior_lens = prior_lens;
  p.max_pages = max_pages;
  p.page = page;
  p.Hkv = Hkv;
  const int units = nseq * p.n_qt * Hq;
  const int grid = std::min(units, max_ctas);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  return d == 128 ? launch_fa<128, true>(tq, tq, tq, p, grid, st) : launch_fa<64, true>(tq, tq, tq, p, grid, st);
}
