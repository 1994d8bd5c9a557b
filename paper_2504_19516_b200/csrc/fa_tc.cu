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
// One CTA owns one (sequence, 256-query pair of 128-row tiles A/B, q head)
// unit at a time (persistent grid = partition SMs; units longest-first in
// "snake" order across CTAs).  Both tiles share every K/V tile.  Warp roles:
//   warp 0      producer: Q_A/Q_B once per unit, then K_j / V_j (128-token
//               tiles) into 2-stage rings (TMA boxes or paged bulk copies)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer:
//                 S_X  = Q_X . K_j^T      (M=128, N=128, K=D; SS)
//                 O_X += P_X . V_j        (M=128, N=D, K=128; A = P from TMEM)
//               ping-ponging the tiles: PV_A(j) QK_A(j+1) PV_B(j) QK_B(j+1)
//   warps 2-5   softmax of tile A, warps 6-9 softmax of tile B: one thread
//               per query row (TMEM lane), causal mask, exp2 online softmax
//               (8-way ILP max/sum chains) with lazy O rescaling (only when a
//               row max grows by > 2^8), P stored as packed bf16 over the S
//               tile's own TMEM columns; epilogue O / l to global.
// TMEM: S_A [0,128) S_B [128,256) O_A [256,256+D) O_B [256+D,256+2D).
// Measured bound (clock64 trace, T = 16384): the tensor core runs PV+QK of
// one tile in ~1.7k cycles against 1k at the UMMA peak -- the SS QK MMA at
// N = 128 plus the K/V TMA writes saturate the 128 B/clk shared-memory port.
#include "common.cuh"
#include "runtime.h"
#include "../../include/hp.h"

#include <algorithm>
#include <cstdlib>
#include <cmath>

namespace hp {

namespace {

constexpr int FQ = 128;    // query rows per unit (UMMA M)
constexpr int FK = 128;    // kv rows per tile
constexpr int KST = 2;     // K ring stages
constexpr int VST = 2;     // V ring stages
constexpr uint32_t BOX = 128 * 128;  // 128 rows x 128 B
constexpr float RESCALE_THRESHOLD = 8.0f;  // log2 units: rescale O when max grows by > 256x


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
  long long* trace;  // optional clock64 trace of CTA 0 (hp_set_fa_trace; development aid)
  uint64_t* cta_times;  // optional [grid][3] = {smid, start_ns, end_ns} (SM-idle measurement)
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

__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

// 2^x for a pair on the FMA pipe (FA4-style MUFU offload): round x to the
// nearest integer n with the 1.5 * 2^23 magic add, 2^(x - n) by a degree-3
// minimax polynomial on [-0.5, 0.5] (relative error 7.7e-5, below bf16's
// 3.9e-3), then n added to the exponent field with one IMAD.  x is clamped
// to -126 (masked scores: -inf -> 2^-126 ~ 1e-38 instead of 0).
__device__ __forceinline__ float2 ex2_poly2(float2 x) {
  x.x = fmaxf(x.x, -126.f);
  x.y = fmaxf(x.y, -126.f);
  const float2 magic = make_float2(12582912.f, 12582912.f);
  const float2 t = __fadd2_rn(x, magic);
  const float2 r = __fadd2_rn(t, make_float2(-12582912.f, -12582912.f));
  const float2 f = __fadd2_rn(x, make_float2(-r.x, -r.y));
  float2 q = __ffma2_rn(f, make_float2(0.055088683807510905f, 0.055088683807510905f),
                        make_float2(0.24260405145947916f, 0.24260405145947916f));
  q = __ffma2_rn(q, f, make_float2(0.6932762416819607f, 0.6932762416819607f));
  q = __ffma2_rn(q, f, make_float2(0.9999289403695112f, 0.9999289403695112f));
  return make_float2(__int_as_float(__float_as_int(t.x) * (1 << 23) + __float_as_int(q.x)),
                     __int_as_float(__float_as_int(t.y) * (1 << 23) + __float_as_int(q.y)));
}

#ifndef HP_FA_POLY
#define HP_FA_POLY 0  // score pairs per 32-pair half computed on the FMA pipe
#endif

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
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

// ---------------------------------------------------------------------------
// k_fa2: two 128-query tiles (A = rows q0.., B = rows q0+128..) of one
// (sequence, head) per unit, sharing every K/V tile.  P never touches shared
// memory: the softmax warps write it as packed bf16 into the TMEM columns of
// the S tile it came from, and O += P.V is issued with A = P from TMEM
// (tcgen05.mma ... [d], [a_tmem], b_desc).  The MMA warp ping-pongs the two
// tiles, so while softmax group A works on S_A(j+1) the tensor core runs
// PV_B(j) and QK_B(j+1), and vice versa:
//     PV_A(j)  QK_A(j+1)  PV_B(j)  QK_B(j+1)  PV_A(j+1) ...
// tcgen05 ops of one issuing thread execute in order, which is what makes
// QK_X(j+1) overwriting S_X/P_X after PV_X(j) safe and makes O_X stable
// whenever s_full_X fires (rescale point).
// Warps: 0 producer, 1 TMEM alloc + MMA issuer, 2-3 idle (warpgroup 0 gives
// registers away: setmaxnreg 96), 4-7 softmax A, 8-11 softmax B
// (setmaxnreg 200: the 128-score row stays in registers without spills).
// TMEM: S_A [0,128) S_B [128,256) O_A [256,256+D) O_B [256+D, 256+2D).
constexpr int FA2_THREADS = 384;
constexpr int FA2_SOFTMAX_WARP0 = 4;

template <int D>
struct Fa2Cfg {
  static constexpr int NB = D / 64;
  static constexpr uint32_t QB = NB * BOX;
  static constexpr uint32_t KB = NB * BOX;
  static constexpr size_t SMEM = 1024 + 2 * QB + KST * KB + VST * KB + 512;
};

struct Unit2 {
  int head, seq, s0, len, prior, kvlen;
  int q0;          // first query row (tile A) within the new span
  int nA, nB;      // kv tiles of tile A / tile B (nB = 0: tile B absent)
};

template <bool PAGED>
__device__ __forceinline__ bool unit2_of(const FaParams& p, int u, Unit2& x) {
  x.head = u % p.Hq;
  const int rest = u / p.Hq;
  x.seq = rest % p.nseq;
  const int qp = p.n_qt - 1 - rest / p.nseq;  // n_qt counts 256-row pairs here
  x.s0 = p.cu_seqlens[x.seq];
  x.len = p.cu_seqlens[x.seq + 1] - x.s0;
  x.q0 = qp * 2 * FQ;
  if (x.q0 >= x.len) return false;
  x.prior = PAGED ? p.prior_lens[x.seq] : 0;
  x.kvlen = x.prior + x.len;
  const int kvt = (x.kvlen + FK - 1) / FK;
  x.nA = min((x.prior + x.q0 + FQ + FK - 1) / FK, kvt);
  x.nB = (x.q0 + FQ < x.len) ? min((x.prior + x.q0 + 2 * FQ + FK - 1) / FK, kvt) : 0;
  return true;
}

__device__ __forceinline__ void umma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                             uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Units are sorted longest-first; CTA b takes unit r*G + b in even rounds and
// r*G + (G-1-b) in odd ones ("snake" order), which balances the causal
// triangle's per-unit work to within a few % of greedy LPT (round-robin
// leaves the first CTAs ~30% over the mean at T = 4096).
__device__ __forceinline__ int snake_unit(int r) {
  return r * int(gridDim.x) + ((r & 1) ? int(gridDim.x) - 1 - int(blockIdx.x) : int(blockIdx.x));
}

template <int D, bool PAGED>
__global__ void __launch_bounds__(FA2_THREADS, 1)
    k_fa2(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
          const __grid_constant__ CUtensorMap tmV, const FaParams p) {
  using C = Fa2Cfg<D>;
  pdl_trigger();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                 // [2][QB]
  uint8_t* sK = sQ + 2 * C::QB;
  uint8_t* sV = sK + KST * C::KB;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + VST * C::KB);
  uint64_t* q_full = bars + 0;
  uint64_t* q_empty = bars + 1;
  uint64_t* k_full = bars + 2;             // [KST]
  uint64_t* k_empty = k_full + KST;
  uint64_t* v_full = k_empty + KST;        // [VST]
  uint64_t* v_empty = v_full + VST;
  uint64_t* s_full = v_empty + VST;        // [2] per tile
  uint64_t* p_full = s_full + 2;           // [2]
  uint64_t* o_full = p_full + 2;           // [2]
  uint64_t* o_empty = o_full + 2;          // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_empty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmQ);
    if (!PAGED) {
      tma_prefetch_desc(&tmK);
      tma_prefetch_desc(&tmV);
    }
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int s = 0; s < KST; ++s) { mbar_init(&k_full[s], 1); mbar_init(&k_empty[s], 1); }
    for (int s = 0; s < VST; ++s) { mbar_init(&v_full[s], 1); mbar_init(&v_empty[s], 1); }
    for (int t = 0; t < 2; ++t) {
      mbar_init(&s_full[t], 1);
      mbar_init(&p_full[t], 4);
      mbar_init(&o_full[t], 1);
      mbar_init(&o_empty[t], 4);
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    tmem_alloc(tmem_slot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_wait();  // qkv from the QKV GEMM / rope_kv_write; `out` may still be read upstream
  uint64_t t_start = 0;
  if (p.cta_times != nullptr && threadIdx.x == 0) t_start = globaltimer();
  const uint32_t tmem = *tmem_slot;
  const int total = p.nseq * p.n_qt * p.Hq;
  // per SM sub-partition: one warp of each warpgroup, 96 + 200 + 200 <= 3 x 168 (the pool the launch got)
  if (warp < FA2_SOFTMAX_WARP0) {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 96;\n" ::: "memory");
  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      uint32_t un = 0, kt = 0, vt = 0;
      for (int r = 0; r * int(gridDim.x) < total; ++r) {
        const int u = snake_unit(r);
        if (u >= total) continue;
        Unit2 x;
        if (!unit2_of<PAGED>(p, u, x)) continue;
        const int kvh = x.head / p.G;
        const int J = max(x.nA, x.nB);
        mbar_wait(q_empty, (un & 1) ^ 1);
        mbar_arrive_expect_tx(q_full, C::QB * (x.nB > 0 ? 2 : 1));
        for (int t = 0; t < (x.nB > 0 ? 2 : 1); ++t)
          for (int b = 0; b < C::NB; ++b)
            tma_load_2d(sQ + t * C::QB + b * BOX, &tmQ, q_full, x.head * D + b * 64, x.s0 + x.q0 + t * FQ);
        for (int j = 0; j < J; ++j, ++kt, ++vt) {
          const int ks = kt % KST, vs = vt % VST;
          mbar_wait(&k_empty[ks], ((kt / KST) & 1) ^ 1);
          mbar_arrive_expect_tx(&k_full[ks], C::KB);
          if constexpr (PAGED) {
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
      uint32_t un = 0, kt = 0, vt = 0;
      uint32_t pc[2] = {0, 0};   // P tiles consumed per softmax group (p_full phases)
      uint32_t oc[2] = {0, 0};   // units per group (o_empty phases)
      auto qk = [&](int t, uint32_t kslot) {
        const uint32_t qa = smem_u32(sQ + t * C::QB), kb = smem_u32(sK + kslot * C::KB);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          umma_bf16(tmem + t * 128, umma_desc_sw128(qa + (kk >> 2) * BOX + (kk & 3) * 32),
                    umma_desc_sw128(kb + (kk >> 2) * BOX + (kk & 3) * 32), idesc_qk, kk > 0 ? 1u : 0u);
        umma_commit(&s_full[t]);
      };
      auto pv = [&](int t, uint32_t vslot, bool first) {
        const uint32_t vb = smem_u32(sV + vslot * C::KB);
#pragma unroll
        for (int kk = 0; kk < FK / 16; ++kk)
          umma_bf16_ts(tmem + 256 + t * D, tmem + t * 128 + kk * 8, desc_mn_sw128(vb + kk * 2048, BOX),
                       idesc_pv, (first && kk == 0) ? 0u : 1u);
      };
      for (int r = 0; r * int(gridDim.x) < total; ++r) {
        const int u = snake_unit(r);
        if (u >= total) continue;
        Unit2 x;
        if (!unit2_of<PAGED>(p, u, x)) continue;
        const int n[2] = {x.nA, x.nB};
        const int J = max(x.nA, x.nB);
        const bool utr = p.trace && blockIdx.x == 0 && un < 256;
        if (utr) p.trace[16 * 256 + un] = clock64();
        mbar_wait(q_full, un & 1);
        if (utr) p.trace[12 * 256 + un] = clock64();
        // prologue: S(0) for both tiles
        {
          const int ks = kt % KST;
          mbar_wait(&k_full[ks], (kt / KST) & 1);
          tc_fence_after();
#pragma unroll
          for (int t = 0; t < 2; ++t)
            if (n[t] > 0) qk(t, ks);
          if (J == 1) umma_commit(q_empty);  // the prologue's QKs were the unit's last
        }
        for (int j = 0; j < J; ++j) {
          const uint32_t vs = (vt + j) % VST;
          const uint32_t ks_cur = (kt + j) % KST, ks_nxt = (kt + j + 1) % KST;
          bool k_next_ready = false;
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            if (j >= n[t]) continue;
            const bool tr = p.trace && blockIdx.x == 0 && pc[t] < 256;
            if (tr) p.trace[(8 + t * 2) * 256 + pc[t]] = clock64();
            mbar_wait(&p_full[t], pc[t] & 1);
            if (tr) p.trace[(8 + t * 2 + 1) * 256 + pc[t]] = clock64();
            ++pc[t];
            if (j == 0) mbar_wait(&o_empty[t], (oc[t] & 1) ^ 1);
            mbar_wait(&v_full[vs], ((vt + j) / VST) & 1);
            tc_fence_after();
            pv(t, vs, j == 0);
            if (j + 1 < n[t]) {
              if (!k_next_ready) {
                mbar_wait(&k_full[ks_nxt], ((kt + j + 1) / KST) & 1);
                tc_fence_after();
                k_next_ready = true;
              }
              qk(t, ks_nxt);
            } else {
              umma_commit(&o_full[t]);
              ++oc[t];
            }
          }
          umma_commit(&v_empty[vs]);
          umma_commit(&k_empty[ks_cur]);  // K_j: read by QK(j) of both tiles, all issued
          // Q is read only by QK: free it once the unit's last QK is issued
          // (j = J - 2), so the producer loads the next unit's Q while this
          // unit's last PV / softmax / epilogue run, not after them
          if (j == J - 2) umma_commit(q_empty);
        }
        if (utr) p.trace[13 * 256 + un] = clock64();
        kt += J;
        vt += J;
        ++un;
      }
    }
  }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 200;\n" ::: "memory");
    // ------------------------------------------------------------- softmax
    const int t = (warp - FA2_SOFTMAX_WARP0) >> 2;  // tile 0 (A) or 1 (B)
    const int q4 = warp & 3;                // TMEM lane quarter
    const int row = q4 * 32 + lane;
    const uint32_t lane_base = uint32_t(q4 * 32) << 16;
    const uint32_t tS = tmem + lane_base + t * 128;
    const uint32_t tO = tmem + lane_base + 256 + t * D;
    uint32_t sc = 0, un = 0;
    for (int r = 0; r * int(gridDim.x) < total; ++r) {
        const int u = snake_unit(r);
        if (u >= total) continue;
      Unit2 x;
      if (!unit2_of<PAGED>(p, u, x)) continue;
      const int nt = t == 0 ? x.nA : x.nB;
      if (nt == 0) continue;
      const int q0 = x.q0 + t * FQ;
      const int qi = q0 + row;
      const int qpos = x.prior + qi;
      float m_run = -INFINITY, l = 0.f;
      for (int j = 0; j < nt; ++j, ++sc) {
        const bool tr = p.trace && blockIdx.x == 0 && lane == 0 && q4 == 0 && sc < 256;
        if (tr) p.trace[(t * 4 + 0) * 256 + sc] = clock64();
        mbar_wait(&s_full[t], sc & 1);
        if (tr) p.trace[(t * 4 + 1) * 256 + sc] = clock64();
        tc_fence_after();
        float s[128];
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_ld32(tS + c * 32, s + c * 32);
        tmem_ld_wait();
        if (tr) p.trace[(t * 4 + 2) * 256 + sc] = clock64();
        const int kbase = j * FK;
        const bool need_mask = (kbase + FK - 1 > x.prior + q0) || (kbase + FK > x.kvlen);
        if (need_mask) {
          const int lim = min(qpos + 1, x.kvlen) - kbase;  // keys [0, lim) visible
#pragma unroll
          for (int c = 0; c < 128; ++c)
            if (c >= lim) s[c] = -INFINITY;
        }
        // raw-score row max with 8 independent chains (ILP), then scale once
        // 3-input FMNMX3: 8 chains take two scores per instruction
        float m8[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) m8[k] = s[k];
#pragma unroll
        for (int c = 8; c < 128; c += 16)
#pragma unroll
          for (int k = 0; k < 8; ++k) m8[k] = fmax3(m8[k], s[c + k], s[c + 8 + k]);
        const float mx = fmax3(fmax3(m8[0], m8[1], m8[2]), fmax3(m8[3], m8[4], m8[5]), fmaxf(m8[6], m8[7])) *
                         p.scale_log2;
        const float m_new = fmaxf(m_run, mx);
        const bool grow = m_new > m_run + RESCALE_THRESHOLD;
        // O_t holds PV(0..j-1), complete (issued before QK(j)); rescale lazily
        if (__any_sync(0xffffffffu, grow) && j > 0) {
          const float alpha = grow ? exp2f(m_run - m_new) : 1.f;
#pragma unroll 1
          for (int c = 0; c < D / 32; ++c) {
            float o[32];
            tmem_ld32(tO + c * 32, o);
            tmem_ld_wait();
#pragma unroll
            for (int k = 0; k < 32; ++k) o[k] *= alpha;
            tmem_st32(tO + c * 32, o);
          }
          if (grow) l *= alpha;
        }
        if (grow) m_run = m_new;
        const float mb = (m_run == -INFINITY) ? 0.f : m_run;
        // P = exp2(s * scale_log2 - m): packed f32x2 FFMA + two MUFU per
        // score pair, bf16 pairs over the first 64 columns of S_t; 4 packed
        // partial row sums (FADD2).  ~3 issue slots per score.
        const float2 sc2 = make_float2(p.scale_log2, p.scale_log2);
        const float2 nm2 = make_float2(-mb, -mb);
        float2 l4[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                        make_float2(0.f, 0.f)};
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          float w[32];
          uint32_t* wu = reinterpret_cast<uint32_t*>(w);
#pragma unroll
          for (int k = 0; k < 32; ++k) {
            float2 x = __ffma2_rn(make_float2(s[h * 64 + 2 * k], s[h * 64 + 2 * k + 1]), sc2, nm2);
            if (k < HP_FA_POLY) {
              x = ex2_poly2(x);
            } else {
              x.x = ex2(x.x);
              x.y = ex2(x.y);
            }
            l4[k & 3] = __fadd2_rn(l4[k & 3], x);
            wu[k] = pack_bf16(x.x, x.y);
          }
          tmem_st32(tS + h * 32, w);
        }
        const float2 ls = __fadd2_rn(__fadd2_rn(l4[0], l4[1]), __fadd2_rn(l4[2], l4[3]));
        l += ls.x + ls.y;
        tmem_st_wait();
        if (tr) p.trace[(t * 4 + 3) * 256 + sc] = clock64();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[t]);
      }
      // epilogue: O / l -> global
      const bool etr = p.trace && blockIdx.x == 0 && lane == 0 && q4 == 0 && t == 0 && un < 256;
      if (etr) p.trace[17 * 256 + un] = clock64();
      mbar_wait(&o_full[t], un & 1);
      if (etr) p.trace[14 * 256 + un] = clock64();
      tc_fence_after();
      const float inv = l > 0.f ? 1.f / l : 0.f;
      const bool ok = qi < x.len;
      __nv_bfloat16* orow = p.out + size_t(x.s0 + qi) * p.ldo + size_t(x.head) * D;
#pragma unroll 1
      for (int c = 0; c < D / 32; ++c) {
        float o[32];
        tmem_ld32(tO + c * 32, o);
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
      if (lane == 0) mbar_arrive(&o_empty[t]);
      if (etr) p.trace[15 * 256 + un] = clock64();
      ++un;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
  if (p.cta_times != nullptr && threadIdx.x == 0) {
    p.cta_times[blockIdx.x * 3 + 0] = smid();
    p.cta_times[blockIdx.x * 3 + 1] = t_start;
    p.cta_times[blockIdx.x * 3 + 2] = globaltimer();
  }
}

// ---------------------------------------------------------------------------
// k_fa2p: the CTA-pair form of k_fa2 (dense operands, D = 128).  A 2-CTA
// cluster owns a (sequence, 512-query block, q head) unit: tile A = rows
// [q0, q0+256), tile B = [q0+256, q0+512), CTA r holding rows 128r.. of
// each.  The leader issues tcgen05.mma.cta_group::2 (M = 256):
//     S_X  = Q_X . K_j^T   (N = 128 keys; each CTA stages 64 keys of K_j)
//     O_X += P_X . V_j     (N = D = 128; each CTA stages 64 dims of V_j,
//                           A = P from each CTA's own TMEM)
// so the pair MMAs run at the full 4096 MAC/clk/SM (the 1-CTA SS M=128 N=128
// QK reaches 58 %, profiles/r01_umma_rates.md) and every K/V byte crosses
// one SM's shared-memory port instead of two.  The two tiles ping-pong as in
// k_fa2: PV_A(j) QK_A(j+1) PV_B(j) QK_B(j+1).  Each CTA's softmax warps work
// on their own 128 rows (TMEM lanes) and arrive on the leader's p_full /
// o_empty (count 8); s_full / o_full / the ring's empty barriers are
// committed to both CTAs.
constexpr int FAP_THREADS = 384;
constexpr int FAP_KST = 3;   // K ring stages (16 KB per CTA each)
constexpr int FAP_VST = 3;   // V ring stages

struct FapCfg {
  static constexpr uint32_t QB = 2 * BOX;           // one CTA's 128 rows x 128 dims (32 KB)
  static constexpr uint32_t KB = 2 * (BOX / 2);     // 64 keys x 128 dims (16 KB)
  static constexpr uint32_t VB = BOX;               // 128 keys x 64 dims (16 KB)
  static constexpr size_t SMEM = 1024 + 2 * QB + FAP_KST * KB + FAP_VST * VB + 512;
};

struct UnitP {
  int head, seq, s0, len;
  int q0;          // first query row of tile A (512-row block)
  int nA, nB;      // kv tiles of tile A / tile B (nB = 0: tile B absent)
};

__device__ __forceinline__ bool unitp_of(const FaParams& p, int u, UnitP& x) {
  x.head = u % p.Hq;
  const int rest = u / p.Hq;
  x.seq = rest % p.nseq;
  const int qb = p.n_qt - 1 - rest / p.nseq;  // n_qt counts 512-row blocks here
  x.s0 = p.cu_seqlens[x.seq];
  x.len = p.cu_seqlens[x.seq + 1] - x.s0;
  x.q0 = qb * 4 * FQ;
  if (x.q0 >= x.len) return false;
  const int kvt = (x.len + FK - 1) / FK;
  x.nA = min((x.q0 + 2 * FQ + FK - 1) / FK, kvt);
  x.nB = (x.q0 + 2 * FQ < x.len) ? min((x.q0 + 4 * FQ + FK - 1) / FK, kvt) : 0;
  return true;
}

__device__ __forceinline__ void umma_bf16_ts_pair(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                                  uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// snake order over the grid's CTA pairs
__device__ __forceinline__ int snake_unit_pair(int r) {
  const int np = int(gridDim.x) >> 1, pi = int(blockIdx.x) >> 1;
  return r * np + ((r & 1) ? np - 1 - pi : pi);
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(FAP_THREADS, 1)
    k_fa2p(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK64,
           const __grid_constant__ CUtensorMap tmV, const FaParams p) {
  constexpr int D = 128;
  using C = FapCfg;
  pdl_trigger();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                 // [2 tiles][QB]
  uint8_t* sK = sQ + 2 * C::QB;       // [KST][KB]
  uint8_t* sV = sK + FAP_KST * C::KB; // [VST][VB]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + FAP_VST * C::VB);
  uint64_t* q_full = bars + 0;
  uint64_t* q_empty = bars + 1;
  uint64_t* k_full = bars + 2;                 // [KST]
  uint64_t* k_empty = k_full + FAP_KST;
  uint64_t* v_full = k_empty + FAP_KST;        // [VST]
  uint64_t* v_empty = v_full + FAP_VST;
  uint64_t* s_full = v_empty + FAP_VST;        // [2] per tile
  uint64_t* p_full = s_full + 2;               // [2] (leader's, count 8)
  uint64_t* o_full = p_full + 2;               // [2]
  uint64_t* o_empty = o_full + 2;              // [2] (leader's, count 8)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_empty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK64);
    tma_prefetch_desc(&tmV);
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int s = 0; s < FAP_KST; ++s) { mbar_init(&k_full[s], 1); mbar_init(&k_empty[s], 1); }
    for (int s = 0; s < FAP_VST; ++s) { mbar_init(&v_full[s], 1); mbar_init(&v_empty[s], 1); }
    for (int t = 0; t < 2; ++t) {
      mbar_init(&s_full[t], 1);
      mbar_init(&p_full[t], 8);
      mbar_init(&o_full[t], 1);
      mbar_init(&o_empty[t], 8);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_pair(tmem_slot, 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  pdl_wait();
  uint64_t t_start = 0;
  if (p.cta_times != nullptr && threadIdx.x == 0) t_start = globaltimer();
  const uint32_t tmem = *tmem_slot;
  const int total = p.nseq * p.n_qt * p.Hq;
  const int npairs = int(gridDim.x) >> 1;
  if (warp < FA2_SOFTMAX_WARP0) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 96;\n" ::: "memory");
    if (warp == 0) {
      // ---------------------------------------------------------- producer
      // this CTA's halves, completing on the LEADER's barriers (pair TMA)
      if (lane == 0) {
        const uint32_t lq = mapa_shared(q_full, 0), lk = mapa_shared(k_full, 0), lv = mapa_shared(v_full, 0);
        uint32_t un = 0, kt = 0, vt = 0;
        for (int r = 0; r * npairs < total; ++r) {
          const int u = snake_unit_pair(r);
          if (u >= total) continue;
          UnitP x;
          if (!unitp_of(p, u, x)) continue;
          const int kvh = x.head / p.G;
          const int ntile = x.nB > 0 ? 2 : 1;
          const int J = max(x.nA, x.nB);
          mbar_wait(q_empty, (un & 1) ^ 1);
          if (leader) mbar_arrive_expect_tx(q_full, 2 * C::QB * ntile);
          for (int t = 0; t < ntile; ++t)
            for (int b = 0; b < 2; ++b)
              tma_load_2d_pair(sQ + t * C::QB + b * BOX, &tmQ, lq, x.head * D + b * 64,
                               x.s0 + x.q0 + t * 2 * FQ + int(rank) * FQ);
          for (int j = 0; j < J; ++j, ++kt, ++vt) {
            const int ks = kt % FAP_KST, vs = vt % FAP_VST;
            mbar_wait(&k_empty[ks], ((kt / FAP_KST) & 1) ^ 1);
            if (leader) mbar_arrive_expect_tx(&k_full[ks], 2 * C::KB);
            for (int b = 0; b < 2; ++b)  // keys [64 rank, +64) of K_j, both 64-dim halves
              tma_load_2d_pair(sK + ks * C::KB + b * (BOX / 2), &tmK64, lk + 8u * ks, kvh * D + b * 64,
                               x.s0 + j * FK + int(rank) * 64);
            mbar_wait(&v_empty[vs], ((vt / FAP_VST) & 1) ^ 1);
            if (leader) mbar_arrive_expect_tx(&v_full[vs], 2 * C::VB);
            // dims [64 rank, +64) of V_j, all 128 keys
            tma_load_2d_pair(sV + vs * C::VB, &tmV, lv + 8u * vs, kvh * D + int(rank) * 64, x.s0 + j * FK);
          }
          ++un;
        }
      }
    } else if (warp == 1 && leader) {
      // ------------------------------------------------------ MMA issuer
      if (lane == 0) {
        constexpr uint32_t idesc_qk = umma_idesc_bf16(2 * FQ, FK);
        constexpr uint32_t idesc_pv = umma_idesc_bf16(2 * FQ, D) | (1u << 16);  // B (V) MN-major
        uint32_t un = 0, kt = 0, vt = 0;
        uint32_t pc[2] = {0, 0};
        uint32_t oc[2] = {0, 0};
        auto qk = [&](int t, uint32_t kslot) {
          const uint32_t qa = smem_u32(sQ + t * C::QB), kb = smem_u32(sK + kslot * C::KB);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk)
            umma_bf16_pair(tmem + t * 128, umma_desc_sw128(qa + (kk >> 2) * BOX + (kk & 3) * 32),
                           umma_desc_sw128(kb + (kk >> 2) * (BOX / 2) + (kk & 3) * 32), idesc_qk,
                           kk > 0 ? 1u : 0u);
          umma_commit_pair(&s_full[t]);
        };
        auto pv = [&](int t, uint32_t vslot, bool first) {
          const uint32_t vb = smem_u32(sV + vslot * C::VB);
#pragma unroll
          for (int kk = 0; kk < FK / 16; ++kk)
            umma_bf16_ts_pair(tmem + 256 + t * D, tmem + t * 128 + kk * 8, desc_mn_sw128(vb + kk * 2048, BOX),
                              idesc_pv, (first && kk == 0) ? 0u : 1u);
        };
        for (int r = 0; r * npairs < total; ++r) {
          const int u = snake_unit_pair(r);
          if (u >= total) continue;
          UnitP x;
          if (!unitp_of(p, u, x)) continue;
          const int n[2] = {x.nA, x.nB};
          const int J = max(x.nA, x.nB);
          mbar_wait(q_full, un & 1);
          {
            const int ks = kt % FAP_KST;
            mbar_wait(&k_full[ks], (kt / FAP_KST) & 1);
            tc_fence_after();
#pragma unroll
            for (int t = 0; t < 2; ++t)
              if (n[t] > 0) qk(t, ks);
            if (J == 1) umma_commit_pair(q_empty);
          }
          for (int j = 0; j < J; ++j) {
            const uint32_t vs = (vt + j) % FAP_VST;
            const uint32_t ks_cur = (kt + j) % FAP_KST, ks_nxt = (kt + j + 1) % FAP_KST;
            bool k_next_ready = false;
#pragma unroll
            for (int t = 0; t < 2; ++t) {
              if (j >= n[t]) continue;
              mbar_wait_cluster(&p_full[t], pc[t] & 1);
              ++pc[t];
              if (j == 0) mbar_wait_cluster(&o_empty[t], (oc[t] & 1) ^ 1);
              mbar_wait(&v_full[vs], ((vt + j) / FAP_VST) & 1);
              tc_fence_after();
              pv(t, vs, j == 0);
              if (j + 1 < n[t]) {
                if (!k_next_ready) {
                  mbar_wait(&k_full[ks_nxt], ((kt + j + 1) / FAP_KST) & 1);
                  tc_fence_after();
                  k_next_ready = true;
                }
                qk(t, ks_nxt);
              } else {
                umma_commit_pair(&o_full[t]);
                ++oc[t];
              }
            }
            umma_commit_pair(&v_empty[vs]);
            umma_commit_pair(&k_empty[ks_cur]);
            if (j == J - 2) umma_commit_pair(q_empty);  // last QK issued (see k_fa2)
          }
          kt += J;
          vt += J;
          ++un;
        }
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 200;\n" ::: "memory");
    // ------------------------------------------------------------- softmax
    const int t = (warp - FA2_SOFTMAX_WARP0) >> 2;  // tile 0 (A) or 1 (B)
    const int q4 = warp & 3;
    const int row = q4 * 32 + lane;
    const uint32_t lane_base = uint32_t(q4 * 32) << 16;
    const uint32_t tS = tmem + lane_base + t * 128;
    const uint32_t tO = tmem + lane_base + 256 + t * D;
    const uint32_t lp_full = mapa_shared(&p_full[t], 0), lo_empty = mapa_shared(&o_empty[t], 0);
    uint32_t sc = 0, un = 0;
    for (int r = 0; r * npairs < total; ++r) {
      const int u = snake_unit_pair(r);
      if (u >= total) continue;
      UnitP x;
      if (!unitp_of(p, u, x)) continue;
      const int nt = t == 0 ? x.nA : x.nB;
      if (nt == 0) continue;
      const int q0 = x.q0 + t * 2 * FQ + int(rank) * FQ;  // this CTA's first row of tile t
      const int qi = q0 + row;
      float m_run = -INFINITY, l = 0.f;
      for (int j = 0; j < nt; ++j, ++sc) {
        mbar_wait(&s_full[t], sc & 1);
        tc_fence_after();
        float s[128];
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_ld32(tS + c * 32, s + c * 32);
        tmem_ld_wait();
        const int kbase = j * FK;
        const bool need_mask = (kbase + FK - 1 > q0) || (kbase + FK > x.len);
        if (need_mask) {
          const int lim = min(qi + 1, x.len) - kbase;  // keys [0, lim) visible
#pragma unroll
          for (int c = 0; c < 128; ++c)
            if (c >= lim) s[c] = -INFINITY;
        }
        // 3-input FMNMX3: 8 chains take two scores per instruction
        float m8[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) m8[k] = s[k];
#pragma unroll
        for (int c = 8; c < 128; c += 16)
#pragma unroll
          for (int k = 0; k < 8; ++k) m8[k] = fmax3(m8[k], s[c + k], s[c + 8 + k]);
        const float mx = fmax3(fmax3(m8[0], m8[1], m8[2]), fmax3(m8[3], m8[4], m8[5]), fmaxf(m8[6], m8[7])) *
                         p.scale_log2;
        const float m_new = fmaxf(m_run, mx);
        const bool grow = m_new > m_run + RESCALE_THRESHOLD;
        if (__any_sync(0xffffffffu, grow) && j > 0) {
          const float alpha = grow ? exp2f(m_run - m_new) : 1.f;
#pragma unroll 1
          for (int c = 0; c < D / 32; ++c) {
            float o[32];
            tmem_ld32(tO + c * 32, o);
            tmem_ld_wait();
#pragma unroll
            for (int k = 0; k < 32; ++k) o[k] *= alpha;
            tmem_st32(tO + c * 32, o);
          }
          if (grow) l *= alpha;
        }
        if (grow) m_run = m_new;
        const float mb = (m_run == -INFINITY) ? 0.f : m_run;
        const float2 sc2 = make_float2(p.scale_log2, p.scale_log2);
        const float2 nm2 = make_float2(-mb, -mb);
        float2 l4[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                        make_float2(0.f, 0.f)};
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          float w[32];
          uint32_t* wu = reinterpret_cast<uint32_t*>(w);
#pragma unroll
          for (int k = 0; k < 32; ++k) {
            float2 v2 = __ffma2_rn(make_float2(s[h * 64 + 2 * k], s[h * 64 + 2 * k + 1]), sc2, nm2);
            if (k < HP_FA_POLY) {
              v2 = ex2_poly2(v2);
            } else {
              v2.x = ex2(v2.x);
              v2.y = ex2(v2.y);
            }
            l4[k & 3] = __fadd2_rn(l4[k & 3], v2);
            wu[k] = pack_bf16(v2.x, v2.y);
          }
          tmem_st32(tS + h * 32, w);
        }
        const float2 ls = __fadd2_rn(__fadd2_rn(l4[0], l4[1]), __fadd2_rn(l4[2], l4[3]));
        l += ls.x + ls.y;
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster_relaxed(lp_full);
      }
      mbar_wait(&o_full[t], un & 1);
      tc_fence_after();
      const float inv = l > 0.f ? 1.f / l : 0.f;
      const bool ok = qi < x.len;
      __nv_bfloat16* orow = p.out + size_t(x.s0 + qi) * p.ldo + size_t(x.head) * D;
#pragma unroll 1
      for (int c = 0; c < D / 32; ++c) {
        float o[32];
        tmem_ld32(tO + c * 32, o);
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
      if (lane == 0) mbar_arrive_cluster_relaxed(lo_empty);
      ++un;
    }
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair(tmem, 512);
  }
  if (p.cta_times != nullptr && threadIdx.x == 0) {
    p.cta_times[blockIdx.x * 3 + 0] = smid();
    p.cta_times[blockIdx.x * 3 + 1] = t_start;
    p.cta_times[blockIdx.x * 3 + 2] = globaltimer();
  }
}

// Pair form for long prompts (max_seqlen >= 8192) on >= 2 SMs: measured
// (tools/fa_ab.py) 1272 vs 1231 TFLOP/s at T = 16384 on 148 SMs, but 923 vs
// 968 at T = 4096 on 140 (512-row units: fewer of them, more causal waste on
// the diagonal).  Either way the pair lifts the MMA rate and halves the K/V
// shared-memory traffic yet gains little: the softmax chain, not the tensor
// core, bounds k_fa2.  HP_FA_PAIR=0|1 forces it off/on.
static bool fa_pair_enabled(int max_ctas, int max_seqlen) {
  static const int forced = [] {
    const char* e = std::getenv("HP_FA_PAIR");
    return e ? (e[0] == '0' ? 0 : 1) : -1;
  }();
  if (max_ctas < 2 || forced == 0) return false;
  return forced == 1 || max_seqlen >= 8192;
}

static int launch_fa2p(const CUtensorMap& tq, const CUtensorMap& tk64, const CUtensorMap& tv, FaParams p,
                       int max_seqlen, int max_ctas, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    HP_CUDA_TRY(cudaFuncSetAttribute(k_fa2p, cudaFuncAttributeMaxDynamicSharedMemorySize, int(FapCfg::SMEM)));
    attr = true;
  }
  p.n_qt = (max_seqlen + 4 * FQ - 1) / (4 * FQ);
  const int pairs = std::min(p.nseq * p.n_qt * p.Hq, max_ctas / 2);
  HP_LAUNCH_PDL("k_fa2p", k_fa2p, dim3(2 * pairs), dim3(FAP_THREADS), FapCfg::SMEM, st, tq, tk64, tv, p);
  return HP_OK;
}

template <int D, bool PAGED>
static int launch_fa2(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv, FaParams p,
                      int max_seqlen, int max_ctas, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    HP_CUDA_TRY(cudaFuncSetAttribute(k_fa2<D, PAGED>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(Fa2Cfg<D>::SMEM)));
    attr = true;
  }
  p.n_qt = (max_seqlen + 2 * FQ - 1) / (2 * FQ);
  const int grid = std::min(p.nseq * p.n_qt * p.Hq, max_ctas);
  HP_LAUNCH_PDL("k_fa2", k_fa2<D, PAGED>, dim3(grid), dim3(FA2_THREADS), Fa2Cfg<D>::SMEM, st, tq, tk, tv, p);
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
  p.Hq = Hq;
  p.G = Hq / Hkv;
  p.out = static_cast<__nv_bfloat16*>(o);
  p.ldo = ldo;
  p.scale_log2 = scale * 1.4426950408889634f;
  p.trace = static_cast<long long*>(trace_buf(TRACE_FA));
  p.cta_times = take_cta_trace();
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (d == 128 && p.trace == nullptr && fa_pair_enabled(max_ctas, max_seqlen)) {
    CUtensorMap tk64;  // the pair stages 64 keys of each K tile per CTA
    rc = cached_tmap_bf16(&tk64, k, rows, uint64_t(Hkv) * d, ldk, 64, 64, true);
    if (rc) return rc;
    return launch_fa2p(tq, tk64, tv, p, max_seqlen, max_ctas, st);
  }
  return d == 128 ? launch_fa2<128, false>(tq, tk, tv, p, max_seqlen, max_ctas, st)
                  : launch_fa2<64, false>(tq, tk, tv, p, max_seqlen, max_ctas, st);
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
  p.cta_times = take_cta_trace();
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  return d == 128 ? launch_fa2<128, true>(tq, tq, tq, p, max_seqlen, max_ctas, st)
                  : launch_fa2<64, true>(tq, tq, tq, p, max_seqlen, max_ctas, st);
}
