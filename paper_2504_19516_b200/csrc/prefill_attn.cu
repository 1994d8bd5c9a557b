// Causal GQA prefill attention over the new span (reference kernel group
// "attn", phase prefill with prior_lens = 0; workload.py:176-183).
//
// Flash-attention tiling: a CTA owns one (sequence, 64-query tile, q head)
// unit; four consumer warps each hold 16 query rows and stream the causal
// prefix of 64-token K/V tiles through a 2-stage TMA ring (128B swizzle) fed
// by a producer warp.  S = Q K^T and O += P V run on mma.sync m16n8k16 with
// fp32 accumulation and an exp2 online softmax; P never leaves registers.
// Units are issued longest-first (descending query tile) so the causal
// triangle load-balances across the persistent grid.
//
// Inputs are the fused qkv projection buffer (q/k/v column blocks, any row
// pitch), so no re-layout copy follows the QKV GEMM.
#include "common.cuh"
#include "runtime.h"
#include "../../include/hp.h"

#include <algorithm>
#include <cmath>

namespace hp {

constexpr int PA_BQ = 64;
constexpr int PA_BK = 64;
constexpr int PA_STAGES = 2;
constexpr int PA_CONSUMERS = 4;
constexpr int PA_THREADS = (PA_CONSUMERS + 1) * 32;
constexpr uint32_t PA_BOX = 64 * 64 * 2;                 // 64 rows x 128 B (64 dims)

template <int D>
struct PaCfg {
  static constexpr int NBOX = D / 64;
  static constexpr uint32_t TILE_BYTES = NBOX * PA_BOX;  // 64 rows x D
  static constexpr uint32_t STAGE_BYTES = 2 * TILE_BYTES;  // K + V
  static constexpr size_t SMEM = 1024 + TILE_BYTES + PA_STAGES * STAGE_BYTES + 128;
};

struct PrefillParams {
  const int* cu_seqlens;
  int nseq, n_qt, Hq, Hkv, G;
  __nv_bfloat16* out;
  int ldo;
  float scale_log2;
};

template <int D>
__global__ void __launch_bounds__(PA_THREADS, 1)
    k_prefill_attn(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                   const __grid_constant__ CUtensorMap tmV, const PrefillParams p) {
  using C = PaCfg<D>;
  constexpr int KK = D / 16;
  constexpr uint32_t PA_TILE_BYTES = C::TILE_BYTES;
  constexpr uint32_t PA_STAGE_BYTES = C::STAGE_BYTES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* ring = smem + PA_TILE_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + PA_STAGES * PA_STAGE_BYTES);
  uint64_t* empty = full + PA_STAGES;
  uint64_t* qfull = empty + PA_STAGES;
  uint64_t* qempty = qfull + 1;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    for (int s = 0; s < PA_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], PA_CONSUMERS);
    }
    mbar_init(qfull, 1);
    mbar_init(qempty, PA_CONSUMERS);
    fence_barrier_init();
  }
  __syncthreads();

  const int total = p.nseq * p.n_qt * p.Hq;
  uint32_t gtile = 0;  // ring position across units
  uint32_t qphase = 0;

  for (int u = blockIdx.x; u < total; u += gridDim.x) {
    const int head = u % p.Hq;
    const int rest = u / p.Hq;
    const int seq = rest % p.nseq;
    const int qt = p.n_qt - 1 - rest / p.nseq;
    const int s0 = p.cu_seqlens[seq];
    const int len = p.cu_seqlens[seq + 1] - s0;
    if (qt * PA_BQ >= len) continue;
    const int kvh = head / p.G;
    const int q0 = qt * PA_BQ;
    const int nkv = min((q0 + PA_BQ + PA_BK - 1) / PA_BK, (len + PA_BK - 1) / PA_BK);

    if (warp == PA_CONSUMERS) {
      if (lane == 0) {
        mbar_wait(qempty, qphase ^ 1);
        mbar_arrive_expect_tx(qfull, PA_TILE_BYTES);
#pragma unroll
        for (int bx = 0; bx < C::NBOX; ++bx)
          tma_load_2d(sQ + bx * PA_BOX, &tmQ, qfull, head * D + bx * 64, s0 + q0);
        for (int j = 0; j < nkv; ++j) {
          const uint32_t g = gtile + j;
          const int st = g % PA_STAGES;
          const uint32_t ph = (g / PA_STAGES) & 1;
          mbar_wait(&empty[st], ph ^ 1);
          mbar_arrive_expect_tx(&full[st], PA_STAGE_BYTES);
          uint8_t* sb = ring + st * PA_STAGE_BYTES;
          const int row = s0 + j * PA_BK;
#pragma unroll
          for (int bx = 0; bx < C::NBOX; ++bx) {
            tma_load_2d(sb + bx * PA_BOX, &tmK, &full[st], kvh * D + bx * 64, row);
            tma_load_2d(sb + PA_TILE_BYTES + bx * PA_BOX, &tmV, &full[st], kvh * D + bx * 64, row);
          }
        }
      }
    } else {
      const int g8 = lane >> 2;
      const int t4 = lane & 3;
      const int mat = lane >> 3;
      // ---- Q fragments (A operand, 16 rows per warp)
      mbar_wait(qfull, qphase);
      uint32_t qf[KK][4];
      {
        const uint32_t qb = smem_u32(sQ);
#pragma unroll
        for (int kk = 0; kk < KK; ++kk) {
          const uint32_t r = warp * 16 + (mat & 1) * 8 + (lane & 7);
          const uint32_t c = (kk & 3) * 2 + (mat >> 1);
          ldmatrix_x4(qb + (kk >> 2) * PA_BOX + sw128(r, c), qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(qempty);

      float o[2 * KK][4];
#pragma unroll
      for (int i = 0; i < 2 * KK; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
      float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
      const int qi0 = q0 + warp * 16 + g8;  // rows owned: qi0 and qi0 + 8
      const int qi1 = qi0 + 8;

      for (int j = 0; j < nkv; ++j) {
        const uint32_t g = gtile + j;
        const int st = g % PA_STAGES;
        const uint32_t ph = (g / PA_STAGES) & 1;
        mbar_wait(&full[st], ph);
        const uint32_t kb = smem_u32(ring + st * PA_STAGE_BYTES);
        const uint32_t vb = kb + PA_TILE_BYTES;
        // ---- S = Q K^T : 16 x 64
        float s[8][4];
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
#pragma unroll
        for (int kk = 0; kk < KK; ++kk) {
#pragma unroll
          for (int np = 0; np < 4; ++np) {
            // two n8 tiles (16 kv tokens) per ldmatrix.x4
            const uint32_t r = np * 16 + (mat >> 1) * 8 + (lane & 7);
            const uint32_t c = (kk & 3) * 2 + (mat & 1);
            uint32_t b[4];
            ldmatrix_x4(kb + (kk >> 2) * PA_BOX + sw128(r, c), b[0], b[1], b[2], b[3]);
            mma_bf16_16816(s[2 * np], qf[kk], b);
            mma_bf16_16816(s[2 * np + 1], qf[kk], b + 2);
          }
        }
        // ---- causal / length mask + online softmax
        const int kbase = j * PA_BK;
        const bool need_mask = (kbase + PA_BK > q0) || (kbase + PA_BK > len);
        float tm0 = -INFINITY, tm1 = -INFINITY;
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) {
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int kj = kbase + nt * 8 + 2 * t4 + e;
            float v0 = s[nt][e] * p.scale_log2;
            float v1 = s[nt][2 + e] * p.scale_log2;
            if (need_mask) {
              if (kj > qi0 || kj >= len) v0 = -INFINITY;
              if (kj > qi1 || kj >= len) v1 = -INFINITY;
            }
            s[nt][e] = v0;
            s[nt][2 + e] = v1;
            tm0 = fmaxf(tm0, v0);
            tm1 = fmaxf(tm1, v1);
          }
        }
        tm0 = fmaxf(tm0, __shfl_xor_sync(0xffffffffu, tm0, 1));
        tm0 = fmaxf(tm0, __shfl_xor_sync(0xffffffffu, tm0, 2));
        tm1 = fmaxf(tm1, __shfl_xor_sync(0xffffffffu, tm1, 1));
        tm1 = fmaxf(tm1, __shfl_xor_sync(0xffffffffu, tm1, 2));
        const float n0 = fmaxf(m0, tm0), n1 = fmaxf(m1, tm1);
        // rows fully masked so far keep m = -inf; guard the rescale
        const float a0 = (n0 == -INFINITY) ? 1.f : exp2f(m0 - n0);
        const float a1 = (n1 == -INFINITY) ? 1.f : exp2f(m1 - n1);
        const float b0 = (n0 == -INFINITY) ? 0.f : n0;
        const float b1 = (n1 == -INFINITY) ? 0.f : n1;
        m0 = n0;
        m1 = n1;
        l0 *= a0;
        l1 *= a1;
#pragma unroll
        for (int dn = 0; dn < 2 * KK; ++dn) {
          o[dn][0] *= a0;
          o[dn][1] *= a0;
          o[dn][2] *= a1;
          o[dn][3] *= a1;
        }
        uint32_t pa[4][4];  // P as A fragments, one per 16-token k step
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) {
          const float p00 = exp2f(s[nt][0] - b0), p01 = exp2f(s[nt][1] - b0);
          const float p10 = exp2f(s[nt][2] - b1), p11 = exp2f(s[nt][3] - b1);
          l0 += p00 + p01;
          l1 += p10 + p11;
          pa[nt >> 1][(nt & 1) * 2 + 0] = pack_bf16(p00, p01);
          pa[nt >> 1][(nt & 1) * 2 + 1] = pack_bf16(p10, p11);
        }
        // ---- O += P V : 16 x 128
#pragma unroll
        for (int kt = 0; kt < 4; ++kt) {
#pragma unroll
          for (int dp = 0; dp < KK; ++dp) {
            // V^T fragments for two n8 d-tiles via transposed ldmatrix
            const uint32_t r = kt * 16 + (mat & 1) * 8 + (lane & 7);
            const uint32_t c = (dp & 3) * 2 + (mat >> 1);
            uint32_t b[4];
            ldmatrix_x4_trans(vb + (dp >> 2) * PA_BOX + sw128(r, c), b[0], b[1], b[2], b[3]);
            mma_bf16_16816(o[2 * dp], pa[kt], b);
            mma_bf16_16816(o[2 * dp + 1], pa[kt], b + 2);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
      }
      // ---- normalise and store
      l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
      l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
      l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
      l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
      const float i0 = l0 > 0.f ? 1.f / l0 : 0.f;
      const float i1 = l1 > 0.f ? 1.f / l1 : 0.f;
      __nv_bfloat16* orow0 = p.out + size_t(s0 + qi0) * p.ldo + size_t(head) * D;
      __nv_bfloat16* orow1 = p.out + size_t(s0 + qi1) * p.ldo + size_t(head) * D;
#pragma unroll
      for (int dn = 0; dn < 2 * KK; ++dn) {
        const int col = dn * 8 + 2 * t4;
        if (qi0 < len) *reinterpret_cast<uint32_t*>(orow0 + col) = pack_bf16(o[dn][0] * i0, o[dn][1] * i0);
        if (qi1 < len) *reinterpret_cast<uint32_t*>(orow1 + col) = pack_bf16(o[dn][2] * i1, o[dn][3] * i1);
      }
    }
    gtile += nkv;
    qphase ^= 1;
  }
}

template <int D>
static int launch_prefill(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                          const PrefillParams& p, int grid, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    HP_CUDA_TRY(cudaFuncSetAttribute(k_prefill_attn<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(PaCfg<D>::SMEM)));
    attr = true;
  }
  k_prefill_attn<D><<<grid, PA_THREADS, PaCfg<D>::SMEM, st>>>(tq, tk, tv, p);
  HP_LAUNCH_CHECK("k_prefill_attn");
  return HP_OK;
}

}  // namespace hp

using namespace hp;

extern "C" int hp_prefill_attn(const void* q, int ldq, const void* k, int ldk, const void* v, int ldv,
                               void* o, int ldo, const int* cu_seqlens, int nseq, int total_tokens, int max_seqlen,
                               int Hq, int Hkv, int d, float scale, int max_ctas, void* stream) {
  HP_CHECK_ARG(q && k && v && o && cu_seqlens, "hp_prefill_attn: null pointer");
  HP_CHECK_ARG(d == 64 || d == 128, "hp_prefill_attn: head_dim must be 64 or 128");
  HP_CHECK_ARG(Hkv >= 1 && Hq % Hkv == 0, "hp_prefill_attn: Hkv must divide Hq");
  HP_CHECK_ARG(nseq >= 1 && max_seqlen >= 1, "hp_prefill_attn: empty batch");
  HP_CHECK_ARG(max_ctas >= 1, "hp_prefill_attn: max_ctas must be >= 1");
  HP_CHECK_ARG(ldo % 2 == 0, "hp_prefill_attn: misaligned output pitch");
  HP_CHECK_ARG(total_tokens >= 1, "hp_prefill_attn: total_tokens must be >= 1");
  const uint64_t rows = uint64_t(total_tokens);  // TMA zero-fills past the last row
  CUtensorMap tq, tk, tv;
  int rc = cached_tmap_bf16(&tq, q, rows, uint64_t(Hq) * d, ldq, 64, 64, true);
  if (rc) return rc;
  rc = cached_tmap_bf16(&tk, k, rows, uint64_t(Hkv) * d, ldk, 64, 64, true);
  if (rc) return rc;
  rc = cached_tmap_bf16(&tv, v, rows, uint64_t(Hkv) * d, ldv, 64, 64, true);
  if (rc) return rc;
  PrefillParams p{};
  p.cu_seqlens = cu_seqlens;
  p.nseq = nseq;
  p.n_qt = (max_seqlen + PA_BQ - 1) / PA_BQ;
  p.Hq = Hq;
  p.Hkv = Hkv;
  p.G = Hq / Hkv;
  p.out = static_cast<__nv_bfloat16*>(o);
  p.ldo = ldo;
  p.scale_log2 = scale * 1.4426950408889634f;
  const int units = nseq * p.n_qt * Hq;
  const int grid = std::min(units, max_ctas);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  return d == 128 ? launch_prefill<128>(tq, tk, tv, p, grid, st) : launch_prefill<64>(tq, tk, tv, p, grid, st);
}
