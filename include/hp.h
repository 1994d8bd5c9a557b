/*
 * hp.h -- C ABI of the B200 co-executed prefill/decode hot path
 * (libb200hot.so, sm_100a only).
 *
 * The reference (smshare, /root/reference/pkg/src/smshare) has no native code:
 * its device boundary is the Python `GroundTruthOracle` (engine.py:159-208),
 * whose `prefill_layer_s(es)` / `decode_step_s(es)` stand in for "one prefill
 * layer on pm SMs" and "one decode step on dm SMs".  This library is what
 * those two calls execute on a B200.  Every entry point below names the
 * reference interface (file:line) whose work it performs.
 *
 * Conventions
 *   - All device memory is owned by the caller (PyTorch); pointers are raw
 *     device addresses, never freed here.  bf16 tensors are row-major.
 *   - Every compute call is asynchronous on `stream` (a cudaStream_t, e.g.
 *     torch.cuda.Stream.cuda_stream or a green-context stream from
 *     hp_partition_stream) and returns 0 or a negative HP_ERR_* code;
 *     hp_last_error() describes the failure.  No CPU fallback exists.
 *   - `max_ctas` is the persistent grid size: the SM count of the partition
 *     the launch is confined to (times resident CTAs per SM).
 */
#ifndef HP_H_
#define HP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HP_ABI_VERSION 1

#define HP_OK 0
#define HP_ERR_INVALID (-1)
#define HP_ERR_CUDA (-2)
#define HP_ERR_UNSUPPORTED (-3)
#define HP_ERR_NO_DEVICE (-4)

/* GEMM epilogues: the fused tails of the reference's kernel groups */
#define HP_EPI_STORE 0 /* qkv projection          (workload.py:164-170) */
#define HP_EPI_RESID 1 /* o_proj / mlp_down + residual (workload.py:191-194, 205-209) */
#define HP_EPI_SILU 2  /* mlp_up_gate, silu(g)*u  (workload.py:198-204) */
#define HP_EPI_PEER 3  /* row-parallel partial scattered to every TP rank (hp_gemm_swap_peer) */
#define HP_MAX_PEERS 8 /* tensor-parallel degree bound of the fused all-reduce */

/* ---------------------------------------------------------------- runtime */
int hp_abi_version(void);
const char* hp_last_error(void);
/* Number of visible CUDA devices (0 on a GPU-less host; never fails). */
int hp_device_count(void);
/* SM count of `device`; the `N` of GpuSpec (perf_model.py:38-57). */
int hp_device_sms(int device, int* sms);

/* ------------------------------------------------------- wave accounting */
/* wave_stats(g, b, n) -- perf_model.py:157-169.  Bit-identical integers and
 * the same IEEE double idle ratio (n - tail) / (n * waves). */
int hp_wave_stats(int64_t g, int64_t b, int64_t n, int64_t* waves, int64_t* tail_sms,
                  double* idle_ratio);

/* ---------------------------------------------------- SM partitions
 * Realises `_request_partition` / `_apply_partitions` (engine.py:440-452):
 * a green-context pair splitting the device into a decode share of
 * `decode_sms` SMs (multiple of 8, CC>=9 rule) and a prefill share holding
 * the remainder.  Each side owns one stream; kernels launched into it run
 * only on that side's SMs.  Switching partitions = launching into another
 * pair's streams (the reference's `reconfig_s`, engine.py:132). */
typedef struct hp_partition hp_partition;
int hp_partition_create(int device, int decode_sms, hp_partition** out);
/* phase: 0 = prefill, 1 = decode. */
int hp_partition_stream(hp_partition* part, int phase, void** stream);
int hp_partition_sms(hp_partition* part, int phase, int* sms);
int hp_partition_destroy(hp_partition* part);

/* ---------------------------------------------------- layer kernels */
/* Pre-attention / pre-MLP RMSNorm (traffic folded into qkv / mlp_up_gate
 * bytes, workload.py:164-168, 200-202): out = x * rsqrt(mean(x^2)+eps) * w. */
int hp_rmsnorm(const void* x, int ldx, const void* weight, void* out, int ldo, int rows, int cols,
               float eps, int max_ctas, void* stream);

/* Weight layout conversion (one-time, at load): row-major W [N, K] ->
 * tiled [N/128][K/128][2][128][64] with the 128B-swizzle chunk permutation,
 * so every [128 x 128] weight tile is one contiguous 32 KB run fetched by a
 * single bulk copy.  N % 128 == 0, K % 128 == 0; `out` holds N*K bf16. */
int hp_tile_weight(const void* w, int ldw, void* out, int N, int K, void* stream);

/* Token-major tcgen05 GEMM (prefill): Y[T,N] = epi(X[T,K] . W[N,K]^T), W
 * tiled by hp_tile_weight (pass ldw = K).
 * SILU: W rows interleaved in blocks of 64 (gate, up), Y has N/2 columns.
 * The qkv / o_proj / mlp_up_gate / mlp_down kernels of layer_kernels
 * (workload.py:162-210) at phase "prefill".  Runs as CTA pairs (2-CTA
 * clusters, tcgen05.mma.cta_group::2 on 256 x 256 tiles) when the planned
 * tile width is 256 and max_ctas >= 2, else as single CTAs (hp_gemm_plan;
 * HP_GEMM_PAIR=0 forces single CTAs for A/B measurement). */
int hp_gemm(const void* X, int ldx, const void* W, int ldw, void* Y, int ldy, const void* R,
            int ldr, int T, int N, int K, int epilogue, int max_ctas, void* stream);
/* The prefill QKV projection with RoPE and the paged K/V write fused into
 * its epilogue (kernel group `qkv` + the `kv_write` bytes of `attn`,
 * workload.py:164-170, 180-182): Y[T, (Hq+2Hkv)d] = X . W^T with q and k heads
 * rotated (as hp_rope_kv_write does) before the bf16 store, and k / v heads
 * also written to kcache / vcache at slot_mapping[t].  Replaces hp_gemm
 * (EPI_STORE) + hp_rope_kv_write on the prefill path. */
int hp_gemm_qkv_rope(const void* X, int ldx, const void* W, int ldw, void* Y, int ldy, int T, int Hq,
                     int Hkv, int d, int K, const int* positions, const float* cos_sin,
                     const int* slot_mapping, void* kcache, void* vcache, int page, int max_ctas,
                     void* stream);
/* Same, recording per-CTA {smid, start_ns, end_ns} into cta_times[grid][3]
 * (config-3 wave measurement: measured idle = 1 - sum(busy) / (n * span),
 * against wave_stats(hp_gemm_tiles(T, N), 1, n), perf_model.py:157-169). */
int hp_gemm_traced(const void* X, int ldx, const void* W, int ldw, void* Y, int ldy, const void* R,
                   int ldr, int T, int N, int K, int epilogue, int max_ctas, uint64_t* cta_times,
                   void* stream);
/* Output tiles (persistent-grid work units) of hp_gemm for T tokens, N
 * features at the 256-wide tile. */
int hp_gemm_tiles(int T, int N);
/* The tiling hp_gemm picks for a `max_ctas`-SM partition: tile width (128
 * or 256: fewer wave-quantised column-rounds, wave_stats perf_model.py:
 * 157-169), tile count, and CTAs per tile (2 = CTA-pair 256 x 256 tiles on
 * tcgen05.mma.cta_group::2; the persistent grid then has max_ctas / 2 units
 * of work-in-flight, i.e. waves = wave_stats(tiles, 1, max_ctas / 2)).
 * tail_tiles: tiles the stream-K tail (hp_set_gemm_tail) splits over every
 * pair instead of running them as the last rounds (0: plain rounds). */
int hp_gemm_plan(int T, int N, int K, int max_ctas, int* bn, int* tiles, int* ctas_per_tile,
                 int* tail_tiles);

/* Swap-AB stream-K tcgen05 GEMM for decode (T <= 256 tokens): same math as
 * hp_gemm; W streams through UMMA-M and the (tile, k-block) space is split
 * evenly over `max_ctas` CTAs.  workspace: fp32, hp_gemm_swap_ws_bytes()
 * bytes (contents irrelevant); counters: int [N/128 * ceil(T/BN)], zero
 * before the first call (the kernel leaves them zero).  layer_kernels phase
 * "decode" (workload.py:153-210). */
size_t hp_gemm_swap_ws_bytes(int T, int N, int K, int max_ctas);
int hp_gemm_swap(const void* X, int ldx, const void* W, int ldw, void* Y, int ldy, const void* R,
                 int ldr, int T, int N, int K, int epilogue, void* workspace, size_t ws_bytes,
                 int* counters, int n_counters, int max_ctas, void* stream);

/* Decode QKV projection with RoPE and the paged K/V write fused into the
 * swap-AB GEMM's epilogue: hp_gemm_swap (epilogue STORE) followed by
 * hp_rope_kv_write, as one launch with the same bits (workload.py:164-170;
 * replaces the GEMM + rope pair of the decode step, engine.py:676).
 * N = (Hq + 2 Hkv) * d; positions / slot_mapping / caches as hp_rope_kv_write,
 * workspace / counters as hp_gemm_swap. */
int hp_gemm_swap_qkv_rope(const void* X, int ldx, const void* W, int ldw, void* Y, int ldy, int T, int Hq,
                          int Hkv, int d, int K, const int* positions, const float* cos_sin,
                          const int* slot_mapping, void* kcache, void* vcache, int page, void* workspace,
                          size_t ws_bytes, int* counters, int n_counters, int max_ctas, void* stream);

/* Fused row-parallel GEMM + all-reduce for tensor-parallel decode (config 5,
 * SURVEY.md §8(f)#4; replaces the NCCL all-reduce after o_proj / mlp_down of
 * a Megatron row-parallel layer).  Symmetric buffers: every
 * rank r owns recv_r = bf16 [2][world][T_max][N] and flags_r = int
 * [2][world][tiles_max] (tiles = hp_peer_tiles(T, N); flags zero at
 * allocation) and maps every peer's pair (hp_ipc_*).  Call e (epoch e >= 1,
 * +1 per call, all ranks in step) uses half (e & 1) of each buffer, i.e.
 * base + (e & 1) * {recv,flags}_half_elems:
 *   hp_gemm_swap_peer: the swap-AB GEMM's epilogue writes this rank's partial
 *     tile straight into slot `rank` of every peer's recv over NVLink, then
 *     raises flags_q[rank][tile] = e (system-scope release) -- the transfer of
 *     tile i overlaps the MMA of tile i+1;
 *   hp_peer_reduce: per output tile, wait for every rank's flag >= e and
 *     write out = sum_r recv[r] + resid (fp32 sum, bf16 out, rank order).
 * peer_recv / peer_flags: the `world` base pointers, indexed by rank.  Epochs
 * come from the host (`epoch`) or, with epoch_dev != NULL, from the device:
 * e = *epoch_dev + 1, and the reduce's last block advances *epoch_dev (`done`:
 * an int that is zero before the first call) -- the form a CUDA graph can
 * replay.  Double buffering makes back-to-back calls safe: a rank can reach
 * epoch e + 2 only after every rank's partial for e + 1, i.e. after they all
 * left epoch e's reduce. */
int hp_peer_tiles(int T, int N);
int hp_gemm_swap_peer(const void* X, int ldx, const void* W, int ldw, int T, int N, int K,
                      void* const* peer_recv, size_t recv_half_elems, int* const* peer_flags,
                      size_t flags_half_elems, int world, int rank, int epoch, const int* epoch_dev,
                      int two_shot, void* workspace, size_t ws_bytes, int* counters, int n_counters,
                      int max_ctas, void* stream);
int hp_peer_reduce(const void* recv, size_t recv_half_elems, const int* flags, size_t flags_half_elems,
                   int world, int T, int N, int epoch, int* epoch_dev, int* done, const void* resid,
                   int ldr, void* out, int ldo, void* stream);
/* Two-shot form (two_shot = 1 in hp_gemm_swap_peer): feature tile mt belongs
 * to rank mt % world and the GEMM sends it only there, (world-1)/world of
 * the message per rank instead of (world-1) x.  hp_peer_rs (owner: wait for
 * the tile's partials, sum + resid, broadcast the bf16 result into every
 * rank's gather buffer gather_r = bf16 [2][T_max][N], raise gflags_r =
 * int [2][ceil(T_max/16)][N/128] on every rank), then hp_peer_ag (every
 * rank: wait for each (16-row block, feature tile) flag, copy to out; with
 * epoch_dev it advances the device epoch).  Bytes moved per rank over
 * NVLink: 2 (world-1)/world T N 2 -- the bandwidth-optimal all-reduce for
 * large decode batches; one-shot has one fewer hop for small ones. */
int hp_peer_rs(const void* recv, size_t recv_half_elems, const int* flags, size_t flags_half_elems,
               void* const* peer_gather, size_t gather_half_elems, int* const* peer_gflags,
               size_t gflags_half_elems, int world, int rank, int T, int N, int epoch, const int* epoch_dev,
               const void* resid, int ldr, void* stream);
int hp_peer_ag(const void* gather, size_t gather_half_elems, const int* gflags, size_t gflags_half_elems,
               int T, int N, int epoch, int* epoch_dev, int* done, void* out, int ldo, void* stream);
/* CUDA IPC for the symmetric buffers: export the handle (HP_IPC_HANDLE_BYTES
 * opaque bytes) of the allocation block holding dev_ptr plus dev_ptr's
 * offset in it; a peer maps the block (hp_ipc_open -> base; its pointer is
 * base + offset) and unmaps it with hp_ipc_close(base). */
#define HP_IPC_HANDLE_BYTES 64
int hp_ipc_handle(void* dev_ptr, void* handle_out, size_t* offset_out);
int hp_ipc_open(const void* handle, void** base_out);
int hp_ipc_close(void* base);

/* RoPE on q,k in the fused qkv buffer [T, (Hq+2Hkv)*d] (in place) and the
 * paged KV-cache write of k,v (the `kv_write` bytes of the attention kernel,
 * workload.py:180-182).  cos_sin: fp32 [max_pos, d] = [cos(d/2) | sin(d/2)].
 * slot_mapping[t] = block * page + offset; kcache/vcache: [blocks, Hkv, page, d]
 * logical, stored per (block, kv head) as [page/64][d/64][64 tokens][64] bf16
 * with the 16-byte chunks of token row r permuted by (r & 7) (128B swizzle),
 * so every 64-token K or V tile is one contiguous 64*d*2-byte run.
 * page % 64 == 0, d % 64 == 0. */
int hp_rope_kv_write(void* qkv, int ldqkv, int T, int Hq, int Hkv, int d, const int* positions,
                     const float* cos_sin, const int* slot_mapping, void* kcache, void* vcache,
                     int page, int max_ctas, void* stream);

/* Causal GQA prefill attention over the new span (workload.py:176-183 with
 * prior_lens = 0): O[T, Hq*d] = softmax(Q K^T * scale, causal) V.
 * cu_seqlens: int [nseq+1] token offsets of the packed sequences (host-side
 * total_tokens = cu_seqlens[nseq] bounds the TMA views). */
int hp_prefill_attn(const void* q, int ldq, const void* k, int ldk, const void* v, int ldv,
                    void* o, int ldo, const int* cu_seqlens, int nseq, int total_tokens,
                    int max_seqlen, int Hq, int Hkv, int d, float scale, int max_ctas,
                    void* stream);

/* Kernel timeline traces.  kind 0: k_fa2 CTA 0 softmax/MMA wait stamps
 * (clock64, int64 [18][256]: rows 0-11 per KV step, 12-17 per unit); kind 1: k_gemm_swap_sk per-CTA globaltimer
 * stamps (uint64 [grid][10]: entry, prologue done, producer done, MMA done,
 * epilogue done, exit; then, for the CTA's last split tile: partial written,
 * arrival counted, partials summed (last arriver), tile emitted); kind 2 (one-shot, SM-idle measurement of config 2/3):
 * the NEXT hp_gemm / hp_gemm_qkv_rope / hp_prefill_attn(_paged) launch on
 * this thread writes per-CTA {smid, start_ns, end_ns} (uint64 [grid][3]) and
 * disarms it.  NULL disables. */
int hp_set_trace(int kind, void* buf);

/* Stream-K tail of the prefill CTA-pair GEMM (hp_gemm, hp_gemm_qkv_rope):
 * mode 1 splits the last full round plus the partial one (or every tile,
 * when there are fewer tiles than pairs) into equal k-block ranges, one per
 * pair, with a deterministic fp32 fix-up in the finishing pair; 0 runs plain
 * persistent rounds (the grid wave_stats describes, perf_model.py:157-169);
 * -1 restores the default (on unless HP_GEMM_TAIL=0).  Per process.  The
 * fix-up workspace is allocated per stream on first use (~21 MB), which
 * must not happen inside a stream capture (the tail is then skipped). */
int hp_set_gemm_tail(int mode);
/* Allocate `stream`'s stream-K fix-up workspace now (setup time, outside
 * any capture) instead of on its first tail GEMM. */
int hp_gemm_tail_reserve(void* stream);

/* Prefix-aware (chunked) prefill attention over the paged cache
 * (workload.py:176-183 with prior_lens > 0; the attention of a hybrid batch,
 * hybrid_kernels workload.py:213-257, as issued by _ChunkedSim engine.py:
 * 741-800 through GroundTruthOracle.hybrid_iteration_s engine.py:200-208).
 * Sequence s has cu_seqlens[s+1]-cu_seqlens[s] new tokens (rows of q) at
 * positions prior_lens[s].. ; their K/V must already be in the cache
 * (hp_rope_kv_write).  Query i attends cache positions [0, prior_lens[s]+i].
 * Caches as for hp_rope_kv_write; block_table: int [nseq, max_pages].
 * Cache blocks must hold finite values (zero-initialised pools). */
int hp_prefill_attn_paged(const void* q, int ldq, const void* kcache, const void* vcache,
                          const int* block_table, int max_pages, const int* cu_seqlens,
                          const int* prior_lens, int nseq, int total_tokens, int max_seqlen,
                          void* o, int ldo, int Hq, int Hkv, int d, int page, int num_blocks,
                          float scale, int max_ctas, void* stream);

/* Paged decode attention (workload.py:184-188): one query token per
 * sequence over ctx_lens[b] cached positions.  q: [B, Hq*d]; out: [B, Hq*d];
 * block_table: int [B, max_pages]; workspace: fp32, hp_decode_attn_ws_bytes.
 * GQA group Hq/Hkv <= 8, or a multiple of 8 (run as Hq/Hkv/8 head blocks).
 * Precondition: 1 <= ctx_lens[b] <= max_pages * page (the row's pages must
 * hold the context); the kernels clamp a longer ctx_lens[b] to that bound
 * rather than read past the block-table row or the split workspace. */
size_t hp_decode_attn_ws_bytes(int B, int Hq, int d, int max_splits);
/* Kernel launches hp_decode_attn issues for this shape (2 when the context
 * is split and a log-sum-exp combine follows; bounded by the workspace). */
int hp_decode_attn_launches(int B, int Hq, int Hkv, int d, int max_pages, int page, int max_ctas);
int hp_decode_attn(const void* q, int ldq, const void* kcache, const void* vcache,
                   const int* block_table, int max_pages, const int* ctx_lens, void* out, int ldo,
                   int B, int Hq, int Hkv, int d, int page, int num_blocks, float scale,
                   void* workspace, size_t ws_bytes, int max_ctas, void* stream);

/* Strided row copy (rows x row_bytes, 16-byte aligned), grid <= 4 x max_ctas
 * CTAs.  Either side may be pinned host memory (UVA-mapped): used for a
 * decode step's per-step input/output (B x hidden) so it crosses PCIe on the
 * decode partition's SMs inside the step's CUDA graph rather than on a copy
 * engine shared with the prefill side's bulk transfers. */
int hp_copy_rows(const void* src, long lds_bytes, void* dst, long ldd_bytes, int rows, int row_bytes,
                 int max_ctas, void* stream);

/* ---------------------------------------------------- instrumentation */
/* Memory-bandwidth probe behind the SRM memory term D_p = D min(1, p/n_d)
 * (perf_model.py:172-180): stream `bytes` from `src` with `ctas` CTAs.
 * method 0 = 128-bit loads, 1 = TMA bulk copies (bytes % 32 KB == 0).
 * `out` receives a dummy reduction. */
int hp_membw(const void* src, size_t bytes, int ctas, int method, float* out, void* stream);
/* Same, through 2-D TMA boxes {64 bf16, box_rows} of a [rows, cols] bf16
 * matrix (the GEMM weight-stream access shape). */
int hp_membw2d(const void* src, int rows, int cols, int box_rows, int ctas, float* out, void* stream);
/* Producer/consumer copy pipeline (a GEMM mainloop without the MMA):
 * `producers` issuing warps, one in-order consumer, chunk_kb KB stages. */
int hp_membw_pipe(const void* src, size_t bytes, int ctas, int chunk_kb, int producers, float* out,
                  void* stream);
/* tcgen05.mma issue/completion rate: n MMAs (M=128, N=bn, K=16, smem
 * operands) over `chains` accumulators; out[cta] = {issue cycles, done cycles}. */
int hp_umma_rate(int n, int bn, int chains, int ctas, long long* out, void* stream);
/* Pair MMA rate: `pairs` 2-CTA clusters issue n tcgen05.mma.cta_group::2
 * (M=256, N=bn, K=16); out[cta] = issue cycles, out[grid + cta] = done cycles. */
int hp_umma2_rate(int n, int bn, int pairs, long long* out, void* stream);

/* Register-direct streaming: `threads` per CTA, `unroll` (2/4/8/16) 128-bit
 * loads per lane in flight twice over, noalloc = L1::no_allocate. */
int hp_membw_ldg(const void* src, size_t bytes, int ctas, int threads, int unroll, int noalloc,
                 float* out, void* stream);
/* Both streaming paths at once: one warp's bulk-copy ring takes bulk_frac/256
 * of each CTA's range, `ldg_warps` warps stream the rest with 128-bit loads. */
int hp_membw_mix(const void* src, size_t bytes, int ctas, int ldg_warps, int bulk_frac, float* out,
                 void* stream);
/* Register-direct streaming behind an L2 prefetch: per-CTA contiguous
 * superchunks of (threads/32) x unroll x 512 bytes; the superchunk `dist`
 * ahead is prefetched into L2 (cp.async.bulk.prefetch.L2), dist 0 = none. */
int hp_membw_pfldg(const void* src, size_t bytes, int ctas, int threads, int unroll, int dist,
                   float* out, void* stream);
/* Staged reader vs register-direct on one SM: bulk_frac/256 of each CTA's
 * 16 KB chunks go through a bulk-copy ring read back by `readers` warps
 * (read_mode 0: released unread), the rest through `ldg_warps` LDG warps. */
int hp_membw_stage(const void* src, size_t bytes, int ctas, int readers, int ldg_warps, int bulk_frac,
                   int read_mode, float* out, void* stream);
/* mma.sync.m16n8k16 (bf16) rate: `chains` independent accumulators per warp,
 * n rounds; out[cta] = cycles. */
int hp_hmma_rate(int n, int chains, int ctas, int threads, long long* out, void* stream);

/* Per-CTA probe: out[i] = {smid, start_ns, end_ns} for `ctas` CTAs spinning
 * `spin_ns` each -- partition confinement (%smid) and measured idle. */
int hp_probe(int ctas, int threads, int64_t spin_ns, uint64_t* out, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* HP_H_ */
