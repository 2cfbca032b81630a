/*
 * vqb.h — C ABI of the B200-native fused vector-quantization kernels.
 *
 * This is the drop-in boundary for the reference's fused-kernel operator API
 * (vqforge, a pure-Python package with no FFI of its own). Each entry point
 * replaces one reference call; the Python mirror in
 * paper_2503_02236_b200/_native.py binds them with ctypes, and INTEGRATION.md
 * shows the binding a vqforge maintainer would add.
 *
 *   vqb_dequant      <- vqforge.codec.dequantize                 (pkg/src/vqforge/codec.py:391-408)
 *   vqb_gemv         <- SimMachine.run_fused_kernel, ComputeOp.gemv (pkg/src/vqforge/sim.py:297-316,
 *                       executed by _matmul/_mm_block, sim.py:697-775; op at dataflow.py:73-75)
 *   vqb_gemm         <- SimMachine.run_fused_kernel, ComputeOp.gemm (sim.py:297-316, dataflow.py:68-71)
 *   vqb_attn_decode  <- SimMachine.run_fused_kernel, ComputeOp.attention_decode
 *                       (sim.py:491-693, dataflow.py:77-82)
 *   vqb_repack       <- QuantizedTensor.packed_codes / bitpack.unpack_indices
 *                       (codec.py:215-218, bitpack.py:31-43): packed stream -> kernel layout
 *   vqb_query_usage  <- sim.KERNEL_USAGE (sim.py:53-57): real per-kernel resource usage
 *                       feeding compute_slack (cacheplan.py:27-62)
 *   vqb_last_error   <- the message of the raised vqforge.errors exception (errors.py:4-25)
 *   vqb_cq_quantize  <- vqforge.codec.quantize / _nearest (codec.py:239-253, 367-389) for KV rows:
 *                       online nearest-centroid quantization of new tokens into a KV cache
 *   vqb_attn_decode_len, vqb_rmsnorm, vqb_qkv_rope, vqb_qkv_rope_append, vqb_silu_mul, vqb_add_len,
 *   vqb_sample,
 *   vqb_take_device_error
 *                    <- the end-to-end decode step around the fused ops (
 *                       no vqforge counterpart: the reference stops at single fused kernels)
 *
 * Conventions
 *  - Plain pointers and sizes only. Every pointer named d_* is DEVICE memory owned
 *    by the caller; the library never allocates or frees caller memory.
 *  - `stream` is a cudaStream_t passed as void*; every call is stream-ordered and
 *    asynchronous (no host synchronisation) and reentrant.
 *  - Return 0 on success, or a negative VQB_E* code whose class maps 1:1 onto the
 *    reference exception hierarchy; vqb_last_error() then holds the message
 *    (thread-local), keeping the reference's wording (e.g. "code out of range").
 *  - Weights follow the reference layout: W is (M = input/reduction, N = output)
 *    and y = x @ W (sim.py:136-144). Sub-vectors run along the last axis
 *    (codec.py:229-236): along N for weights, along C for the KV cache.
 */
#ifndef VQB_H_
#define VQB_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VQB_ABI_VERSION 2

/* ---- status codes (errors.py:4-25) ---- */
#define VQB_OK 0
#define VQB_ESHAPE -1     /* ShapeError */
#define VQB_ECONFIG -2    /* ConfigError */
#define VQB_ECODERANGE -3 /* CodeRangeError */
#define VQB_ECAPACITY -4  /* CapacityError */
#define VQB_EMAPPING -5   /* MappingError */
#define VQB_ECUDA -10     /* CUDA runtime failure (RuntimeError in Python) */

/* ---- element types ---- */
#define VQB_F32 0
#define VQB_F16 1
#define VQB_BF16 2

/* ---- codebook sharing (codec.py:23-57) ---- */
#define VQB_SHARE_WHOLE 0
#define VQB_SHARE_TILE 1
#define VQB_SHARE_CHANNEL_GROUP 2

/* ---- code-stream layouts ----
 * PACKED   : the reference stream, level-major, `log2_entries` bits per code,
 *            LSB-first, byte padded at the end only (bitpack.py:13-28). Any width 1..16.
 * GEMV_IL  : weight codes interleaved for 128-bit lane loads, per level
 *            [M/RPL][G][RPL] with G = N/v sub-vectors per row and RPL = 16/code_bytes
 *            rows per 16-byte load (8 rows of u16 codes, 16 rows of u8 codes).
 *            Levels are stored one after another (level-major, like the reference).
 * KV_IL    : KV-cache codes interleaved for the decode-attention kernel (u8 codes,
 *            G = C/v in {32, 64}), per level and per (b, h) row block of T tokens,
 *            per 32-token batch: [G/16 words][32 lanes][16 bytes]. Lane (h, ll) =
 *            (lane / 8, lane % 8) owns groups ll + 8*(j ^ h), j < G/8, and stores
 *            token 8h + (i ^ ll) at slot i (0..7), byte i*(G/8) + j.
 * PLAIN    : the reference `codes` array (R, S) level-major in the narrowest unsigned
 *            type: u8 when log2_entries <= 8, else u16.
 */
#define VQB_LAYOUT_PACKED 0
#define VQB_LAYOUT_GEMV_IL 1
#define VQB_LAYOUT_KV_IL 2
#define VQB_LAYOUT_PLAIN 3

/* One quantized tensor as the kernels see it (QuantizedTensor, codec.py:180-226). */
typedef struct VqbTensor {
  int32_t vector_size;  /* v in {2,4,8,16} */
  int32_t log2_entries; /* b in [1,16]; K = 2^b entries per codebook */
  int32_t residuals;    /* R >= 1 */
  int32_t sharing;      /* VQB_SHARE_* */
  int32_t tile_rows, tile_cols, group_width;
  int32_t ndim;         /* 1..4 */
  int64_t dims[4];      /* tensor shape, last axis split into sub-vectors */
  int32_t n_regions;    /* regions per level (region_layout, codec.py:135-177) */
  int32_t layout;       /* VQB_LAYOUT_* of d_codes */
  const void* d_codes;  /* code stream in `layout` */
  int64_t codes_bytes;  /* allocated bytes behind d_codes (bounds check) */
  int32_t codebook_dtype;   /* VQB_F32 / VQB_F16 / VQB_BF16 */
  const void* d_codebooks;  /* (R*n_regions, K, v) contiguous, level-major (codec.py:208-209) */
  int32_t max_code;         /* largest code in the stream if known (from the upload-time range
                               check / profiling), else -1; lets a kernel drop its global tier */
  const void* d_codebooks_t;  /* optional (may be NULL): channel-group books of a (B, H, T, C) KV
                               tensor re-laid per head as [H][K][C/v][v] (same dtype), so the
                               attention kernel pulls a head's books with one bulk copy each */
} VqbTensor;

/* Launch knobs from the planner (FusedPlans, sim.py:229-236). Zero-initialise
 * for defaults. */
typedef struct VqbLaunch {
  int32_t n_reg;        /* CachePlan.n_reg: register-resident entries (reserved, 0 on B200) */
  int32_t n_shared;     /* CachePlan.n_shared: entries resident in shared memory; 0 = planner default */
  int32_t split_axis;   /* 0 none, 'M', 'R', 'C', 'T' as char codes (DataflowPlan.split_axis) */
  int32_t split_factor; /* DataflowPlan.split_factor; 0 = kernel default */
  int32_t fusion_level; /* 0 register, 1 shared (informational on B200) */
  int32_t grid_limit;   /* max CTAs (0 = SM count x occupancy) */
  int32_t flags;        /* VQB_FLAG_* */
} VqbLaunch;

#define VQB_FLAG_FORCE_GENERIC 1 /* use the generic (any-config) kernel */
#define VQB_FLAG_NO_SHARED 2     /* no shared-memory tier: every lookup from global/L2 ("GC") */
#define VQB_FLAG_NO_PDL 4        /* launch without programmatic dependent launch */
#define VQB_FLAG_EXACT_ACCUM 8   /* GEMV: fp32 accumulation of every product (mixed-precision
                                    FMA, quarter rate) instead of 8-row fp16x2 windows */
#define VQB_FLAG_NO_MMA 16       /* GEMV batch 4-8: CUDA-core FMAs instead of the tensor-core
                                    (mma.sync) inner product */
#define VQB_FLAG_NO_PAIR 128     /* GEMM: the one-CTA tcgen05 kernel instead of the CTA-pair
                                    (cta_group::2) kernel at prefill sizes */
#define VQB_FLAG_PAIR_N128 256   /* GEMM: CTA-pair kernel with 256 x 128 tiles (N % 128) */
#define VQB_FLAG_GEMV_TC 2048    /* GEMV: the tcgen05 decode GEMV (batch as the UMMA N) also below its
                                    default batch range */
#define VQB_FLAG_NO_GEMV_TC 4096 /* GEMV: never the tcgen05 decode GEMV (mma.sync / CUDA-core kernels) */
#define VQB_FLAG_NO_COLSPLIT 8192 /* GEMV batch 1/2/4: the stream-K kernel (split over M) instead of
                                     the column-split kernel for N = 16 x 256-column outputs */
#define VQB_FLAG_GEMM_FUSED 512  /* GEMM: keep the fused (dequantise-in-the-producers) kernels at
                                    prefill sizes where the two-phase path is the default */
#define VQB_FLAG_GEMM_TWO_PHASE 1024 /* GEMM (rows > 256, v = 8, N % 256 == 0): dequantise W to an fp16
                                    scratch in the workspace, then the dense CTA-pair tcgen05 GEMM
                                    (default for two-level / AQLM codes at rows >= 512) */
#define VQB_FLAG_COOPERATIVE 64  /* GEMV / attention: cooperative launch. The split reduction's
                                    finisher CTAs wait for partials of later CTAs, which needs
                                    the whole (<= 1 CTA per SM) grid resident; the default launch
                                    relies on that (grid <= SMs, occupancy checked) and on any
                                    concurrent kernel finishing. With this flag the driver
                                    guarantees co-residency (or the launch fails loudly) — for
                                    streams that overlap with kernels waiting on this one. */

/* Kernel resource usage (KernelUsage, gpumodel.py:30-36) measured with
 * cudaFuncGetAttributes on the loaded cubin. */
typedef struct VqbUsage {
  int32_t shared_bytes;      /* static + dynamic shared memory per CTA at the default plan */
  int32_t regs_per_thread;
  int32_t threads_per_block;
  int32_t max_blocks_per_sm; /* occupancy at that usage */
  int32_t sm_count;
} VqbUsage;

#define VQB_KERNEL_DEQUANT 0
#define VQB_KERNEL_GEMV 1
#define VQB_KERNEL_GEMM 2
#define VQB_KERNEL_ATTN 3

int vqb_abi_version(void);
const char* vqb_last_error(void);
/* Name of the last kernel this thread launched ("gemv_fast", "attn_cq", ...):
 * lets tests and the benchmark prove which path ran. */
const char* vqb_last_kernel(void);
/* {grid CTAs, threads per CTA, shared-tier entries, register-tier entries} of this
 * thread's last fused launch: shows which plan the kernel actually ran with. */
int vqb_last_launch(int32_t* out4);

/* Reconstruct the dense tensor (dequantize, codec.py:391-408): fp32 output is
 * bit-exact with the reference (accumulation from +0.0f in level order);
 * fp16/bf16 outputs are RN-even casts of that fp32 value. */
int vqb_dequant(const VqbTensor* t, void* d_out, int32_t out_dtype, void* stream);

/* Workspace bytes a fused call needs. The first VQB_WS_COUNTER_BYTES of every
 * workspace are the self-resetting head: split-arrival counters (attention) and
 * tagged split partials (GEMV). Zero it once when the workspace is allocated;
 * kernels restore it to zero after use and never leave anything else there. */
#define VQB_WS_COUNTER_BYTES 16777216
/* Workspace bytes a fused call needs (split partials + arrival counters).
 * kind = VQB_KERNEL_*; rows = batch rows (GEMV/GEMM) or B*H (attention). */
int64_t vqb_workspace_bytes(int32_t kind, const VqbTensor* t, int64_t rows,
                            const VqbLaunch* launch);

/* y(rows, N) = x(rows, M) @ dequant(W)(M, N). rows 1, 2, 4, 8 and 16 take the decode
 * kernel (CUDA cores at 1-2, mma.sync at 4-16); other row counts the generic kernel,
 * larger batches should use vqb_gemm. The workspace must be zeroed
 * once before first use (counters self-reset afterwards). */
int vqb_gemv(const VqbTensor* w, const void* d_x, int32_t x_dtype, int32_t rows,
             void* d_y, int32_t y_dtype, const VqbLaunch* launch, void* d_ws,
             size_t ws_bytes, void* stream);

/* Grouped decode GEMV: n independent problems y_i(rows, N_i) = x_i(rows, M_i) @
 * dequant(W_i), all of one VQ configuration (v = 8, one level, whole-tensor
 * books with every code < 256 resident in shared memory, GEMV_IL codes, fp16),
 * as ONE persistent stream-K launch over the units of every problem: a step's
 * independent linears pay one prologue / tail instead of one per linear. w points
 * to n consecutive VqbTensor; n <= 192. No vqforge counterpart (the reference runs
 * one fused kernel per call, sim.py:297-316); per problem the result equals
 * vqb_gemv's. */
int vqb_gemv_grouped(const VqbTensor* w, int32_t n, const void* const* d_xs, int32_t x_dtype, int32_t rows,
                     void* const* d_ys, int32_t y_dtype, const VqbLaunch* launch, void* d_ws,
                     size_t ws_bytes, void* stream);

/* Prefill GEMM: y(rows, N) = x(rows, M) @ dequant(W). Dequantised W tiles are
 * written to shared memory in the UMMA canonical layout and consumed by
 * tcgen05.mma with the accumulator in TMEM. x must be fp16 or bf16 matching the
 * codebook dtype, M % 64 == 0, N % 128 == 0 (otherwise VQB_ESHAPE). */
int vqb_gemm(const VqbTensor* w, const void* d_x, int32_t x_dtype, int32_t rows,
             void* d_y, int32_t y_dtype, const VqbLaunch* launch, void* d_ws,
             size_t ws_bytes, void* stream);

/* Decode attention over a VQ KV cache: out(B,H,C) = softmax(q.K^T / sqrt(C)) V
 * with K, V (B,H,T,C) quantized tensors (sim.py:491-521, oracle sim.py:145-155). */
int vqb_attn_decode(const VqbTensor* k, const VqbTensor* v, const void* d_q,
                    int32_t q_dtype, int32_t B, int32_t H, int32_t T, int32_t C,
                    void* d_out, int32_t out_dtype, const VqbLaunch* launch,
                    void* d_ws, size_t ws_bytes, void* stream);

/* Decode attention over the first T tokens of a KV cache whose capacity is dims[2]
 * (a partial last 32-token batch is masked). If d_len is non-NULL the valid length
 * is read on the device at launch (d_len[0], clamped to the capacity), so a decode
 * step can replay as a CUDA graph while the cache grows; T is then ignored except
 * for validation (1 <= T <= capacity). */
int vqb_attn_decode_len(const VqbTensor* k, const VqbTensor* v, const void* d_q, int32_t q_dtype, int32_t B,
                        int32_t H, int32_t T, int32_t C, const int32_t* d_len, void* d_out, int32_t out_dtype,
                        const VqbLaunch* launch, void* d_ws, size_t ws_bytes, void* stream);

/* Fused decode front end + attention: d_qkv is the fused qkv projection output
 * (B, 3*H*C) fp16 of the new token; the kernel ropes q, and the CTA covering position
 * d_len[0]-1 of each (b, h) ropes k and quantizes the new K and V rows (as
 * vqb_qkv_rope_append) against the books it holds in shared memory, writes the codes
 * into the caches and attends over the first d_len[0] tokens (as vqb_attn_decode_len).
 * CQ-4 configuration (v = 2, C = 128, KV_IL caches, fp16 books); one launch instead of
 * two, and the books are read once per step. */
int vqb_attn_decode_append(const VqbTensor* k_cache, const VqbTensor* v_cache, const void* d_qkv, int32_t B,
                           int32_t H, int32_t C, const int32_t* d_len, float theta, void* d_out, int32_t out_dtype,
                           const VqbLaunch* launch, void* d_ws, size_t ws_bytes, void* stream);

/* Online KV quantization (codec.py:367-389): nearest centroid (float64 distance,
 * lowest index on ties) of n_tok new rows per (b, h) into the (B, H, T_cap, C) code
 * stream of t (KV_IL or PLAIN layout, fp16 codebooks, any R). Row (b, h, j) of the
 * input is at d_x + b*xs_b + h*xs_h + j*xs_t elements (channels contiguous, fp16 or
 * fp32). The rows land at tokens [tok0, tok0 + n_tok), or, if d_len is non-NULL, at
 * [d_len[0] - n_tok, d_len[0]) read on the device. */
int vqb_cq_quantize(const VqbTensor* t, const void* d_x, int32_t x_dtype, int64_t xs_b, int64_t xs_h,
                    int64_t xs_t, int32_t n_tok, int32_t tok0, const int32_t* d_len, void* stream);

/* Llama decode glue (fp16): h = x + residual (residual updated; x may be NULL),
 * out = weight * rmsnorm(h) with fp32 statistics. */
int vqb_rmsnorm(const void* d_x, void* d_residual, const void* d_weight, void* d_out, int32_t rows,
                int32_t dim, float eps, void* stream);
/* RoPE (rotate-half) at position d_len[0]-1 on the q and k thirds of the fused qkv
 * output (B, 3*H*C): roped q -> d_q_out (B, H, C), k roped in place. */
int vqb_qkv_rope(void* d_qkv, void* d_q_out, int32_t B, int32_t H, int32_t C, const int32_t* d_len, float theta,
                 void* stream);
/* Fused decode front end: vqb_qkv_rope, then online quantization (as vqb_cq_quantize)
 * of the roped k and the v rows into k_cache / v_cache at position d_len[0]-1. */
int vqb_qkv_rope_append(const void* d_qkv, void* d_q_out, const VqbTensor* k_cache, const VqbTensor* v_cache,
                        int32_t B, int32_t H, int32_t C, const int32_t* d_len, float theta, void* stream);
/* out (rows, F) = silu(gate) * up for a fused [gate | up] (rows, 2F) input. */
int vqb_silu_mul(const void* d_gate_up, void* d_out, int32_t rows, int32_t ffn, void* stream);
/* Next tokens of a decode step: d_tokens[b] (int64) drawn from softmax(logits[b] / T)
 * restricted to the logits >= the top_k-th largest (top_k 0 = all), then to the nucleus
 * (the largest threshold whose kept probability mass is >= top_p; 1 = off; ties at the
 * threshold kept), by the Gumbel-max trick with a counter-based hash of
 * (seed, *d_step, b, i) as the noise (d_step may be NULL = step 0; pass the decode length
 * so graph replays draw fresh noise); temperature 0 = greedy argmax. Ties resolve to the
 * lowest index. logits (B, vocab) fp16 or fp32. */
int vqb_sample(const void* d_logits, int32_t logits_dtype, int32_t B, int32_t vocab, float temperature,
               int32_t top_k, float top_p, uint64_t seed, const int32_t* d_step, int64_t* d_tokens, void* stream);
/* d_len[0] += delta on the stream (advances a graph-replayed decode loop). */
int vqb_add_len(int32_t* d_len, int32_t delta, void* stream);
/* Read and clear the device error word (synchronises the device): bit 0 = a KV
 * append (vqb_cq_quantize / vqb_qkv_rope_append with a device length) found its
 * write position outside [0, capacity) and skipped the write. */
int vqb_take_device_error(int32_t* out);

/* Decode GEMV with its input transform fused into the prologue (batch 1; the
 * QuiP#-style v = 8 whole-tensor configurations with every code < 256): each CTA
 * builds the transformed activation row in shared memory, so the standalone
 * RMSNorm / SiLU launch before the linear disappears. Same arithmetic as
 * vqb_rmsnorm / vqb_silu_mul (bit-identical results).
 *  VQB_XF_RMSNORM : h = res_in + x (x may be NULL), res_out = h (res_out may be NULL;
 *                   must not alias res_in), y = (weight * rmsnorm(h, eps)) @ dequant(W)
 *  VQB_XF_SILU_MUL: x = [gate | up] (2M halves), y = (silu(gate) * up) @ dequant(W) */
#define VQB_XF_RMSNORM 1
#define VQB_XF_SILU_MUL 2
#define VQB_XF_SWIGLU_OUT 4 /* or-ed into mode: W's 256-column blocks hold [gate 128 | up 128] (the
                               fused gate_up projection interleaved per 128 columns); the epilogue
                               writes y = silu(gate) * up, N/2 fp16 columns (the silu_mul arithmetic) */
int vqb_gemv_xf(const VqbTensor* w, const void* d_x, int32_t x_dtype, int32_t mode, const void* d_res_in,
                void* d_res_out, const void* d_weight, float eps, void* d_y, int32_t y_dtype,
                const VqbLaunch* launch, void* d_ws, size_t ws_bytes, void* stream);

/* ---- tensor-parallel collectives fused into the decode GEMV ----
 * No vqforge counterpart (the reference is single-device; TP is the paper's future
 * work). Replaces the NCCL all-reduce / all-gather that follows a
 * row- / column-parallel linear (paper_2503_02236_b200/tp.py) with peer-memory
 * stores issued by the GEMV's own epilogue: each output element travels to every
 * rank as soon as its column block is reduced, overlapping the transfer with the
 * remaining tiles. Every rank owns one symmetric buffer of vqb_tp_buffer_bytes,
 * zeroed once and mapped on every peer with the IPC calls below (one process per
 * GPU; on NVSwitch the peer stores travel over NVLink). Collectives run in epochs:
 * the GEMV writes slot parity (epoch & 1) of every rank and the grid's last CTA
 * signals each rank once; vqb_tp_finish waits for all `world` signals, reduces the
 * slots in rank order (identical bits on every rank) or copies the gathered row,
 * and advances the epoch. Stream-ordered and graph-capturable; a rank waits at
 * most ~10 s for its peers, then sets bit 0 of the header's error word
 * (vqb_tp_take_error) instead of hanging. */
#define VQB_TP_HEADER_BYTES 4096
#define VQB_TP_MAX_WORLD 8
#define VQB_TP_ALLREDUCE 0 /* row-parallel: y = sum over ranks of the partial outputs */
#define VQB_TP_ALLGATHER 1 /* column-parallel: y = [y_0 | y_1 | ... ] along N */
typedef struct VqbPeerComm {
  int32_t rank, world;                 /* 1 <= world <= VQB_TP_MAX_WORLD */
  void* d_peer[VQB_TP_MAX_WORLD];      /* every rank's symmetric buffer as mapped here (d_peer[rank] is local) */
  int64_t slot_elems;                  /* fp32 elements per slot: >= rows*N (all-reduce), >= rows*N*world (all-gather) */
} VqbPeerComm;
int64_t vqb_tp_buffer_bytes(int32_t world, int64_t slot_elems);
/* CUDA IPC of a device pointer inside any allocation: 64-byte handle + offset. */
int vqb_ipc_get_handle(const void* d_ptr, void* handle64, int64_t* offset);
int vqb_ipc_open_handle(const void* handle64, int64_t offset, void** d_ptr);
int vqb_ipc_close_handle(void* d_ptr);
/* The decode GEMV (as vqb_gemv, fast configurations only) whose outputs go to the
 * current slot of every rank instead of a local y. */
int vqb_gemv_tp(const VqbTensor* w, const void* d_x, int32_t x_dtype, int32_t rows, int32_t mode,
                const VqbPeerComm* comm, const VqbLaunch* launch, void* d_ws, size_t ws_bytes, void* stream);
/* Wait for every rank's signal, then y (rows, n_local) = sum of the slots
 * (all-reduce) or y (rows, n_local * world) = the gathered slot (all-gather). */
int vqb_tp_finish(const VqbPeerComm* comm, int32_t mode, int32_t rows, int32_t n_local, void* d_y,
                  int32_t y_dtype, void* stream);
/* Read and clear the symmetric buffer's error word (synchronises the device). */
int vqb_tp_take_error(const VqbPeerComm* comm, int32_t* out);

/* Convert a PACKED stream (src, layout must be VQB_LAYOUT_PACKED) into
 * `dst_layout`, writing into d_dst (dst_bytes available). Bytes needed are
 * returned by vqb_layout_bytes. */
int64_t vqb_layout_bytes(const VqbTensor* t, int32_t layout);
int vqb_repack(const VqbTensor* src, int32_t dst_layout, void* d_dst,
               int64_t dst_bytes, void* stream);

/* Measured resource usage of a kernel family at its default configuration for
 * tensor `t` (may be NULL for the family default). */
int vqb_query_usage(int32_t kind, const VqbTensor* t, VqbUsage* out);

/* Debug: write the shared-window offset of dynamic shared memory (kernel with no
 * static shared memory) to d_out[0]. */
int vqb_debug_smem_base(uint32_t* d_out, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* VQB_H_ */
