// common.cuh — shared device/host helpers for the B200 VQ kernels.
//
// Device-side restatement of the reference's tensor addressing:
//   * region of a sub-vector   : region_layout (pkg/src/vqforge/codec.py:135-177)
//   * codebook index           : level * n_regions + region (codec.py:208-209)
//   * packed code stream       : bitpack.pack_indices, LSB-first (bitpack.py:13-28)
// computed inline from coordinates instead of materialising int64 temporaries.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>
#include <string>
#include <utility>

#include "../../include/vqb.h"

namespace vqb {

// ---------------------------------------------------------------------------
// error plumbing (host)

int set_error(int code, const char* fmt, ...);
int cuda_error(cudaError_t e, const char* what);
int sm_count();
void set_kernel(const char* name);
// Persistent grid for `units` equal work units: the fewest CTAs that still give the
// minimal per-CTA load ceil(units / SMs). Same makespan as one CTA per SM, but
// every CTA gets the same whole number of units (no CTA waits on a longer
// neighbour, fewer split outputs / codebook switches).
inline int balanced_grid(int64_t units, int sms) {
  if (units <= 0) return 1;
  const int64_t per = (units + sms - 1) / sms;
  return (int)((units + per - 1) / per);
}
// grid, threads, shared-tier entries and register-tier entries of the last fused launch
void set_launch(int grid, int threads, int n_shared, int n_reg);

#define VQB_CUDA_CHECK(expr)                            \
  do {                                                  \
    cudaError_t _e = (expr);                            \
    if (_e != cudaSuccess) return ::vqb::cuda_error(_e, #expr); \
  } while (0)

#define VQB_LAUNCH_CHECK(what)                               \
  do {                                                       \
    cudaError_t _e = cudaGetLastError();                     \
    if (_e != cudaSuccess) return ::vqb::cuda_error(_e, what); \
  } while (0)

// ---------------------------------------------------------------------------
// tensor geometry, flattened for kernels (passed by value)

struct Geom {
  int v;          // vector size
  int bits;       // log2 entries
  int R;          // residual levels
  int K;          // entries per codebook
  int sharing;
  int tile_rows, tile_cols, group_width;
  int ndim;
  int64_t dims[4];
  int n_regions;
  int64_t cols;   // last axis
  int64_t gpr;    // sub-vectors per row (G)
  int64_t rows;   // product of leading axes
  int64_t S;      // sub-vectors per level
  int layout;
  int code_bytes; // 1 or 2 for PLAIN / IL layouts
  int64_t d_H;    // dims[1] of a 4-D tensor (heads)
  int64_t d_T;    // dims[ndim-2] (tokens of a 4-D tensor, rows of the last 2-D slice)
};

int make_geom(const VqbTensor* t, Geom* g);  // validates, returns VQB_* status

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Region of sub-vector s (row-major sub-vector order), codec.py:135-177.
__device__ __forceinline__ int region_of(const Geom& g, int64_t s) {
  if (g.sharing == VQB_SHARE_WHOLE) return 0;
  const int64_t row = s / g.gpr;
  const int64_t col = (s - row * g.gpr) * g.v;
  if (g.sharing == VQB_SHARE_CHANNEL_GROUP) {
    const int64_t n_groups = g.cols / g.group_width;
    const int64_t grp = col / g.group_width;
    if (g.ndim == 4) {
      const int64_t head = (row / g.d_T) % g.d_H;
      return (int)(head * n_groups + grp);
    }
    return (int)grp;
  }
  // tile sharing over the last two axes, shared across leading axes
  const int64_t r2 = g.d_T;
  const int64_t n_tc = ceil_div(g.cols, g.tile_cols);
  const int64_t local_row = row % r2;
  return (int)((local_row / g.tile_rows) * n_tc + col / g.tile_cols);
}

// KV_IL inside one (b, h) block (G = C/v groups, 32 or 64), per 32-token batch:
// [G/16 words][32 lanes][16 bytes]. The warp is cut into 32/kKvLanes lane sets; set h
// = lane / kKvLanes holds tokens kKvLanes*h + (0..kKvLanes-1), and lane (h, ll = lane %
// kKvLanes) owns groups ll + kKvLanes*(j ^ h), j < G/kKvLanes, storing token
// kKvLanes*h + (i ^ ll) at slot i, byte i*(G/kKvLanes) + j. The XOR orders make the
// attention kernel's cross-lane logit reduction select-free (log2(kKvLanes) shuffle
// levels inside each set), and the (j ^ h) swap puts the sets of every shared load on
// distinct banks.
constexpr int kKvLanes = 8;
__host__ __device__ __forceinline__ int64_t kvil_offset(int64_t t, int grp, int G) {
  const int gph = G / kKvLanes;
  const int h = (int)(t & 31) / kKvLanes, ll = grp % kKvLanes, j = (grp / kKvLanes) ^ h;
  const int lane = h * kKvLanes + ll, slot = (int)(t % kKvLanes) ^ ll;
  const int byte = slot * gph + j;
  return (t >> 5) * 32 * (int64_t)G + ((byte >> 4) * 32 + lane) * 16 + (byte & 15);
}

// Offset (in codes) of code (level r, sub-vector s) inside an interleaved layout.
__device__ __forceinline__ int64_t il_offset(const Geom& g, int r, int64_t s) {
  if (g.layout == VQB_LAYOUT_GEMV_IL) {
    // column-blocked: per level [N/256 column blocks][M/rpl row groups][256/v groups][rpl rows]
    // (the last block may be narrower), so one block's chunk of rows is contiguous
    const int rpl = 16 / g.code_bytes;
    const int64_t gcb = 256 / g.v;
    const int64_t m = s / g.gpr, grp = s - (s / g.gpr) * g.gpr;
    const int64_t cb = grp / gcb, gi = grp - cb * gcb;
    const int64_t wb = min(gcb, g.gpr - cb * gcb);
    return (int64_t)r * g.S + cb * gcb * g.rows + ((m / rpl) * wb + gi) * rpl + (m % rpl);
  }
  const int64_t T = g.d_T;
  const int64_t row = s / g.gpr, grp = s - (s / g.gpr) * g.gpr;
  const int64_t bh = row / T, t = row - (row / T) * T;
  return (int64_t)r * g.S + bh * T * g.gpr + kvil_offset(t, (int)grp, (int)g.gpr);
}

// Code of level r for sub-vector s, from any layout.
__device__ __forceinline__ uint32_t code_at(const Geom& g, const void* codes, int r, int64_t s) {
  if (g.layout == VQB_LAYOUT_PACKED) {
    const uint32_t* w = reinterpret_cast<const uint32_t*>(codes);
    const int64_t bit = ((int64_t)r * g.S + s) * g.bits;
    const int64_t wi = bit >> 5;
    const int sh = (int)(bit & 31);
    uint32_t lo = __ldg(w + wi);
    uint32_t val = lo >> sh;
    if (sh + g.bits > 32) val |= __ldg(w + wi + 1) << (32 - sh);
    return val & ((1u << g.bits) - 1u);
  }
  int64_t off = (g.layout == VQB_LAYOUT_PLAIN) ? (int64_t)r * g.S + s : il_offset(g, r, s);
  if (g.code_bytes == 1) return __ldg(reinterpret_cast<const uint8_t*>(codes) + off);
  return __ldg(reinterpret_cast<const uint16_t*>(codes) + off);
}

template <typename T>
__device__ __forceinline__ float to_f32(T x);
template <>
__device__ __forceinline__ float to_f32<float>(float x) { return x; }
template <>
__device__ __forceinline__ float to_f32<__half>(__half x) { return __half2float(x); }
template <>
__device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 x) { return __bfloat162float(x); }

__device__ __forceinline__ float load_as_f32(const void* p, int dtype, int64_t i) {
  if (dtype == VQB_F32) return __ldg(reinterpret_cast<const float*>(p) + i);
  if (dtype == VQB_F16) return __half2float(reinterpret_cast<const __half*>(p)[i]);
  return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[i]);
}

__device__ __forceinline__ void store_from_f32(void* p, int dtype, int64_t i, float v) {
  if (dtype == VQB_F32) reinterpret_cast<float*>(p)[i] = v;
  else if (dtype == VQB_F16) reinterpret_cast<__half*>(p)[i] = __float2half_rn(v);
  else reinterpret_cast<__nv_bfloat16*>(p)[i] = __float2bfloat16_rn(v);
}

// fp32 += fp16 * fp16, single rounding (sm_100 FHFMA): products of two halves are
// exact in fp32, so this is an fp32 FMA on exactly-widened operands.
__device__ __forceinline__ float fma_h(uint16_t a, uint16_t b, float c) {
  float d;
  asm("fma.rn.f32.f16 %0, %1, %2, %3;" : "=f"(d) : "h"(a), "h"(b), "f"(c));
  return d;
}

// packed fp16x2 fused multiply-add (HFMA2), round-to-nearest
__device__ __forceinline__ uint32_t hfma2(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

// HFMA2 with the activation half (lo or hi of a packed pair) broadcast to both
// lanes: ptxas folds the splat into the .H0_H0 / .H1_H1 operand selector.
template <int HI>
__device__ __forceinline__ uint32_t hfma2_bcast(uint32_t a, uint32_t xw, uint32_t c) {
  uint32_t d;
  if constexpr (HI)
    asm("{.reg .f16 xl, xh; .reg .b32 xx; mov.b32 {xl, xh}, %2; mov.b32 xx, {xh, xh}; fma.rn.f16x2 %0, %1, xx, %3;}"
        : "=r"(d) : "r"(a), "r"(xw), "r"(c));
  else
    asm("{.reg .f16 xl, xh; .reg .b32 xx; mov.b32 {xl, xh}, %2; mov.b32 xx, {xl, xl}; fma.rn.f16x2 %0, %1, xx, %3;}"
        : "=r"(d) : "r"(a), "r"(xw), "r"(c));
  return d;
}

__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint2 lds64(uint32_t addr) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ float lds_f32(uint32_t addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint4 ldg_stream(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
// L2 policy for single-use streams (decode weight codes, KV codes): the lines are the
// first evicted, so the small reused data of a step (codebooks, activations, partial
// slots) stays resident in L2 from one kernel and one step to the next
__device__ __forceinline__ uint64_t l2_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint4 ldg_stream_hint(const void* p, uint64_t pol) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---- mbarrier + bulk-async-copy (TMA) primitives (sm_90+/sm_100a PTX) ----------

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
// 1-D bulk copy global -> shared, completing `bytes` of transaction on `bar`.
__device__ __forceinline__ void tma_load_1d(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma_load_1d_hint(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar,
                                                 uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          dst),
      "l"(src), "r"(bytes), "r"(bar), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa_rank(uint32_t addr, uint32_t rank) {
  uint32_t d;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(d) : "r"(addr), "r"(rank));
  return d;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Launch with programmatic dependent launch allowed: the kernel may start while its
// predecessor on the stream drains; it must call pdl_wait() before touching that
// predecessor's outputs and calls pdl_launch_dependents() to let its successor start.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// Launch attributes of the persistent split-reduction kernels: programmatic
// dependent launch (unless VQB_FLAG_NO_PDL) and, with VQB_FLAG_COOPERATIVE, a
// cooperative launch (co-residency of the whole grid guaranteed by the driver).
inline int persistent_attrs(cudaLaunchAttribute* attr, int flags) {
  int n = 0;
  if (flags & VQB_FLAG_COOPERATIVE) {
    attr[n].id = cudaLaunchAttributeCooperative;
    attr[n].val.cooperative = 1;
    ++n;
  } else if (!(flags & VQB_FLAG_NO_PDL)) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  return n;
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// A partial travels as one 64-bit word {fp32 value, tag}: an aligned 8-byte store
// is single-copy atomic, so a reader that sees the tag also sees the value — no
// fence or flag round trip between producer and consumer.
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long tag_partial(float v) {
  return (1ull << 32) | (unsigned long long)__float_as_uint(v);
}


// ---------------------------------------------------------------------------
// Tensor-parallel collectives over peer memory (tp.cu, vqb_gemv_tp): every rank owns
// one symmetric buffer, VQB_TP_HEADER_BYTES of header then two parities of fp32
// slots. Header words: [0] arrive[2] (u64, incremented remotely by every rank's
// producer, one per collective), [64] producer CTA counter, [128] epoch (collectives
// finished on this rank), [192] finish-kernel CTA counter, [256] error word.
constexpr int kTpMaxWorld = 8;
constexpr int kTpOffDone = 64, kTpOffEpoch = 128, kTpOffFinish = 192, kTpOffErr = 256;

__device__ __forceinline__ int tp_epoch_of(const char* me) {
  return *reinterpret_cast<const volatile int*>(me + kTpOffEpoch);
}
// slot element of output (b, n): all-reduce [par][rank][b][N]; all-gather
// [par][b][world * N] with this rank's N columns at rank * N
__device__ __forceinline__ int64_t tp_slot_offset(int mode, int par, int world, int rank, int64_t slot_elems, int b,
                                                  int n, int N) {
  return mode == 0 ? ((int64_t)par * world + rank) * slot_elems + (int64_t)b * N + n
                   : (int64_t)par * slot_elems + ((int64_t)b * world + rank) * N + n;
}
// the value into every rank's slot (peer-memory stores over NVLink; the own rank's
// buffer is local)
__device__ __forceinline__ void tp_push(char* const* peer, int world, int64_t off, float v) {
#pragma unroll 1
  for (int p = 0; p < world; ++p)
    reinterpret_cast<float*>(peer[p] + VQB_TP_HEADER_BYTES)[off] = v;
}
// End of a producer grid: every CTA fences its pushes system-wide and counts itself;
// the last one signals arrive[par] on every rank (release at system scope).
__device__ __forceinline__ void tp_signal(char* const* peer, int world, int rank, int par) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    unsigned* done = reinterpret_cast<unsigned*>(peer[rank] + kTpOffDone);
    unsigned prev;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(done) : "memory");
    if (prev == gridDim.x - 1) {
      *reinterpret_cast<volatile unsigned*>(done) = 0u;  // every CTA arrived: reset for the next launch
      __threadfence_system();
      for (int p = 0; p < world; ++p) {
        unsigned long long* arr = reinterpret_cast<unsigned long long*>(peer[p]) + par;
        asm volatile("red.release.sys.global.add.u64 [%0], 1;" ::"l"(arr) : "memory");
      }
    }
  }
}

}  // namespace vqb
