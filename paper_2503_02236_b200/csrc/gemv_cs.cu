// gemv_cs.cu — column-split decode GEMV for narrow outputs (batch 1).
//
// Same operator as gemv.cu (SimMachine._matmul's GEMV branch, sim.py:697-775:
// y = x @ dequant(W), W (M, N) with v = 8 sub-vectors along N), for the shapes where
// the stream-K kernel has to split the reduction over M: N = 4096 (o_proj, down_proj)
// gives 16 column blocks of 256, so ~8 CTAs share a block and the block's CTA holding
// chunk 0 waits for the others' partials through L2 — a per-CTA trace
// (tools/gemv_trace.py) shows that tail at ~1.7 us of a 5 us o_proj call.
//
// Here every CTA owns a 32-column slice (4 sub-vector groups) of one column block for
// ALL M rows, so the reduction stays inside the CTA: no partials, no polling, no
// tail. The codes are read from the same GEMV_IL layout (a row group's 32 words of a
// block are contiguous; a slice reads 64 of its 512 bytes) with plain 16-byte loads
// kept several words deep per thread; the codebook (every code < 256) sits in shared
// memory replicated 8x exactly as in gemv.cu (lane l of each quarter-warp reads
// replica l % 8: conflict-free 4-wavefront LDS.128), and the products accumulate in
// the same 8-row fp16x2 windows flushed into fp32 (the fast GEMV's arithmetic class).
#include "common.cuh"

namespace vqb {

constexpr int kCsDepth = 8;                   // 16-byte code words in flight per thread
constexpr int kCsRep = 8;                     // codebook replicas (16-byte entries, 128-byte rows)

struct GemvCsArgs {
  const uint8_t* codes;  // GEMV_IL, u16 codes, one level
  const __half* books;   // (K, 8) fp16, entries [0, n_sh) used
  const __half* x;       // (B, M)
  void* y;
  int y_dtype;
  int M, N, n_sh;
};

// B batch rows, SG sub-vector groups (of 8 columns) per CTA, NT threads
template <int B, int SG, int NT>
__global__ void __launch_bounds__(NT) gemv_cs_kernel(GemvCsArgs a) {
  constexpr int kCsThreads = NT, kCsWarps = NT / 32, kCsGroups = SG, kCsRowLanes = 32 / SG, CPC = SG * 8;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* books_s = smem;                                            // n_sh x 128 B
  __half* x_s = reinterpret_cast<__half*>(smem + 256 * 128);          // B x M halves
  float* red = reinterpret_cast<float*>(smem + 256 * 128 + ((B * a.M * 2 + 15) & ~15));  // warps x B x CPC

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gl = lane % kCsGroups, rl = lane / kCsGroups;
  const int n_slices = 32 / kCsGroups;
  const int cb = blockIdx.x / n_slices, sl = blockIdx.x % n_slices;
  const int gi = sl * kCsGroups + gl;  // this lane's group inside the column block
  const int M8 = a.M / 8;               // row groups (8 rows per 16-byte word)
  // block cb of the level: 32 groups x M rows of u16 codes; word (m8, gi) at (m8*32 + gi)*16
  const uint8_t* base = a.codes + (int64_t)cb * 32 * a.M * 2 + (int64_t)gi * 16;
  const uint64_t pol = l2_evict_first();
  pdl_launch_dependents();

  // row groups of this thread: rg(k) = (k * kCsWarps + warp) * kCsRowLanes + rl
  const int stride = kCsWarps * kCsRowLanes;
  const int first = warp * kCsRowLanes + rl;
  const int n_mine = first < M8 ? (M8 - first + stride - 1) / stride : 0;
  uint4 cw[kCsDepth];
#pragma unroll
  for (int d = 0; d < kCsDepth; ++d)
    if (d < n_mine) cw[d] = ldg_stream_hint(base + (int64_t)(first + d * stride) * 512, pol);

  // codebook: entry e -> row e of 8 replicas (rotated so a row's 8 stores hit distinct banks)
  for (int e = tid; e < a.n_sh; e += kCsThreads) {
    const uint4 q = __ldg(reinterpret_cast<const uint4*>(a.books) + e);
#pragma unroll
    for (int r = 0; r < kCsRep; ++r)
      *reinterpret_cast<uint4*>(books_s + (size_t)e * 128 + ((r + e) % kCsRep) * 16) = q;
  }
  pdl_wait();  // x comes from the previous kernel
  for (int i = tid; i < B * a.M / 8; i += kCsThreads)
    reinterpret_cast<uint4*>(x_s)[i] = __ldg(reinterpret_cast<const uint4*>(a.x) + i);
  __syncthreads();

  const uint32_t bk = smem_u32(books_s) + (uint32_t)(lane % kCsRep) * 16;
  const uint32_t xb = smem_u32(x_s);
  float acc[B][8];
#pragma unroll
  for (int b = 0; b < B; ++b)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[b][j] = 0.f;
  for (int k0 = 0; k0 < n_mine; k0 += kCsDepth) {
#pragma unroll
    for (int d = 0; d < kCsDepth; ++d) {
      const int k = k0 + d;
      if (k < n_mine) {
        const uint4 w = cw[d];
        if (k + kCsDepth < n_mine) cw[d] = ldg_stream_hint(base + (int64_t)(first + (k + kCsDepth) * stride) * 512, pol);
        const int rg = first + k * stride;
        uint4 xv[B];
#pragma unroll
        for (int b = 0; b < B; ++b) xv[b] = lds128(xb + (uint32_t)(b * a.M * 2) + (uint32_t)rg * 16);  // rows 8rg..+7
        uint32_t hw[B][4];
#pragma unroll
        for (int b = 0; b < B; ++b)
#pragma unroll
          for (int j = 0; j < 4; ++j) hw[b][j] = 0u;
#pragma unroll
        for (int kr = 0; kr < 8; ++kr) {
          const uint32_t ww = (&w.x)[kr / 2];
          const uint32_t code = (kr & 1) ? (ww >> 16) : (ww & 0xffffu);
          // every slot of a row holds the entry: lane l reads slot l % 8, so each
          // quarter-warp's eight 16-byte reads hit eight distinct bank groups
          const uint4 q = lds128(bk + code * 128);
#pragma unroll
          for (int b = 0; b < B; ++b) {
            const uint32_t xw = (&xv[b].x)[kr / 2];
#pragma unroll
            for (int j = 0; j < 4; ++j)
              hw[b][j] = (kr & 1) ? hfma2_bcast<1>((&q.x)[j], xw, hw[b][j]) : hfma2_bcast<0>((&q.x)[j], xw, hw[b][j]);
          }
        }
#pragma unroll
        for (int b = 0; b < B; ++b)
#pragma unroll
          for (int j = 0; j < 4; ++j) {  // flush the 8-row window (exact widening)
            acc[b][2 * j] = fma_h((uint16_t)(hw[b][j] & 0xffff), (uint16_t)0x3C00, acc[b][2 * j]);
            acc[b][2 * j + 1] = fma_h((uint16_t)(hw[b][j] >> 16), (uint16_t)0x3C00, acc[b][2 * j + 1]);
          }
      }
    }
  }
  // reduce over the row lanes of each group (fixed order), then over the warps
#pragma unroll
  for (int o = kCsGroups; o < 32; o <<= 1)
#pragma unroll
    for (int b = 0; b < B; ++b)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[b][j] += __shfl_xor_sync(0xffffffffu, acc[b][j], o);
  if (rl == 0)
#pragma unroll
    for (int b = 0; b < B; ++b)
#pragma unroll
      for (int j = 0; j < 8; ++j) red[(warp * B + b) * CPC + gl * 8 + j] = acc[b][j];
  __syncthreads();
  for (int i = tid; i < B * CPC; i += NT) {
    const int b = i / CPC, c = i % CPC;
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < kCsWarps; ++w) s += red[(w * B + b) * CPC + c];
    store_from_f32(a.y, a.y_dtype, (int64_t)b * a.N + (int64_t)cb * 256 + sl * CPC + c, s);
  }
}

typedef void (*GemvCsKernel)(GemvCsArgs);
static GemvCsKernel pick_cs(int rows) {
  return rows == 1 ? gemv_cs_kernel<1, 4, 512> : rows == 2 ? gemv_cs_kernel<2, 4, 512> : gemv_cs_kernel<4, 4, 512>;
}

// 1 = not covered (the caller falls back to the stream-K kernels)
int gemv_cs_dispatch(const Geom& g, const VqbTensor* w, const void* x, int x_dtype, int rows, void* y, int y_dtype,
                     const VqbLaunch* L, cudaStream_t st) {
  if (L && (L->flags & (VQB_FLAG_FORCE_GENERIC | VQB_FLAG_NO_SHARED | VQB_FLAG_EXACT_ACCUM | VQB_FLAG_NO_COLSPLIT)))
    return 1;
  if (L && (L->split_factor > 0 || L->grid_limit > 0 || L->n_reg > 0)) return 1;  // planner-directed launches
  if ((rows != 1 && rows != 2 && rows != 4) || x_dtype != VQB_F16 || g.v != 8 || g.R != 1 || g.code_bytes != 2 || g.ndim != 2 ||
      g.sharing != VQB_SHARE_WHOLE || w->layout != VQB_LAYOUT_GEMV_IL || w->codebook_dtype != VQB_F16)
    return 1;
  const int n_sh = g.K <= 256 ? g.K : ((w->max_code >= 0 && w->max_code < 256) ? (int)w->max_code + 1 : -1);
  if (n_sh <= 0 || (g.cols % 256) != 0 || (g.rows % 8) != 0 || (reinterpret_cast<uintptr_t>(x) & 15) != 0) return 1;
  const int n_cblk = (int)(g.cols / 256);
  // one wave of n_cblk x 8 CTAs (o / down: 16 blocks). Measured: wider outputs with 8- or
  // 16-group slices on 256-thread CTAs sharing SMs (qkv 192 CTAs, gate_up 172) are slower
  // than the stream-K kernel (9.8 vs 8.6 us, 18.7 vs 11.5 us at batch 1).
  const int sms = sm_count();
  const int SG = 4;
  if (n_cblk * 8 > sms || n_cblk * 8 < sms * 3 / 4) return 1;
  const int NT = 512;
  const int grid = n_cblk * (32 / SG);
  GemvCsArgs a;
  a.codes = reinterpret_cast<const uint8_t*>(w->d_codes);
  a.books = reinterpret_cast<const __half*>(w->d_codebooks);
  a.x = reinterpret_cast<const __half*>(x);
  a.y = y;
  a.y_dtype = y_dtype;
  a.M = (int)g.rows;
  a.N = (int)g.cols;
  a.n_sh = n_sh;
  const size_t smem = 256 * 128 + ((size_t)(rows * g.rows * 2 + 15) & ~(size_t)15) + (size_t)(NT / 32) * rows * SG * 8 * 4;
  if (smem > 232448) return 1;
  GemvCsKernel kern = pick_cs(rows);
  const int ki = rows == 1 ? 0 : rows == 2 ? 1 : 2;
  static bool configured[3][64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!configured[ki][dev & 63]) {
    VQB_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448));
    configured[ki][dev & 63] = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  cfg.attrs = attr;
  cfg.numAttrs = persistent_attrs(attr, L ? (L->flags & ~VQB_FLAG_COOPERATIVE) : 0);
  VQB_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, a));
  set_kernel("gemv_cs");
  set_launch(grid, NT, n_sh, 0);
  return 0;
}

}  // namespace vqb
