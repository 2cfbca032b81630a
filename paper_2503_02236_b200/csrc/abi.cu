#include <algorithm>
// abi.cu — C-ABI plumbing, tensor validation, bit-exact dequantization and
// code-layout repacking.
//
// vqb_dequant restates vqforge.codec.dequantize (pkg/src/vqforge/codec.py:391-408):
//   recon = +0.0f; for r in levels: recon += books[r*n_regions + region][code]
// One thread reconstructs one sub-vector; the region comes from coordinates
// (region_layout, codec.py:135-177) and the code from whichever layout the
// tensor is stored in. Accumulation uses __fadd_rn from +0.0f in level order so
// the fp32 result (including -0.0 -> +0.0) is bit-identical to numpy's.
#include <mutex>

#include "common.cuh"

namespace vqb {

static thread_local std::string g_last_error;
static thread_local const char* g_last_kernel = "";

static thread_local int32_t g_last_launch[4] = {0, 0, 0, 0};

void set_kernel(const char* name) { g_last_kernel = name; }
void set_launch(int grid, int threads, int n_shared, int n_reg) {
  g_last_launch[0] = grid;
  g_last_launch[1] = threads;
  g_last_launch[2] = n_shared;
  g_last_launch[3] = n_reg;
}

int set_error(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

int cuda_error(cudaError_t e, const char* what) {
  return set_error(VQB_ECUDA, "CUDA error in %s: %s", what, cudaGetErrorString(e));
}

int sm_count() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (cached[dev] == 0) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cached[dev] = n > 0 ? n : 148;
  }
  return cached[dev];
}

int make_geom(const VqbTensor* t, Geom* g) {
  if (!t) return set_error(VQB_ECONFIG, "null tensor descriptor");
  *g = Geom{};
  g->v = t->vector_size;
  g->bits = t->log2_entries;
  g->R = t->residuals;
  g->sharing = t->sharing;
  g->tile_rows = t->tile_rows;
  g->tile_cols = t->tile_cols;
  g->group_width = t->group_width;
  g->ndim = t->ndim;
  g->layout = t->layout;
  if (!(g->v == 2 || g->v == 4 || g->v == 8 || g->v == 16))
    return set_error(VQB_ECONFIG, "vector_size must be one of (2, 4, 8, 16), got %d", g->v);
  if (g->bits < 1 || g->bits > 16)
    return set_error(VQB_ECONFIG, "log2_entries must be in [1, 16], got %d", g->bits);
  if (g->R < 1) return set_error(VQB_ECONFIG, "residuals must be >= 1, got %d", g->R);
  if (g->ndim < 1 || g->ndim > 4) return set_error(VQB_ESHAPE, "tensor rank %d not in [1, 4]", g->ndim);
  g->K = 1 << g->bits;
  g->rows = 1;
  for (int i = 0; i < g->ndim; ++i) {
    g->dims[i] = t->dims[i];
    if (t->dims[i] < 1) return set_error(VQB_ESHAPE, "non-positive extent %lld", (long long)t->dims[i]);
    if (i < g->ndim - 1) g->rows *= t->dims[i];
  }
  g->cols = t->dims[g->ndim - 1];
  g->d_T = g->ndim >= 2 ? t->dims[g->ndim - 2] : 1;
  g->d_H = g->ndim == 4 ? t->dims[1] : 1;
  if (g->cols % g->v != 0)
    return set_error(VQB_ESHAPE, "last axis %lld not divisible by vector_size %d",
                     (long long)g->cols, g->v);
  g->gpr = g->cols / g->v;
  g->S = g->rows * g->gpr;

  int64_t n_regions = 1;
  if (g->sharing == VQB_SHARE_WHOLE) {
    n_regions = 1;
  } else if (g->sharing == VQB_SHARE_CHANNEL_GROUP) {
    if (g->group_width <= 0) return set_error(VQB_ECONFIG, "channel_group sharing needs positive group_width");
    if (g->group_width % g->v != 0) return set_error(VQB_ECONFIG, "group_width must be a multiple of vector_size");
    if (g->cols % g->group_width != 0)
      return set_error(VQB_ESHAPE, "last axis %lld not divisible by group_width %d",
                       (long long)g->cols, g->group_width);
    n_regions = g->cols / g->group_width;
    if (g->ndim == 4) n_regions *= g->dims[1];
  } else if (g->sharing == VQB_SHARE_TILE) {
    if (g->tile_rows <= 0 || g->tile_cols <= 0)
      return set_error(VQB_ECONFIG, "tile sharing needs positive tile_rows/tile_cols");
    if (g->tile_cols % g->v != 0) return set_error(VQB_ECONFIG, "tile_cols must be a multiple of vector_size");
    if (g->ndim < 2) return set_error(VQB_ESHAPE, "tile sharing requires at least 2-D tensors");
    n_regions = ceil_div(g->dims[g->ndim - 2], g->tile_rows) * ceil_div(g->cols, g->tile_cols);
  } else {
    return set_error(VQB_ECONFIG, "unknown sharing granularity %d", g->sharing);
  }
  if (n_regions != t->n_regions)
    return set_error(VQB_ESHAPE, "descriptor has %d regions, layout implies %lld", t->n_regions,
                     (long long)n_regions);
  g->n_regions = (int)n_regions;
  g->code_bytes = g->bits <= 8 ? 1 : 2;

  int64_t need = 0;
  switch (g->layout) {
    case VQB_LAYOUT_PACKED:
      need = ceil_div((int64_t)g->R * g->S * g->bits, 8);
      break;
    case VQB_LAYOUT_PLAIN:
      need = (int64_t)g->R * g->S * g->code_bytes;
      break;
    case VQB_LAYOUT_GEMV_IL: {
      if (g->ndim != 2) return set_error(VQB_ESHAPE, "GEMV_IL layout needs a 2-D weight");
      const int rpl = 16 / g->code_bytes;
      if (g->rows % rpl != 0)
        return set_error(VQB_ESHAPE, "GEMV_IL layout needs M %% %d == 0, got M=%lld", rpl, (long long)g->rows);
      need = (int64_t)g->R * g->S * g->code_bytes;
      break;
    }
    case VQB_LAYOUT_KV_IL: {
      if (g->ndim != 4) return set_error(VQB_ESHAPE, "KV_IL layout needs a 4-D (B,H,T,C) tensor");
      if (g->bits > 8) return set_error(VQB_ECONFIG, "KV_IL layout needs codes of at most 8 bits");
      if (g->gpr != 32 && g->gpr != 64)
        return set_error(VQB_ESHAPE, "KV_IL layout needs C/v in {32, 64}, got %lld", (long long)g->gpr);
      if (g->dims[2] % 32 != 0)
        return set_error(VQB_ESHAPE, "KV_IL layout needs T %% 32 == 0, got T=%lld", (long long)g->dims[2]);
      need = (int64_t)g->R * g->S;
      break;
    }
    default:
      return set_error(VQB_ECONFIG, "unknown code layout %d", g->layout);
  }
  if (t->d_codes == nullptr && need > 0) return set_error(VQB_ECONFIG, "null code stream");
  if (t->codes_bytes < need)
    return set_error(VQB_ESHAPE, "packed stream truncated: %lld < %lld bytes", (long long)t->codes_bytes,
                     (long long)need);
  if (t->d_codebooks == nullptr) return set_error(VQB_ECONFIG, "null codebooks");
  if (t->codebook_dtype < VQB_F32 || t->codebook_dtype > VQB_BF16)
    return set_error(VQB_ECONFIG, "unknown codebook dtype %d", t->codebook_dtype);
  return VQB_OK;
}

// ---------------------------------------------------------------------------
// dequantize

template <int V, typename CB>
__global__ void __launch_bounds__(256) dequant_kernel(Geom g, const void* __restrict__ codes,
                                                      const CB* __restrict__ books,
                                                      void* __restrict__ out, int out_dtype) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < g.S; s += stride) {
    const int region = region_of(g, s);
    float acc[V];
#pragma unroll
    for (int j = 0; j < V; ++j) acc[j] = 0.0f;
    for (int r = 0; r < g.R; ++r) {
      const uint32_t c = code_at(g, codes, r, s);
      const CB* e = books + ((int64_t)(r * g.n_regions + region) * g.K + c) * V;
#pragma unroll
      for (int j = 0; j < V; ++j) acc[j] = __fadd_rn(acc[j], to_f32<CB>(e[j]));
    }
    const int64_t base = s * V;
    if (out_dtype == VQB_F32 && (V % 4) == 0) {
      float4* o = reinterpret_cast<float4*>(reinterpret_cast<float*>(out) + base);
#pragma unroll
      for (int j = 0; j < V / 4; ++j) o[j] = make_float4(acc[4 * j], acc[4 * j + 1], acc[4 * j + 2], acc[4 * j + 3]);
    } else {
#pragma unroll
      for (int j = 0; j < V; ++j) store_from_f32(out, out_dtype, base + j, acc[j]);
    }
  }
}

template <typename CB>
static void launch_dequant_cb(const Geom& g, const void* codes, const void* books, void* out, int out_dtype,
                              cudaStream_t st) {
  const int threads = 256;
  int64_t blocks = ceil_div(g.S, threads);
  const int64_t cap = (int64_t)sm_count() * 16;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  const CB* b = reinterpret_cast<const CB*>(books);
  switch (g.v) {
    case 2: dequant_kernel<2, CB><<<(unsigned)blocks, threads, 0, st>>>(g, codes, b, out, out_dtype); break;
    case 4: dequant_kernel<4, CB><<<(unsigned)blocks, threads, 0, st>>>(g, codes, b, out, out_dtype); break;
    case 8: dequant_kernel<8, CB><<<(unsigned)blocks, threads, 0, st>>>(g, codes, b, out, out_dtype); break;
    default: dequant_kernel<16, CB><<<(unsigned)blocks, threads, 0, st>>>(g, codes, b, out, out_dtype); break;
  }
}

int launch_dequant(const Geom& g, const VqbTensor* t, void* out, int out_dtype, cudaStream_t st) {
  if (g.S == 0) return VQB_OK;
  if (t->codebook_dtype == VQB_F32) launch_dequant_cb<float>(g, t->d_codes, t->d_codebooks, out, out_dtype, st);
  else if (t->codebook_dtype == VQB_F16) launch_dequant_cb<__half>(g, t->d_codes, t->d_codebooks, out, out_dtype, st);
  else launch_dequant_cb<__nv_bfloat16>(g, t->d_codes, t->d_codebooks, out, out_dtype, st);
  VQB_LAUNCH_CHECK("dequant_kernel");
  set_kernel("dequant");
  return VQB_OK;
}

// ---------------------------------------------------------------------------
// repack: any source layout -> PLAIN / GEMV_IL / KV_IL

__global__ void __launch_bounds__(256) repack_kernel(Geom src, const void* __restrict__ codes, Geom dst,
                                                     void* __restrict__ out) {
  const int64_t total = (int64_t)src.R * src.S;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
    const int r = (int)(i / src.S);
    const int64_t s = i - (int64_t)r * src.S;
    const uint32_t c = code_at(src, codes, r, s);
    const int64_t off = dst.layout == VQB_LAYOUT_PLAIN ? i : il_offset(dst, r, s);
    if (dst.code_bytes == 1) reinterpret_cast<uint8_t*>(out)[off] = (uint8_t)c;
    else reinterpret_cast<uint16_t*>(out)[off] = (uint16_t)c;
  }
}

static int dest_geom(const VqbTensor* t, int32_t layout, Geom* g) {
  VqbTensor d = *t;
  d.layout = layout;
  d.codes_bytes = INT64_MAX;
  const void* fake = reinterpret_cast<const void*>(uintptr_t(1));
  if (d.d_codes == nullptr) d.d_codes = fake;
  if (d.d_codebooks == nullptr) d.d_codebooks = fake;
  return make_geom(&d, g);
}

// Shared-window offset of dynamic shared memory in a kernel without static
// shared memory: the kernels fold region bases into PRMT-built addresses when
// this is 64 KB aligned (tested by tests/test_gpu_kernels.py).
__global__ void smem_base_probe_kernel(uint32_t* out) {
  extern __shared__ __align__(16) uint8_t dyn[];
  if (threadIdx.x == 0) out[0] = smem_u32(dyn);
}

int gemv_usage(VqbUsage* u);
int attn_usage(VqbUsage* u);
int gemm_usage(VqbUsage* u);

}  // namespace vqb

using namespace vqb;

extern "C" {

int vqb_abi_version(void) { return VQB_ABI_VERSION; }

const char* vqb_last_error(void) { return g_last_error.c_str(); }

const char* vqb_last_kernel(void) { return g_last_kernel; }
int vqb_last_launch(int32_t* out4) {
  for (int i = 0; i < 4; ++i) out4[i] = g_last_launch[i];
  return VQB_OK;
}

int vqb_dequant(const VqbTensor* t, void* d_out, int32_t out_dtype, void* stream) {
  Geom g;
  int st = make_geom(t, &g);
  if (st) return st;
  if (out_dtype < VQB_F32 || out_dtype > VQB_BF16) return set_error(VQB_ECONFIG, "unknown output dtype %d", out_dtype);
  if (!d_out && g.S) return set_error(VQB_ECONFIG, "null output");
  return launch_dequant(g, t, d_out, out_dtype, reinterpret_cast<cudaStream_t>(stream));
}

int64_t vqb_layout_bytes(const VqbTensor* t, int32_t layout) {
  Geom g;
  int st = dest_geom(t, layout, &g);
  if (st) return st;
  switch (layout) {
    case VQB_LAYOUT_PACKED: return (ceil_div((int64_t)g.R * g.S * g.bits, 32) + 1) * 4;
    case VQB_LAYOUT_KV_IL: return (int64_t)g.R * g.S;
    default: return (int64_t)g.R * g.S * g.code_bytes;
  }
}

int vqb_repack(const VqbTensor* src, int32_t dst_layout, void* d_dst, int64_t dst_bytes, void* stream) {
  Geom gs, gd;
  int st = make_geom(src, &gs);
  if (st) return st;
  if (dst_layout == VQB_LAYOUT_PACKED) return set_error(VQB_ECONFIG, "repack to PACKED is host-side (bitpack)");
  st = dest_geom(src, dst_layout, &gd);
  if (st) return st;
  const int64_t need = vqb_layout_bytes(src, dst_layout);
  if (need < 0) return (int)need;
  if (dst_bytes < need) return set_error(VQB_ESHAPE, "repack destination too small: %lld < %lld", (long long)dst_bytes,
                                         (long long)need);
  const int64_t total = (int64_t)gs.R * gs.S;
  if (total == 0) return VQB_OK;
  int64_t blocks = ceil_div(total, 256);
  if (blocks > (int64_t)sm_count() * 32) blocks = (int64_t)sm_count() * 32;
  repack_kernel<<<(unsigned)blocks, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(gs, src->d_codes, gd, d_dst);
  VQB_LAUNCH_CHECK("repack_kernel");
  set_kernel("repack");
  return VQB_OK;
}

int vqb_debug_smem_base(uint32_t* d_out, void* stream) {
  smem_base_probe_kernel<<<1, 32, 65536 + 1024, reinterpret_cast<cudaStream_t>(stream)>>>(d_out);
  cudaError_t e = cudaGetLastError();
  if (e == cudaErrorInvalidValue) {
    cudaFuncSetAttribute(smem_base_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    smem_base_probe_kernel<<<1, 32, 65536 + 1024, reinterpret_cast<cudaStream_t>(stream)>>>(d_out);
    e = cudaGetLastError();
  }
  if (e != cudaSuccess) return cuda_error(e, "smem_base_probe_kernel");
  return VQB_OK;
}

int vqb_query_usage(int32_t kind, const VqbTensor* t, VqbUsage* out) {
  (void)t;
  if (!out) return set_error(VQB_ECONFIG, "null usage output");
  *out = VqbUsage{};
  out->sm_count = sm_count();
  switch (kind) {
    case VQB_KERNEL_DEQUANT: {
      cudaFuncAttributes a;
      VQB_CUDA_CHECK(cudaFuncGetAttributes(&a, dequant_kernel<8, __half>));
      out->shared_bytes = (int)a.sharedSizeBytes;
      out->regs_per_thread = a.numRegs;
      out->threads_per_block = 256;
      int nb = 0;
      VQB_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, dequant_kernel<8, __half>, 256, 0));
      out->max_blocks_per_sm = nb;
      return VQB_OK;
    }
    case VQB_KERNEL_GEMV: return gemv_usage(out);
    case VQB_KERNEL_ATTN: return attn_usage(out);
    case VQB_KERNEL_GEMM: return gemm_usage(out);
    default: return set_error(VQB_ECONFIG, "unknown kernel kind %d", kind);
  }
}

}  // extern "C"

namespace vqb {
int64_t gemv_ws_bytes(const VqbTensor* w, int64_t rows, const VqbLaunch* L);
int64_t attn_ws_bytes(const VqbTensor* k, int64_t BH, const VqbLaunch* L);
int64_t gemm_ws_bytes(const VqbTensor* w, int64_t rows, const VqbLaunch* L);
}  // namespace vqb

extern "C" int64_t vqb_workspace_bytes(int32_t kind, const VqbTensor* t, int64_t rows, const VqbLaunch* launch) {
  switch (kind) {
    case VQB_KERNEL_GEMV: return vqb::gemv_ws_bytes(t, rows, launch);
    case VQB_KERNEL_GEMM: {
      const int64_t a = vqb::gemv_ws_bytes(t, rows, launch);
      if (a < 0) return a;
      return std::max(a, vqb::gemm_ws_bytes(t, rows, launch));  // split-K partials / two-phase scratch, or the generic fallback
    }
    case VQB_KERNEL_ATTN: return vqb::attn_ws_bytes(t, rows, launch);
    case VQB_KERNEL_DEQUANT: return 0;
    default: return vqb::set_error(VQB_ECONFIG, "unknown kernel kind %d", kind);
  }
}
