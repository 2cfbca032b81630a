// gemv.cu — fused VQ dequantisation + decode GEMV, y(rows, N) = x(rows, M) @ W.
//
// Replaces SimMachine._matmul/_mm_block (pkg/src/vqforge/sim.py:697-775) for
// ComputeOp.gemv (dataflow.py:73-75); the numerics the reference checks are
// reference_compute's `a @ dequantize(W)` (sim.py:136-144) within 1e-4 rel-to-max
// (verify.py:200-215).
//
// Fast kernel (B200 design):
//  * codebook cache — the first n_shared entries of every codebook the CTA needs
//    live in shared memory REPLICATED 128/EB times (EB = entry bytes): entry e
//    occupies one 128-byte bank row and lane l reads replica (l mod 128/EB), so a
//    warp-wide random gather is conflict-free by construction (8 lanes of an
//    LDS.128 quarter-warp or 16 lanes of an LDS.64 half-warp always hit distinct
//    bank groups). Entries >= n_shared are read from the global/L2 tier.
//  * codebook-centric dataflow — a CTA tile is 32*WG sub-vector columns x a part of
//    M; for tile-shared codebooks (GPTVQ) a 256-row chunk lies inside one codebook
//    region, so the CTA loads exactly one codebook per chunk; whole-tensor books
//    are loaded once per persistent CTA. M is split f ways (DataflowPlan
//    split_factor on "M"), partials reduced deterministically by the last CTA.
//  * codes stream as 16-byte lane loads (GEMV_IL layout: 8 u16 or 16 u8 codes of
//    one column for consecutive rows), fully coalesced 512 B per warp load.
//  * register-level fusion — each lane owns one sub-vector column and multiplies
//    its looked-up fp16 entry straight into fp32 accumulators with the sm_100
//    mixed-precision FMA (fma.rn.f32.f16): no staging, no shuffles.
//
// Generic kernel: any VQConfig / sharing / layout / dtype, fp32 math, bit-exact
// dequantised W (same +0.0f level-order accumulation as vqb_dequant), used for
// parity mode (fp32 codebooks) and for configurations outside the fast table.
#include "common.cuh"

namespace vqb {

constexpr int kGemvThreads = 256;
constexpr int kChunkRows = 256;

struct GemvFastArgs {
  const uint8_t* codes;   // GEMV_IL, level r at codes + r * level_bytes
  int64_t level_bytes;
  const __half* books;    // (R*n_regions, K, V)
  const __half* x;        // (B, M)
  void* y;
  int y_dtype;
  float* part;            // (f, B, N) partials when f > 1
  int* counters;          // n_cblk arrival counters
  int M, N, G, K, n_regions;
  int tile_rows, tile_cols, n_tc;
  int f, chunks_per_part, n_cblk, n_sh;
};

template <int V, int CBYTES, int R, int B, int WG, bool TILE>
__global__ void __launch_bounds__(kGemvThreads) gemv_fast_kernel(GemvFastArgs a) {
  constexpr int EB = V * 2;              // fp16 entry bytes
  constexpr int REP = 128 / EB;          // replicas per bank row
  constexpr int RPL = 16 / CBYTES;       // rows per 16-byte code load
  constexpr int WM = 8 / WG;             // warps along M
  constexpr int RW = kChunkRows / WM;    // rows per warp per chunk
  constexpr int LOADS = RW / RPL;        // 16-byte code loads per lane per level
  constexpr int COLS = 32 * WG * V;      // output columns per CTA tile
  static_assert(LOADS >= 1 && RW % 8 == 0, "bad tiling");

  extern __shared__ __align__(128) uint8_t smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / WG, wg = warp % WG;
  uint8_t* books_s = smem;                                   // R * n_sh * 128
  float* red = reinterpret_cast<float*>(smem + (size_t)R * a.n_sh * 128);  // WM*B*COLS
  __shared__ int s_last;
  const uint32_t books_base = smem_u32(books_s);
  const uint32_t rep_off = (uint32_t)(lane % REP) * EB;

  auto fill = [&](int region) {
    // copy entries [0, n_sh) of each level's codebook into replicated rows
    for (int r = 0; r < R; ++r) {
      const uint8_t* src = reinterpret_cast<const uint8_t*>(a.books) +
                           ((int64_t)(r * a.n_regions + region) * a.K) * EB;
      uint8_t* dst = books_s + (size_t)r * a.n_sh * 128;
      for (int e = tid; e < a.n_sh; e += kGemvThreads) {
        if constexpr (EB == 16) {
          const uint4 v = __ldg(reinterpret_cast<const uint4*>(src) + e);
#pragma unroll
          for (int q = 0; q < REP; ++q)
            *reinterpret_cast<uint4*>(dst + e * 128 + ((q + e) % REP) * EB) = v;
        } else {
          const uint2 v = __ldg(reinterpret_cast<const uint2*>(src) + e);
#pragma unroll
          for (int q = 0; q < REP; ++q)
            *reinterpret_cast<uint2*>(dst + e * 128 + ((q + e) % REP) * EB) = v;
        }
      }
    }
  };

  int cur_region = -1;
  if constexpr (!TILE) {
    fill(0);
    cur_region = 0;
    __syncthreads();
  }

  const int n_tiles = a.n_cblk * a.f;
  for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int cblk = tile % a.n_cblk;
    const int part = tile / a.n_cblk;
    const int g = cblk * 32 * WG + wg * 32 + lane;  // this lane's sub-vector column
    float acc[B][V];
#pragma unroll
    for (int b = 0; b < B; ++b)
#pragma unroll
      for (int j = 0; j < V; ++j) acc[b][j] = 0.f;

    for (int ch = 0; ch < a.chunks_per_part; ++ch) {
      const int chunk = part * a.chunks_per_part + ch;
      const int m0 = chunk * kChunkRows + wm * RW;
      // issue the code stream loads first so their latency overlaps the codebook switch
      uint4 c[R][LOADS];
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int i = 0; i < LOADS; ++i)
          c[r][i] = ldg_stream(a.codes + r * a.level_bytes +
                               ((int64_t)(m0 / RPL + i) * a.G + g) * 16);
      if constexpr (TILE) {
        const int region = (chunk * kChunkRows / a.tile_rows) * a.n_tc + (cblk * COLS) / a.tile_cols;
        if (region != cur_region) {
          __syncthreads();  // every warp is done with the previous codebook
          fill(region);
          cur_region = region;
          __syncthreads();
        }
      }
#pragma unroll
      for (int i = 0; i < LOADS; ++i) {
        // activations of this load's RPL rows (same address on every lane: broadcast)
        uint4 xv[B][RPL / 8];
#pragma unroll
        for (int b = 0; b < B; ++b)
#pragma unroll
          for (int q = 0; q < RPL / 8; ++q)
            xv[b][q] = __ldg(reinterpret_cast<const uint4*>(a.x + (int64_t)b * a.M + m0 + i * RPL) + q);
#pragma unroll
        for (int k = 0; k < RPL; ++k) {
          uint16_t xh[B];
#pragma unroll
          for (int b = 0; b < B; ++b) {
            const uint32_t w = (&xv[b][k / 8].x)[(k % 8) / 2];
            xh[b] = (uint16_t)((k & 1) ? (w >> 16) : (w & 0xffff));
          }
#pragma unroll
          for (int r = 0; r < R; ++r) {
            uint32_t code;
            if constexpr (CBYTES == 2) {
              const uint32_t w = (&c[r][i].x)[k / 2];
              code = (k & 1) ? (w >> 16) : (w & 0xffff);
            } else {
              const uint32_t w = (&c[r][i].x)[k / 4];
              code = (w >> (8 * (k % 4))) & 0xff;
            }
            uint32_t e[V / 2];
            if (code < (uint32_t)a.n_sh) {
              const uint32_t addr = books_base + (uint32_t)r * a.n_sh * 128 + (code << 7) + rep_off;
              if constexpr (EB == 16) {
                const uint4 q = lds128(addr);
                e[0] = q.x; e[1] = q.y; e[2] = q.z; e[3] = q.w;
              } else {
                const uint2 q = lds64(addr);
                e[0] = q.x; e[1] = q.y;
              }
            } else {
              const int region = cur_region < 0 ? 0 : cur_region;
              const uint8_t* gp = reinterpret_cast<const uint8_t*>(a.books) +
                                  (((int64_t)(r * a.n_regions + region) * a.K) + code) * EB;
              if constexpr (EB == 16) {
                const uint4 q = __ldg(reinterpret_cast<const uint4*>(gp));
                e[0] = q.x; e[1] = q.y; e[2] = q.z; e[3] = q.w;
              } else {
                const uint2 q = __ldg(reinterpret_cast<const uint2*>(gp));
                e[0] = q.x; e[1] = q.y;
              }
            }
#pragma unroll
            for (int b = 0; b < B; ++b)
#pragma unroll
              for (int j = 0; j < V / 2; ++j) {
                acc[b][2 * j] = fma_h((uint16_t)(e[j] & 0xffff), xh[b], acc[b][2 * j]);
                acc[b][2 * j + 1] = fma_h((uint16_t)(e[j] >> 16), xh[b], acc[b][2 * j + 1]);
              }
          }
        }
      }
    }

    // ---- reduce the WM row-slabs of this tile in a fixed order ----
#pragma unroll
    for (int b = 0; b < B; ++b)
#pragma unroll
      for (int j = 0; j < V; ++j)
        red[((size_t)wm * B + b) * COLS + (wg * 32 + lane) * V + j] = acc[b][j];
    __syncthreads();
    const int n0 = cblk * COLS;
    for (int o = tid; o < B * COLS; o += kGemvThreads) {
      const int b = o / COLS, col = o % COLS;
      float s = 0.f;
#pragma unroll
      for (int w = 0; w < WM; ++w) s += red[((size_t)w * B + b) * COLS + col];
      if (a.f == 1) store_from_f32(a.y, a.y_dtype, (int64_t)b * a.N + n0 + col, s);
      else a.part[((int64_t)part * B + b) * a.N + n0 + col] = s;
    }
    if (a.f > 1) {
      __threadfence();
      __syncthreads();
      if (tid == 0) s_last = (atomicAdd(a.counters + cblk, 1) == a.f - 1);
      __syncthreads();
      if (s_last) {
        __threadfence();
        for (int o = tid; o < B * COLS; o += kGemvThreads) {
          const int b = o / COLS, col = o % COLS;
          float s = 0.f;
          for (int p = 0; p < a.f; ++p) s += __ldcg(a.part + ((int64_t)p * B + b) * a.N + n0 + col);
          store_from_f32(a.y, a.y_dtype, (int64_t)b * a.N + n0 + col, s);
        }
        if (tid == 0) a.counters[cblk] = 0;  // self-reset for the next launch
      }
    }
    __syncthreads();  // red / s_last reuse by the next tile
  }
}

// ---------------------------------------------------------------------------
// generic path

constexpr int kGenericRowBlock = 4;

template <typename CB, int V>
__global__ void __launch_bounds__(128) gemv_generic_kernel(Geom g, const void* __restrict__ codes,
                                                           const CB* __restrict__ books,
                                                           const void* __restrict__ x, int x_dtype,
                                                           int rows, int chunk_rows,
                                                           float* __restrict__ part) {
  const int64_t gi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // sub-vector column
  const int mc = blockIdx.y;
  const int rb = blockIdx.z * kGenericRowBlock;
  if (gi >= g.gpr) return;
  const int64_t M = g.rows, N = g.cols;
  float acc[kGenericRowBlock][V];
#pragma unroll
  for (int i = 0; i < kGenericRowBlock; ++i)
#pragma unroll
    for (int j = 0; j < V; ++j) acc[i][j] = 0.f;
  const int64_t m_end = min((int64_t)(mc + 1) * chunk_rows, M);
  for (int64_t m = (int64_t)mc * chunk_rows; m < m_end; ++m) {
    const int64_t s = m * g.gpr + gi;
    const int region = region_of(g, s);
    float w[V];
#pragma unroll
    for (int j = 0; j < V; ++j) w[j] = 0.0f;
    for (int r = 0; r < g.R; ++r) {
      const uint32_t c = code_at(g, codes, r, s);
      const CB* e = books + ((int64_t)(r * g.n_regions + region) * g.K + c) * V;
#pragma unroll
      for (int j = 0; j < V; ++j) w[j] = __fadd_rn(w[j], to_f32<CB>(e[j]));
    }
#pragma unroll
    for (int i = 0; i < kGenericRowBlock; ++i) {
      if (rb + i < rows) {
        const float xv = load_as_f32(x, x_dtype, (int64_t)(rb + i) * M + m);
#pragma unroll
        for (int j = 0; j < V; ++j) acc[i][j] = fmaf(xv, w[j], acc[i][j]);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < kGenericRowBlock; ++i)
    if (rb + i < rows)
#pragma unroll
      for (int j = 0; j < V; ++j) part[((int64_t)mc * rows + rb + i) * N + gi * V + j] = acc[i][j];
}

__global__ void __launch_bounds__(256) reduce_parts_kernel(const float* __restrict__ part, int n_parts,
                                                           int64_t n_out, void* __restrict__ y, int y_dtype) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < n_out; o += stride) {
    float s = 0.f;
    for (int p = 0; p < n_parts; ++p) s += part[(int64_t)p * n_out + o];
    store_from_f32(y, y_dtype, o, s);
  }
}

// ---------------------------------------------------------------------------
// dispatch

struct FastPlan {
  bool ok = false;
  int V = 0, cbytes = 0, R = 0, WG = 1;
  bool tile = false;
  int n_sh = 0, f = 1, n_cblk = 0, n_chunks = 0;
  size_t smem = 0;
};

static FastPlan plan_fast(const Geom& g, const VqbTensor* t, int rows, int x_dtype, const VqbLaunch* L) {
  FastPlan p;
  if (L && (L->flags & VQB_FLAG_FORCE_GENERIC)) return p;
  if (t->layout != VQB_LAYOUT_GEMV_IL || t->codebook_dtype != VQB_F16 || x_dtype != VQB_F16) return p;
  if (!(rows == 1 || rows == 2 || rows == 4 || rows == 8)) return p;
  if (!(g.v == 4 || g.v == 8) || g.R > 2) return p;
  if (!(g.bits == 8 || g.bits == 16)) return p;
  if (g.bits == 16 && g.R != 1) return p;
  p.V = g.v;
  p.cbytes = g.code_bytes;
  p.R = g.R;
  p.WG = (g.v == 4) ? 2 : 1;
  const int cols_per_cta = 32 * p.WG * g.v;
  if (g.rows % kChunkRows != 0 || g.cols % cols_per_cta != 0) return p;
  if (g.sharing == VQB_SHARE_TILE) {
    if (g.tile_rows % kChunkRows != 0 || g.tile_cols % cols_per_cta != 0) return p;
    p.tile = true;
  } else if (g.sharing != VQB_SHARE_WHOLE) {
    return p;
  }
  int n_sh = (L && L->n_shared > 0) ? L->n_shared : 256;
  n_sh = std::min(n_sh, g.K);
  n_sh = std::min(n_sh, 1024 / g.R);
  p.n_sh = n_sh;
  p.n_cblk = (int)(g.cols / cols_per_cta);
  p.n_chunks = (int)(g.rows / kChunkRows);
  int f = 0;
  if (L && L->split_factor > 0 && (L->split_axis == 'M' || L->split_axis == 0) &&
      p.n_chunks % L->split_factor == 0)
    f = L->split_factor;
  if (f == 0) {
    const int want = 2 * sm_count();
    f = p.n_chunks;
    for (int d = 1; d <= p.n_chunks; ++d)
      if (p.n_chunks % d == 0 && p.n_cblk * d >= want) { f = d; break; }
  }
  p.f = f;
  const int WM = 8 / p.WG;
  p.smem = (size_t)p.R * p.n_sh * 128 + (size_t)WM * rows * cols_per_cta * sizeof(float);
  p.ok = true;
  return p;
}

static int64_t align256(int64_t x) { return (x + 255) & ~int64_t(255); }

static int64_t fast_ws_bytes(const FastPlan& p, const Geom& g, int rows) {
  if (!p.ok) return 0;
  return align256((int64_t)p.n_cblk * sizeof(int)) + (p.f > 1 ? (int64_t)p.f * rows * g.cols * 4 : 0);
}

static int generic_chunk_rows(const Geom& g) { return g.rows > 4096 ? 512 : 256; }

static int64_t generic_ws_bytes(const Geom& g, int rows) {
  const int64_t n_mc = ceil_div(g.rows, generic_chunk_rows(g));
  return n_mc * rows * g.cols * 4;
}

template <int V, int CBYTES, int R, int WG, bool TILE>
static int launch_fast_t(const FastPlan& p, GemvFastArgs& a, int rows, cudaStream_t st, int grid_limit) {
  auto pick = [&](auto kernel) -> int {
    static bool configured[64] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    if (p.smem > 48 * 1024 && !configured[dev & 63]) {
      VQB_CUDA_CHECK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      configured[dev & 63] = true;
    }
    int occ = 0;
    VQB_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kGemvThreads, p.smem));
    if (occ < 1) return set_error(VQB_ECAPACITY, "GEMV plan (n_shared=%d) does not fit one CTA per SM", p.n_sh);
    int grid = std::min(p.n_cblk * p.f, occ * sm_count());
    if (grid_limit > 0) grid = std::min(grid, grid_limit);
    kernel<<<grid, kGemvThreads, p.smem, st>>>(a);
    VQB_LAUNCH_CHECK("gemv_fast_kernel");
    set_kernel("gemv_fast");
    return VQB_OK;
  };
  switch (rows) {
    case 1: return pick(gemv_fast_kernel<V, CBYTES, R, 1, WG, TILE>);
    case 2: return pick(gemv_fast_kernel<V, CBYTES, R, 2, WG, TILE>);
    case 4: return pick(gemv_fast_kernel<V, CBYTES, R, 4, WG, TILE>);
    default: return pick(gemv_fast_kernel<V, CBYTES, R, 8, WG, TILE>);
  }
}

static int launch_fast(const FastPlan& p, GemvFastArgs& a, int rows, cudaStream_t st, int grid_limit) {
  // (V, code bytes, R, WG, tile-shared) combinations covering the BASELINE configs
  if (p.V == 8 && p.cbytes == 2 && p.R == 1 && !p.tile) return launch_fast_t<8, 2, 1, 1, false>(p, a, rows, st, grid_limit);
  if (p.V == 8 && p.cbytes == 1 && p.R == 2 && !p.tile) return launch_fast_t<8, 1, 2, 1, false>(p, a, rows, st, grid_limit);
  if (p.V == 8 && p.cbytes == 1 && p.R == 1 && !p.tile) return launch_fast_t<8, 1, 1, 1, false>(p, a, rows, st, grid_limit);
  if (p.V == 4 && p.cbytes == 1 && p.R == 1 && p.tile) return launch_fast_t<4, 1, 1, 2, true>(p, a, rows, st, grid_limit);
  if (p.V == 4 && p.cbytes == 1 && p.R == 1 && !p.tile) return launch_fast_t<4, 1, 1, 2, false>(p, a, rows, st, grid_limit);
  if (p.V == 8 && p.cbytes == 1 && p.R == 1 && p.tile) return launch_fast_t<8, 1, 1, 1, true>(p, a, rows, st, grid_limit);
  return set_error(VQB_ECONFIG, "no fast GEMV instance for this configuration");
}

static bool has_fast_instance(const FastPlan& p) {
  return (p.V == 8 && p.cbytes == 2 && p.R == 1 && !p.tile) || (p.V == 8 && p.cbytes == 1 && p.R == 2 && !p.tile) ||
         (p.V == 8 && p.cbytes == 1 && p.R == 1) || (p.V == 4 && p.cbytes == 1 && p.R == 1);
}

int gemv_dispatch(const VqbTensor* w, const void* x, int x_dtype, int rows, void* y, int y_dtype,
                  const VqbLaunch* L, void* ws, size_t ws_bytes, cudaStream_t st, bool* used_fast) {
  Geom g;
  int s = make_geom(w, &g);
  if (s) return s;
  if (g.ndim != 2) return set_error(VQB_ESHAPE, "quantized weight must be 2-D (M, N), got rank %d", g.ndim);
  if (rows < 1) return set_error(VQB_ESHAPE, "activation rows must be >= 1, got %d", rows);
  if (x_dtype < VQB_F32 || x_dtype > VQB_BF16 || y_dtype < VQB_F32 || y_dtype > VQB_BF16)
    return set_error(VQB_ECONFIG, "unknown activation/output dtype");
  FastPlan p = plan_fast(g, w, rows, x_dtype, L);
  if (p.ok && !has_fast_instance(p)) p.ok = false;
  if (used_fast) *used_fast = p.ok;
  if (p.ok) {
    const int64_t need = fast_ws_bytes(p, g, rows);
    if ((int64_t)ws_bytes < need || (need > 0 && !ws))
      return set_error(VQB_ECAPACITY, "GEMV workspace too small: %zu < %lld", ws_bytes, (long long)need);
    GemvFastArgs a;
    a.codes = reinterpret_cast<const uint8_t*>(w->d_codes);
    a.level_bytes = g.S * g.code_bytes;
    a.books = reinterpret_cast<const __half*>(w->d_codebooks);
    a.x = reinterpret_cast<const __half*>(x);
    a.y = y;
    a.y_dtype = y_dtype;
    a.counters = reinterpret_cast<int*>(ws);
    a.part = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ws) + align256((int64_t)p.n_cblk * sizeof(int)));
    a.M = (int)g.rows;
    a.N = (int)g.cols;
    a.G = (int)g.gpr;
    a.K = g.K;
    a.n_regions = g.n_regions;
    a.tile_rows = g.tile_rows;
    a.tile_cols = g.tile_cols;
    a.n_tc = g.sharing == VQB_SHARE_TILE ? (int)ceil_div(g.cols, g.tile_cols) : 1;
    a.f = p.f;
    a.chunks_per_part = p.n_chunks / p.f;
    a.n_cblk = p.n_cblk;
    a.n_sh = p.n_sh;
    return launch_fast(p, a, rows, st, L ? L->grid_limit : 0);
  }
  // generic: per-chunk partials then an ordered reduction
  const int chunk_rows = generic_chunk_rows(g);
  const int n_mc = (int)ceil_div(g.rows, chunk_rows);
  const int64_t need = generic_ws_bytes(g, rows);
  if ((int64_t)ws_bytes < need || !ws)
    return set_error(VQB_ECAPACITY, "GEMV workspace too small: %zu < %lld", ws_bytes, (long long)need);
  float* part = reinterpret_cast<float*>(ws);
  dim3 grid((unsigned)ceil_div(g.gpr, 128), (unsigned)n_mc, (unsigned)ceil_div(rows, kGenericRowBlock));
  if (grid.z > 65535) return set_error(VQB_ESHAPE, "too many activation rows for the generic GEMV (%d)", rows);
#define VQB_GEN(CBT, VV) \
  gemv_generic_kernel<CBT, VV><<<grid, 128, 0, st>>>(g, w->d_codes, reinterpret_cast<const CBT*>(w->d_codebooks), x, x_dtype, rows, chunk_rows, part)
#define VQB_GEN_V(CBT)                    \
  switch (g.v) {                          \
    case 2: VQB_GEN(CBT, 2); break;       \
    case 4: VQB_GEN(CBT, 4); break;       \
    case 8: VQB_GEN(CBT, 8); break;       \
    default: VQB_GEN(CBT, 16); break;     \
  }
  if (w->codebook_dtype == VQB_F32) { VQB_GEN_V(float) }
  else if (w->codebook_dtype == VQB_F16) { VQB_GEN_V(__half) }
  else { VQB_GEN_V(__nv_bfloat16) }
#undef VQB_GEN_V
#undef VQB_GEN
  VQB_LAUNCH_CHECK("gemv_generic_kernel");
  const int64_t n_out = (int64_t)rows * g.cols;
  int64_t blocks = std::min<int64_t>(ceil_div(n_out, 256), (int64_t)sm_count() * 8);
  reduce_parts_kernel<<<(unsigned)std::max<int64_t>(blocks, 1), 256, 0, st>>>(part, n_mc, n_out, y, y_dtype);
  VQB_LAUNCH_CHECK("reduce_parts_kernel");
  set_kernel("gemv_generic");
  return VQB_OK;
}

int64_t gemv_ws_bytes(const VqbTensor* w, int64_t rows, const VqbLaunch* L) {
  Geom g;
  int s = make_geom(w, &g);
  if (s) return s;
  FastPlan p = plan_fast(g, w, (int)rows, VQB_F16, L);
  int64_t a = (p.ok && has_fast_instance(p)) ? fast_ws_bytes(p, g, (int)rows) : 0;
  return std::max(a, generic_ws_bytes(g, (int)rows));
}

int gemv_usage(VqbUsage* u) {
  cudaFuncAttributes at;
  auto k = gemv_fast_kernel<8, 2, 1, 1, 1, false>;
  VQB_CUDA_CHECK(cudaFuncGetAttributes(&at, k));
  const size_t smem = 256 * 128 + 8 * 1 * 256 * 4;
  u->shared_bytes = (int)(at.sharedSizeBytes + smem);
  u->regs_per_thread = at.numRegs;
  u->threads_per_block = kGemvThreads;
  int occ = 0;
  VQB_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, kGemvThreads, smem));
  u->max_blocks_per_sm = occ;
  return VQB_OK;
}

}  // namespace vqb

extern "C" int vqb_gemv(const VqbTensor* w, const void* d_x, int32_t x_dtype, int32_t rows, void* d_y,
                        int32_t y_dtype, const VqbLaunch* launch, void* d_ws, size_t ws_bytes, void* stream) {
  return vqb::gemv_dispatch(w, d_x, x_dtype, rows, d_y, y_dtype, launch, d_ws, ws_bytes,
                            reinterpret_cast<cudaStream_t>(stream), nullptr);
}
