// gemv.cu — fused VQ dequantisation + decode GEMV, y(rows, N) = x(rows, M) @ W.
//
// Replaces SimMachine._matmul/_mm_block (pkg/src/vqforge/sim.py:697-775) for
// ComputeOp.gemv (dataflow.py:73-75); the numerics the reference checks are
// reference_compute's `a @ dequantize(W)` (sim.py:136-144) within 1e-4 rel-to-max
// (verify.py:200-215).
//
// Fast kernel (B200 design):
//  * TMA-staged index stream — a producer warp streams each work unit's codes
//    (GEMV_IL layout: 512-byte contiguous row-group segments) into a 4-stage
//    shared-memory ring with cp.async.bulk + mbarrier transaction counts, so a
//    CTA keeps up to 64 KB of code loads in flight independent of registers;
//    consumer warps read their 16-byte code words from shared memory.
//  * codebook cache — the first n_shared entries of every codebook a CTA needs
//    live in shared memory REPLICATED 128/EB times (EB = entry bytes): entry e
//    owns one 128-byte bank row and lane l reads replica (l mod 128/EB), so a
//    warp-wide random gather is conflict-free by construction (the 8 lanes of an
//    LDS.128 quarter-warp / 16 lanes of an LDS.64 half-warp always hit distinct
//    bank groups). Entries >= n_shared come from the global/L2 tier; when the
//    tensor's max code is known to be < n_shared the global tier is compiled out.
//  * codebook-centric dataflow — work units are (column block of 32*WG
//    sub-vector columns, 256-row chunk); a tile-shared book (GPTVQ) covers whole
//    chunks, the next region's book is prefetched while the current chunk
//    computes; whole-tensor books are loaded once per persistent CTA.
//  * persistent CTAs own contiguous unit ranges and accumulate consecutive
//    chunks of a column block in registers; spans that do not cover a whole
//    column block leave a partial that the last arriving CTA sums in chunk order
//    (deterministic, like the reference's ordered split reduction, sim.py:735).
//  * programmatic dependent launch — the code stream and the codebook fill start
//    before griddepcontrol.wait, overlapping the previous kernel's tail; x, y and
//    the workspace are only touched after it.
//  * register-level fusion — a lane owns one sub-vector column and multiplies
//    the looked-up fp16 entry straight into fp32 accumulators with the sm_100
//    mixed-precision FMA (fma.rn.f32.f16): no staging, no shuffles.
//
// Generic kernel: any VQConfig / sharing / layout / dtype, fp32 math on the
// bit-exact dequantised W, used for parity mode (fp32 codebooks) and for
// configurations outside the fast table.
#include <mutex>
#include <unordered_map>

#include "common.cuh"

namespace vqb {

constexpr int kConsumerWarps = 16;
constexpr int kConsumers = kConsumerWarps * 32;
constexpr int kGemvThreads = kConsumers + 32;  // + one producer warp
constexpr int kChunkRows = 256;
constexpr int kStages = 4;
constexpr uint16_t kHalfOne = 0x3C00;  // fp16 1.0
// bytes of one work unit's codes (= one ring stage): R levels x 256 rows x 32*WG columns
__host__ __device__ constexpr int stage_bytes(int R, int cbytes, int WG) { return R * cbytes * WG * kChunkRows * 32; }

struct GemvFastArgs {
  const uint8_t* codes;   // GEMV_IL, level r at codes + r * level_bytes
  int64_t level_bytes;
  const __half* books;    // (R*n_regions, K, V)
  const __half* x;        // (B, M)
  void* y;
  int y_dtype;
  float* part;            // (n_cblk * n_chunks, B, COLS) span partials
  int* span_len;          // (n_cblk * n_chunks) chunks covered by the partial at that slot
  int* counters;          // (n_cblk) chunks reduced so far
  int M, N, G, K, n_regions;
  int tile_rows, tile_cols, n_tc;
  int n_chunks, n_cblk, n_sh;
};

template <int V, int CBYTES, int R, int B, int WG, bool TILE, bool GTIER, bool H2>
__global__ void __launch_bounds__(kGemvThreads) gemv_fast_kernel(GemvFastArgs a) {
  constexpr int EB = V * 2;              // fp16 entry bytes
  constexpr int REP = 128 / EB;          // replicas per bank row
  constexpr int RPL = 16 / CBYTES;       // rows per 16-byte code word
  constexpr int WM = kConsumerWarps / WG;  // warps along M
  constexpr int RW = kChunkRows / WM;    // rows per warp per chunk
  constexpr int LOADS = RW / RPL;        // code words per lane per level per chunk
  constexpr int COLS = 32 * WG * V;      // output columns per column block
  constexpr int NSEG = kChunkRows / RPL; // row-group segments per level per unit
  constexpr int SEGB = 32 * WG * 16;     // bytes per segment
  constexpr int LEVB = NSEG * SEGB;      // bytes per level per unit
  constexpr int NBUF = TILE ? 2 : 1;     // codebook buffers
  static_assert(LOADS >= 1 && RW % 8 == 0, "bad tiling");
  constexpr int STAGEB = R * LEVB;
  static_assert(STAGEB == stage_bytes(R, CBYTES, WG), "stage size");
  static_assert(NSEG <= 32, "one segment per producer lane");

  extern __shared__ __align__(1024) uint8_t smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint8_t* stages = smem;                                        // kStages x STAGEB
  uint8_t* books_s = smem + kStages * STAGEB;                    // NBUF x R x n_sh x 128
  const size_t book_bytes = (size_t)R * a.n_sh * 128;
  float* red = reinterpret_cast<float*>(books_s + NBUF * book_bytes);  // WM * COLS
  uint64_t* bars = reinterpret_cast<uint64_t*>(red + WM * COLS);       // full[kStages], empty[kStages]
  int* s_last = reinterpret_cast<int*>(bars + 2 * kStages);
  const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + kStages);

  const int U = a.n_cblk * a.n_chunks;
  const int u0 = (int)((int64_t)blockIdx.x * U / gridDim.x);
  const int u1 = (int)((int64_t)(blockIdx.x + 1) * U / gridDim.x);

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, kConsumerWarps);
    }
    mbar_fence_init();
  }
  __syncthreads();
  pdl_launch_dependents();

  if (warp == kConsumerWarps) {
    // ===== producer: stream each unit's code segments into the stage ring =====
    for (int idx = 0; idx < u1 - u0; ++idx) {
      const int u = u0 + idx;
      const int cblk = u / a.n_chunks, chunk = u - cblk * a.n_chunks;
      const int s = idx % kStages;
      if (idx >= kStages) mbar_wait(empty0 + 8 * s, ((idx / kStages) + 1) & 1);
      if (lane == 0) mbar_arrive_expect_tx(full0 + 8 * s, STAGEB);
      __syncwarp();
      if (lane < NSEG) {
        const int64_t rg = (int64_t)chunk * NSEG + lane;  // row-group index along M
#pragma unroll
        for (int r = 0; r < R; ++r)
          tma_load_1d(smem_u32(stages + s * STAGEB + r * LEVB + lane * SEGB),
                      a.codes + r * a.level_bytes + (rg * a.G + (int64_t)cblk * 32 * WG) * 16, SEGB,
                      full0 + 8 * s);
      }
    }
    return;
  }

  // ===== consumers =====
  const int wm = warp / WG, wg = warp % WG;
  const uint32_t rep_off = (uint32_t)(lane % REP) * EB;

  constexpr int MAX_PER_THREAD = (1024 + kConsumers - 1) / kConsumers;  // n_sh * R <= 1024 entries
  auto book_issue = [&](int region, uint4 (&buf)[MAX_PER_THREAD]) {
#pragma unroll
    for (int k = 0; k < MAX_PER_THREAD; ++k) {
      const int idx = tid + k * kConsumers;
      if (idx < R * a.n_sh) {
        const int r = idx / a.n_sh, e = idx - r * a.n_sh;
        const uint8_t* src = reinterpret_cast<const uint8_t*>(a.books) +
                             (((int64_t)(r * a.n_regions + region) * a.K) + e) * EB;
        if constexpr (EB == 16) buf[k] = __ldg(reinterpret_cast<const uint4*>(src));
        else {
          const uint2 t = __ldg(reinterpret_cast<const uint2*>(src));
          buf[k] = make_uint4(t.x, t.y, 0, 0);
        }
      }
    }
  };
  auto book_commit = [&](int bufi, const uint4 (&buf)[MAX_PER_THREAD]) {
#pragma unroll
    for (int k = 0; k < MAX_PER_THREAD; ++k) {
      const int idx = tid + k * kConsumers;
      if (idx < R * a.n_sh) {
        const int r = idx / a.n_sh, e = idx - r * a.n_sh;
        uint8_t* row = books_s + bufi * book_bytes + ((size_t)r * a.n_sh + e) * 128;
#pragma unroll
        for (int q = 0; q < REP; ++q) {
          uint8_t* d = row + ((q + e) % REP) * EB;  // rotate so 8/16 threads hit distinct banks
          if constexpr (EB == 16) *reinterpret_cast<uint4*>(d) = buf[k];
          else *reinterpret_cast<uint2*>(d) = make_uint2(buf[k].x, buf[k].y);
        }
      }
    }
  };
  auto csync = [&]() { named_bar_sync(1, kConsumers); };

  if constexpr (!TILE) {
    uint4 bb[MAX_PER_THREAD];
    book_issue(0, bb);
    book_commit(0, bb);
  }
  pdl_wait();  // x / y / workspace may belong to the previous kernel
  csync();

  int idx = 0;
  int cur_buf = 0;
  for (int u = u0; u < u1;) {
    const int cblk = u / a.n_chunks;
    const int c0 = u - cblk * a.n_chunks;
    const int c1 = min(a.n_chunks, c0 + (u1 - u));
    const int g_local = wg * 32 + lane;
    const int col_tile = TILE ? (cblk * COLS) / a.tile_cols : 0;
    auto region_of_chunk = [&](int chunk) {
      return TILE ? (chunk * kChunkRows / a.tile_rows) * a.n_tc + col_tile : 0;
    };
    if constexpr (TILE) {
      uint4 bb[MAX_PER_THREAD];
      book_issue(region_of_chunk(c0), bb);
      csync();  // the previous span is done with both buffers
      book_commit(0, bb);
      cur_buf = 0;
      csync();
    }

    float acc[B][V];
#pragma unroll
    for (int b = 0; b < B; ++b)
#pragma unroll
      for (int j = 0; j < V; ++j) acc[b][j] = 0.f;

    for (int chunk = c0; chunk < c1; ++chunk, ++idx) {
      const int s = idx % kStages;
      uint4 nb[MAX_PER_THREAD];
      bool sw = false;
      if constexpr (TILE) {
        sw = (chunk + 1 < c1) && region_of_chunk(chunk + 1) != region_of_chunk(chunk);
        if (sw) book_issue(region_of_chunk(chunk + 1), nb);
      }
      mbar_wait(full0 + 8 * s, (idx / kStages) & 1);
      const uint8_t* st = stages + s * STAGEB;
      const uint8_t* bsm = books_s + cur_buf * book_bytes + rep_off;
      const int region = region_of_chunk(chunk);
      const int m0 = chunk * kChunkRows + wm * RW;
#pragma unroll
      for (int i = 0; i < LOADS; ++i) {
        uint4 cw[R];
#pragma unroll
        for (int r = 0; r < R; ++r)
          cw[r] = *reinterpret_cast<const uint4*>(st + r * LEVB + (wm * LOADS + i) * SEGB + g_local * 16);
        uint4 xv[B][RPL / 8];
#pragma unroll
        for (int b = 0; b < B; ++b)
#pragma unroll
          for (int q = 0; q < RPL / 8; ++q)
            xv[b][q] = __ldg(reinterpret_cast<const uint4*>(a.x + (int64_t)b * a.M + m0 + i * RPL) + q);
        uint32_t hw[B][V / 2];  // fp16x2 window accumulators (H2 path)
#pragma unroll
        for (int b = 0; b < B; ++b)
#pragma unroll
          for (int j = 0; j < V / 2; ++j) hw[b][j] = 0u;
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
              const uint32_t w = (&cw[r].x)[k / 2];
              code = (k & 1) ? (w >> 16) : (w & 0xffff);
            } else {
              const uint32_t w = (&cw[r].x)[k / 4];
              code = (w >> (8 * (k % 4))) & 0xff;
            }
            bool in_smem = true;
            if constexpr (GTIER) in_smem = code < (uint32_t)a.n_sh;
            uint32_t e[V / 2];
            const uint8_t* src = in_smem ? bsm + (size_t)r * a.n_sh * 128 + ((size_t)code << 7)
                                         : reinterpret_cast<const uint8_t*>(a.books) +
                                               (((int64_t)(r * a.n_regions + region) * a.K) + code) * EB;
            if constexpr (EB == 16) {
              const uint4 q = in_smem ? *reinterpret_cast<const uint4*>(src) : __ldg(reinterpret_cast<const uint4*>(src));
              e[0] = q.x; e[1] = q.y; e[2] = q.z; e[3] = q.w;
            } else {
              const uint2 q = in_smem ? *reinterpret_cast<const uint2*>(src) : __ldg(reinterpret_cast<const uint2*>(src));
              e[0] = q.x; e[1] = q.y;
            }
            if constexpr (H2) {
              // packed fp16x2 FMA into an 8-row fp16 window (full-rate HFMA2; the
              // mixed-precision FHFMA issues at a quarter of that rate on sm_100)
#pragma unroll
              for (int b = 0; b < B; ++b) {
                const uint32_t x2 = (uint32_t)xh[b] * 0x10001u;
#pragma unroll
                for (int j = 0; j < V / 2; ++j) hw[b][j] = hfma2(e[j], x2, hw[b][j]);
              }
            } else {
#pragma unroll
              for (int b = 0; b < B; ++b)
#pragma unroll
                for (int j = 0; j < V / 2; ++j) {
                  acc[b][2 * j] = fma_h((uint16_t)(e[j] & 0xffff), xh[b], acc[b][2 * j]);
                  acc[b][2 * j + 1] = fma_h((uint16_t)(e[j] >> 16), xh[b], acc[b][2 * j + 1]);
                }
            }
          }
          if constexpr (H2) {
            if ((k & 7) == 7) {  // flush the window into the fp32 accumulators (exact widening)
#pragma unroll
              for (int b = 0; b < B; ++b)
#pragma unroll
                for (int j = 0; j < V / 2; ++j) {
                  acc[b][2 * j] = fma_h((uint16_t)(hw[b][j] & 0xffff), kHalfOne, acc[b][2 * j]);
                  acc[b][2 * j + 1] = fma_h((uint16_t)(hw[b][j] >> 16), kHalfOne, acc[b][2 * j + 1]);
                  hw[b][j] = 0u;
                }
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty0 + 8 * s);
      if constexpr (TILE) {
        if (sw) {
          book_commit(cur_buf ^ 1, nb);
          csync();
          cur_buf ^= 1;
        }
      }
    }

    // ---- reduce the WM row-slabs of this span in a fixed order, one batch row at a time
    const int n0 = cblk * COLS;
    const bool whole = (c0 == 0 && c1 == a.n_chunks);
    const int slot = cblk * a.n_chunks + c0;
#pragma unroll
    for (int b = 0; b < B; ++b) {
#pragma unroll
      for (int j = 0; j < V; ++j) red[(size_t)wm * COLS + g_local * V + j] = acc[b][j];
      csync();
      for (int col = tid; col < COLS; col += kConsumers) {
        float sum = 0.f;
#pragma unroll
        for (int w = 0; w < WM; ++w) sum += red[(size_t)w * COLS + col];
        if (whole) store_from_f32(a.y, a.y_dtype, (int64_t)b * a.N + n0 + col, sum);
        else a.part[((int64_t)slot * B + b) * COLS + col] = sum;
      }
      csync();
    }
    if (!whole) {
      if (tid == 0) a.span_len[slot] = c1 - c0;
      __threadfence();
      csync();
      if (tid == 0) *s_last = (atomicAdd(a.counters + cblk, c1 - c0) + (c1 - c0) == a.n_chunks);
      csync();
      if (*s_last) {
        __threadfence();
        for (int o = tid; o < B * COLS; o += kConsumers) {
          const int b = o / COLS, col = o - (o / COLS) * COLS;
          float sum = 0.f;
          for (int c = 0; c < a.n_chunks;) {
            const int sl = cblk * a.n_chunks + c;
            sum += __ldcg(a.part + (int64_t)sl * B * COLS + o);
            c += __ldcg(a.span_len + sl);
          }
          store_from_f32(a.y, a.y_dtype, (int64_t)b * a.N + n0 + col, sum);
        }
        if (tid == 0) a.counters[cblk] = 0;  // self-reset for the next launch
      }
    }
    csync();  // red / s_last reuse by the next span
    u += c1 - c0;
  }
}

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
  bool tile = false, gtier = true, h2 = true;
  int n_sh = 0, n_cblk = 0, n_chunks = 0;
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
  if (L && (L->flags & VQB_FLAG_NO_SHARED)) n_sh = 0;
  p.n_sh = n_sh;
  p.gtier = !(t->max_code >= 0 && t->max_code < n_sh);
  p.h2 = !(L && (L->flags & VQB_FLAG_EXACT_ACCUM));
  p.n_cblk = (int)(g.cols / cols_per_cta);
  p.n_chunks = (int)(g.rows / kChunkRows);
  const int WM = kConsumerWarps / p.WG;
  p.smem = (size_t)kStages * stage_bytes(p.R, p.cbytes, p.WG) + (size_t)(p.tile ? 2 : 1) * p.R * p.n_sh * 128 +
           (size_t)WM * cols_per_cta * sizeof(float) + 2 * kStages * 8 + 16;
  p.ok = true;
  return p;
}

static int64_t align256(int64_t x) { return (x + 255) & ~int64_t(255); }

static int64_t fast_ws_bytes(const FastPlan& p, const Geom& g, int rows) {
  if (!p.ok) return 0;
  const int64_t slots = (int64_t)p.n_cblk * p.n_chunks;
  const int64_t cols = 32 * p.WG * p.V;
  return VQB_WS_COUNTER_BYTES + align256(slots * 4) + slots * rows * cols * 4;
}

static int generic_chunk_rows(const Geom& g) { return g.rows > 4096 ? 512 : 256; }

static int64_t generic_ws_bytes(const Geom& g, int rows) {
  const int64_t n_mc = ceil_div(g.rows, generic_chunk_rows(g));
  return VQB_WS_COUNTER_BYTES + n_mc * rows * g.cols * 4;
}

typedef void (*GemvKernel)(GemvFastArgs);

static int launch_gemv_kernel(GemvKernel kernel, const FastPlan& p, const GemvFastArgs& a, cudaStream_t st,
                              const VqbLaunch* L) {
  static std::mutex mu;
  static std::unordered_map<const void*, int> occ_cache;  // kernel x smem -> occupancy
  int occ = 0;
  {
    std::lock_guard<std::mutex> lock(mu);
    int dev = 0;
    cudaGetDevice(&dev);
    const void* key = reinterpret_cast<const void*>(
        reinterpret_cast<uintptr_t>(kernel) ^ ((uintptr_t)p.smem << 20) ^ ((uintptr_t)dev << 56));
    auto it = occ_cache.find(key);
    if (it == occ_cache.end()) {
      // always opt in: static shared memory pushes even a 48 KB dynamic request over the default
      VQB_CUDA_CHECK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448));
      VQB_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kGemvThreads, p.smem));
      occ_cache[key] = occ;
    } else {
      occ = it->second;
    }
  }
  if (occ < 1) return set_error(VQB_ECAPACITY, "GEMV plan (n_shared=%d) does not fit one CTA per SM", p.n_sh);
  int grid = std::min(p.n_cblk * p.n_chunks, occ * sm_count());
  if (L && L->grid_limit > 0) grid = std::min(grid, L->grid_limit);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kGemvThreads);
  cfg.dynamicSmemBytes = p.smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (L && (L->flags & VQB_FLAG_NO_PDL)) ? 0 : 1;
  VQB_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kernel, a));
  set_kernel("gemv_fast");
  return VQB_OK;
}

template <int V, int CBYTES, int R, int WG, bool TILE>
static GemvKernel pick_kernel(int rows, bool gtier, bool h2) {
#define VQB_K(B)                                                                        \
  (gtier ? (h2 ? gemv_fast_kernel<V, CBYTES, R, B, WG, TILE, true, true>                  \
               : gemv_fast_kernel<V, CBYTES, R, B, WG, TILE, true, false>)                \
         : (h2 ? gemv_fast_kernel<V, CBYTES, R, B, WG, TILE, false, true>                 \
               : gemv_fast_kernel<V, CBYTES, R, B, WG, TILE, false, false>))
  switch (rows) {
    case 1: return VQB_K(1);
    case 2: return VQB_K(2);
    case 4: return VQB_K(4);
    default: return VQB_K(8);
  }
#undef VQB_K
}

static GemvKernel fast_kernel_for(const FastPlan& p, int rows) {
  // (V, code bytes, R, WG, tile-shared) combinations covering the BASELINE configs
  if (p.V == 8 && p.cbytes == 2 && p.R == 1 && !p.tile) return pick_kernel<8, 2, 1, 1, false>(rows, p.gtier, p.h2);
  if (p.V == 8 && p.cbytes == 1 && p.R == 2 && !p.tile) return pick_kernel<8, 1, 2, 1, false>(rows, p.gtier, p.h2);
  if (p.V == 8 && p.cbytes == 1 && p.R == 1 && !p.tile) return pick_kernel<8, 1, 1, 1, false>(rows, p.gtier, p.h2);
  if (p.V == 8 && p.cbytes == 1 && p.R == 1 && p.tile) return pick_kernel<8, 1, 1, 1, true>(rows, p.gtier, p.h2);
  if (p.V == 4 && p.cbytes == 1 && p.R == 1 && p.tile) return pick_kernel<4, 1, 1, 2, true>(rows, p.gtier, p.h2);
  if (p.V == 4 && p.cbytes == 1 && p.R == 1 && !p.tile) return pick_kernel<4, 1, 1, 2, false>(rows, p.gtier, p.h2);
  return nullptr;
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
  GemvKernel kernel = p.ok ? fast_kernel_for(p, rows) : nullptr;
  if (used_fast) *used_fast = kernel != nullptr;
  if (kernel) {
    const int64_t need = fast_ws_bytes(p, g, rows);
    if ((int64_t)ws_bytes < need || !ws)
      return set_error(VQB_ECAPACITY, "GEMV workspace too small: %zu < %lld", ws_bytes, (long long)need);
    const int64_t slots = (int64_t)p.n_cblk * p.n_chunks;
    if ((int64_t)p.n_cblk * 4 > VQB_WS_COUNTER_BYTES)
      return set_error(VQB_ECAPACITY, "too many GEMV column blocks (%d) for the counter region", p.n_cblk);
    uint8_t* wsb = reinterpret_cast<uint8_t*>(ws);
    GemvFastArgs a;
    a.codes = reinterpret_cast<const uint8_t*>(w->d_codes);
    a.level_bytes = g.S * g.code_bytes;
    a.books = reinterpret_cast<const __half*>(w->d_codebooks);
    a.x = reinterpret_cast<const __half*>(x);
    a.y = y;
    a.y_dtype = y_dtype;
    a.counters = reinterpret_cast<int*>(wsb);
    a.span_len = reinterpret_cast<int*>(wsb + VQB_WS_COUNTER_BYTES);
    a.part = reinterpret_cast<float*>(wsb + VQB_WS_COUNTER_BYTES + align256(slots * 4));
    a.M = (int)g.rows;
    a.N = (int)g.cols;
    a.G = (int)g.gpr;
    a.K = g.K;
    a.n_regions = g.n_regions;
    a.tile_rows = g.tile_rows;
    a.tile_cols = g.tile_cols;
    a.n_tc = g.sharing == VQB_SHARE_TILE ? (int)ceil_div(g.cols, g.tile_cols) : 1;
    a.n_chunks = p.n_chunks;
    a.n_cblk = p.n_cblk;
    a.n_sh = p.n_sh;
    return launch_gemv_kernel(kernel, p, a, st, L);
  }
  // generic: per-chunk partials then an ordered reduction
  const int chunk_rows = generic_chunk_rows(g);
  const int n_mc = (int)ceil_div(g.rows, chunk_rows);
  const int64_t need = generic_ws_bytes(g, rows);
  if ((int64_t)ws_bytes < need || !ws)
    return set_error(VQB_ECAPACITY, "GEMV workspace too small: %zu < %lld", ws_bytes, (long long)need);
  float* part = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ws) + VQB_WS_COUNTER_BYTES);
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
  int64_t a = (p.ok && fast_kernel_for(p, (int)rows)) ? fast_ws_bytes(p, g, (int)rows) : 0;
  return std::max(a, generic_ws_bytes(g, (int)rows));
}

int gemv_usage(VqbUsage* u) {
  cudaFuncAttributes at;
  auto k = gemv_fast_kernel<8, 2, 1, 1, 1, false, true, true>;
  VQB_CUDA_CHECK(cudaFuncGetAttributes(&at, k));
  const size_t smem = kStages * stage_bytes(1, 2, 1) + 256 * 128 + kConsumerWarps * 256 * 4 + 2 * kStages * 8 + 16;
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
