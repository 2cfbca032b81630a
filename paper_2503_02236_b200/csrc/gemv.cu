// gemv.cu — fused VQ dequantisation + decode GEMV, y(rows, N) = x(rows, M) @ W.
//
// Replaces SimMachine._matmul/_mm_block (pkg/src/vqforge/sim.py:697-775) for
// ComputeOp.gemv (dataflow.py:73-75); the numerics the reference checks are
// reference_compute's `a @ dequantize(W)` (sim.py:136-144) within 1e-4 rel-to-max
// (verify.py:200-215).
//
// Fast kernel (B200 design):
//  * TMA-staged index stream — the GEMV_IL layout is column-blocked (256 output
//    columns per block, row groups of 8/16 rows inside), so one block's 256-row
//    chunk is a single contiguous run: a producer warp streams each chunk with ONE
//    cp.async.bulk per level (+ one per activation row) into a 3-stage ring with
//    mbarrier transaction counts; consumer warps read 16-byte code words from it.
//  * codebook cache — the first n_shared entries of every codebook a CTA needs
//    live in shared memory REPLICATED 128/EB times (EB = entry bytes): entry e
//    owns one 128-byte bank row and lane l reads replica (l mod 128/EB), so a
//    warp-wide random gather is conflict-free by construction (the 8 lanes of an
//    LDS.128 quarter-warp / 16 lanes of an LDS.64 half-warp always hit distinct
//    bank groups). Entries >= n_shared come from the global/L2 tier; when the
//    tensor's max code is known to be < n_shared the global tier is compiled out.
//  * codebook-centric, persistent stream-K dataflow — one CTA per SM owns a
//    contiguous range of (column block, chunk) units (balanced to one unit); a
//    whole-tensor book is loaded once per CTA, a tile-shared book (GPTVQ) is
//    prefetched for the next unit while the current one computes. A column block
//    split across CTAs is finished by the CTA holding its first chunk, which adds
//    the later CTAs' published fp32 partials in chunk order (deterministic, like
//    the reference's ordered split reduction, sim.py:735).
//  * programmatic dependent launch — the code stream and the codebook fill start
//    before griddepcontrol.wait, overlapping the previous kernel's tail; x and y
//    are only touched after it.
//  * register-level fusion — a lane owns one sub-vector column and multiplies
//    the looked-up fp16 entry straight into fp32 accumulators with the sm_100
//    mixed-precision FMA (fma.rn.f32.f16): no staging, no shuffles.
//
// Generic kernel: any VQConfig / sharing / layout / dtype, fp32 math on the
// bit-exact dequantised W, used for parity mode (fp32 codebooks) and for
// configurations outside the fast table.
#include <algorithm>
#include <mutex>
#include <unordered_map>

#include "common.cuh"

namespace vqb {

// Every warp computes; thread 0 also feeds the TMA ring. 16 warps (one 512-thread
// CTA per SM) hide the shared-memory gather latency at batch 1-4; at batch 8 each
// looked-up entry feeds 8 FMAs, so 8 warps with more registers keep the B x V fp32
// accumulators in registers. Measured: 8 warps at batch 1 with two CTAs per SM (so
// the next launch's prologue could overlap this one's tail) is 6 % slower.
// The tensor-core path (batch 4-8) keeps 16 warps: its accumulators do not grow with B.
__host__ __device__ constexpr int gemv_warps(int B, bool mma = false) { return (B >= 8 && !mma) ? 8 : 16; }
// rows a warp handles per chunk: 32 (two 16-byte code words of u8 codes, four of u16).
// Measured: 8-row slabs double the per-chunk overhead; 16-row slabs leave half the
// code words in flight; 64-row slabs no longer fit the ring with the codebook.
__host__ __device__ constexpr int gemv_slab_rows(int cbytes) { return 32; }
constexpr uint16_t kHalfOne = 0x3C00;  // fp16 1.0
// chunk rows: the warps along M each take one 16-row slab (WG = warps across N)
// (the tensor-core path at batch 16 splits a column block's 16 column pairs over
// (B + 7) / 8 warps, so fewer warps run along M)
__host__ __device__ constexpr int gemv_chunk_rows(int WG, int B, int cbytes, bool mma = false) {
  return gemv_slab_rows(cbytes) * (gemv_warps(B, mma) / WG / (mma ? (B + 7) / 8 : 1));
}
// bytes of one chunk's codes: R levels x chunk rows x 32*WG columns
__host__ __device__ constexpr int stage_bytes(int R, int cbytes, int WG, int B, bool mma = false) {
  return R * cbytes * WG * gemv_chunk_rows(WG, B, cbytes, mma) * 32;
}
// a ring stage also carries the chunk's activations: B rows x chunk rows fp16
__host__ __device__ constexpr int stage_total(int R, int cbytes, int WG, int B, bool mma = false) {
  return stage_bytes(R, cbytes, WG, B, mma) + B * gemv_chunk_rows(WG, B, cbytes, mma) * 2;
}
// ring depth: ~96 KB of code loads in flight per SM (HBM latency x per-SM share of
// the bandwidth), 3..12 stages
__host__ __device__ constexpr int gemv_stages(int R, int cbytes, int WG, int B, bool mma = false) {
  return (98304 / stage_total(R, cbytes, WG, B, mma)) < 3    ? 3
         : (98304 / stage_total(R, cbytes, WG, B, mma)) > 12 ? 12
                                                             : 98304 / stage_total(R, cbytes, WG, B, mma);
}

struct GemvFastArgs {
  const uint8_t* codes;   // GEMV_IL (column-blocked), level r at codes + r * level_bytes
  int64_t level_bytes;
  const __half* books;    // (R*n_regions, K, V)
  const __half* x;        // (B, M)
  void* y;
  int y_dtype;
  int M, N, G, K, n_regions;
  int tile_rows, tile_cols, n_tc;
  int n_chunks, n_cblk, n_sh;
  unsigned long long* part;  // (grid, B, COLS) tagged partials {fp32 value, tag 1}, one slot per CTA,
                             // in the self-resetting workspace head (zeroed by the consumer)
  unsigned long long* trace;  // optional per-CTA phase timestamps (debug flag 32), 8 per CTA
  int n_reg;                  // register tier: entries [0, n_reg) held in registers (REGT kernels, <= 4)
  int total_units;            // grouped launch: units over every problem of the table
  int n_probs;                // grouped launch: problems in the table (0: the single problem above)
  // tensor-parallel push epilogue (vqb_gemv_tp; tp_world 0 = plain store into y): every
  // output element goes straight from the reducing CTA into each rank's symmetric
  // buffer over peer memory, then the grid's last CTA signals every rank (tp.cu)
  int tp_world, tp_rank, tp_mode;
  char* tp_peer[kTpMaxWorld];
  int64_t tp_slot_elems;
  // fused activation transform (XF kernels, vqb_gemv_xf; batch 1): the CTA builds the
  // whole transformed x in shared memory once instead of streaming x per unit.
  //  1 RMSNorm with residual: h = res_in + x (x may be null), res_out = h (CTA 0),
  //    x' = w * rmsnorm(h) (the rmsnorm_kernel arithmetic, decode.cu)
  //  2 SiLU gate: x' = silu(x[:M]) * x[M:2M] for x = [gate | up] (silu_mul_kernel)
  int xf_mode;
  int swiglu;  // XF kernels: W's 256-column blocks hold [gate 128 | up 128]; y = silu(gate) * up (N/2 columns)
  const __half* xf_add;  // RMSNorm: the input added to the residual (null: none)
  const __half* xf_res_in;
  __half* xf_res_out;
  const __half* xf_w;
  float xf_eps;
};

// One linear of a grouped launch (vqb_gemv_grouped): same VQ config and batch as
// every other problem of the launch, its own codes, codebook, x and y. Units of all
// problems form one stream-K range, so a step's independent GEMVs run as one
// persistent kernel with no per-launch prologue / tail.
struct GemvProblem {
  const uint8_t* codes;
  int64_t level_bytes;
  const __half* books;
  const __half* x;
  void* y;
  int M, N, n_cblk, n_chunks, unit_base, pad;
};
constexpr int kMaxGroup = 192;  // problems per grouped launch (kernel parameter table, 12 KB)
struct GemvTable {
  GemvProblem p[kMaxGroup];
};

// The problem a unit belongs to, seen through a forward-only cursor (CTAs walk
// their units in order). For a single-problem launch it never moves.
struct ProbCursor {
  const uint8_t* codes;
  int64_t level_bytes;
  const __half* books;
  const __half* x;
  void* y;
  int M, N, n_cblk, n_chunks, base, end, idx;
  int last_wb;  // sub-vector groups of the (possibly narrower) last column block
};

__device__ __forceinline__ void trace_at(unsigned long long* tr, int slot) {
  if (tr) tr[blockIdx.x * 8 + slot] = gtimer();
}
// Fused activation transform of the XF kernels (batch 1): every CTA computes the whole
// transformed activation row into shared memory (x is 8-22 KB and L2-resident, so the
// redundant reads cost less than a separate launch), with the exact arithmetic of the
// standalone kernels (decode.cu rmsnorm_kernel / silu_mul_kernel) so the fused and
// unfused decode steps agree bit for bit. `red` (>= THREADS/32 floats) is scratch.
template <int THREADS>
__device__ __forceinline__ void gemv_xf_preload(const GemvFastArgs& a, uint4 (&wv)[4]) {
  // the norm weight does not depend on the previous kernel: fetched before griddepcontrol.wait
  if (a.xf_mode != 1) return;
  int nv = 0;
  for (int i = threadIdx.x; i < a.M / 8 && nv < 4; i += THREADS, ++nv) wv[nv] = __ldg(reinterpret_cast<const uint4*>(a.xf_w) + i);
}

template <int THREADS>
__device__ __forceinline__ void gemv_xf_prologue(const GemvFastArgs& a, uint8_t* xres, float* red, const uint4 (&wv)[4]) {
  const int M = a.M, nvec = M / 8;
  uint4* xo = reinterpret_cast<uint4*>(xres);
  if (a.xf_mode == 2) {
    const __half* gu = a.x;
    for (int i = threadIdx.x; i < nvec; i += THREADS) {
      const uint4 gv = __ldg(reinterpret_cast<const uint4*>(gu) + i);
      const uint4 uv = __ldg(reinterpret_cast<const uint4*>(gu + M) + i);
      const __half* gp = reinterpret_cast<const __half*>(&gv);
      const __half* up = reinterpret_cast<const __half*>(&uv);
      uint4 o;
      __half* op = reinterpret_cast<__half*>(&o);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float g = __half2float(gp[j]);
        const __half sg = __float2half_rn(g / (1.0f + __expf(-g)));
        op[j] = __float2half_rn(__half2float(sg) * __half2float(up[j]));
      }
      xo[i] = o;
    }
    return;
  }
  // RMSNorm: the per-thread strided partial sums, warp then block reduction of
  // rmsnorm_kernel<THREADS> (same thread count, so the same float order)
  const __half* xr = a.xf_add;  // may be null (first layer: h = residual)
  float ss = 0.f;
  for (int i = threadIdx.x; i < nvec; i += THREADS) {
    uint4 h = __ldg(reinterpret_cast<const uint4*>(a.xf_res_in) + i);
    if (xr) {
      const uint4 av = __ldg(reinterpret_cast<const uint4*>(xr) + i);
      __half2* hp = reinterpret_cast<__half2*>(&h);
      const __half2* ap = reinterpret_cast<const __half2*>(&av);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = __half22float2(hp[j]), g = __half22float2(ap[j]);
        hp[j] = __floats2half2_rn(f.x + g.x, f.y + g.y);
      }
    }
    xo[i] = h;  // h for now; normalised in place below
    if (blockIdx.x == 0 && a.xf_res_out) reinterpret_cast<uint4*>(a.xf_res_out)[i] = h;
    const __half2* hp = reinterpret_cast<const __half2*>(&h);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 f = __half22float2(hp[j]);
      ss += f.x * f.x + f.y * f.y;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float t = threadIdx.x < THREADS / 32 ? red[threadIdx.x] : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) red[THREADS / 32] = t;
  }
  __syncthreads();
  const float inv = rsqrtf(red[THREADS / 32] / (float)M + a.xf_eps);
  int nv = 0;
  for (int i = threadIdx.x; i < nvec; i += THREADS, ++nv) {
    const uint4 h = xo[i];
    const uint4 wi = nv < 4 ? wv[nv] : __ldg(reinterpret_cast<const uint4*>(a.xf_w) + i);
    const __half2* hp = reinterpret_cast<const __half2*>(&h);
    const __half2* wp = reinterpret_cast<const __half2*>(&wi);
    uint4 o;
    __half2* op = reinterpret_cast<__half2*>(&o);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 f = __half22float2(hp[j]), ww = __half22float2(wp[j]);
      const float2 hf = __half22float2(__floats2half2_rn(f.x * inv, f.y * inv));
      op[j] = __floats2half2_rn(ww.x * hf.x, ww.y * hf.y);
    }
    xo[i] = o;
  }
}

// Persistent stream-K decode GEMV. Work units are (column block, chunk of CR rows),
// ordered column-block major; CTA i owns the contiguous unit range
// [i*U/grid, (i+1)*U/grid) and walks it as "spans" (maximal runs inside one column
// block), accumulating a span in registers. A span that covers its whole column
// block writes y. A column block split across CTAs is finished by the CTA holding
// its first chunk — for that CTA it is the last span of its range — which adds the
// later CTAs' fp32 partials (computed at the start of their ranges, so normally
// already published) in chunk order: deterministic, like the reference's ordered
// split reduction (sim.py:735), with no atomics and no extra launch.
// ACC selects the inner product: 0 exact fp32 (FHFMA, parity mode), 1 fp16x2 windows
// (HFMA2, batch 1-2), 2 tensor cores (mma.sync m16n8k16, batch 4-8): the looked-up
// entries become A fragments through ldmatrix.trans straight from the replicated
// shared codebook (W^T: 16 columns x 16 rows per column pair), the activations the
// B fragment (16 rows x 8 batch rows), fp32 accumulation.
template <int V, int CBYTES, int R, int B, int WG, bool TILE, bool GTIER, int ACC, bool GROUP, bool REGT = false,
          bool XF = false>
__device__ __forceinline__ void gemv_fast_body(const GemvFastArgs& a, const GemvProblem* __restrict__ probs) {
  constexpr bool H2 = ACC == 1;
  static_assert(!XF || (B == 1 && !GROUP && ACC != 2), "fused activation transform: batch 1, single problem");
  constexpr bool MMA = ACC == 2;
  static_assert(!MMA || (V == 8 && WG == 1 && !GTIER && !TILE), "tensor-core GEMV: v = 8, codes in shared memory");
  static_assert(!GROUP || (!TILE && !GTIER && R == 1), "grouped GEMV: whole-tensor books resident in shared memory");
  static_assert(!REGT || (V == 8 && R == 1 && !TILE && !GROUP && ACC != 2), "register tier: one whole-tensor book, CUDA cores");
  constexpr int kGemvWarps = gemv_warps(B, MMA);
  constexpr int kGemvThreads = kGemvWarps * 32;
  constexpr int EB = V * 2;              // fp16 entry bytes
  constexpr int REP = 128 / EB;          // replicas per bank row
  constexpr int RPL = 16 / CBYTES;       // rows per 16-byte code word
  constexpr int QS = MMA ? (B + 7) / 8 : 1;  // MMA: warps sharing a column block's 16 column pairs
  constexpr int QW = 16 / QS;               // MMA: column pairs per warp
  constexpr int NTL = QS;                   // MMA: 8-row batch tiles (n8 of m16n8k16)
  static_assert(!MMA || (16 % QS == 0 && QW * NTL * 4 == 64), "MMA accumulators: 64 registers per lane");
  constexpr int WM = kGemvWarps / WG / QS;  // warps along M
  constexpr int CR = gemv_chunk_rows(WG, B, CBYTES, MMA);
  constexpr int kSlabRows = gemv_slab_rows(CBYTES);
  constexpr int LOADS = kSlabRows / RPL;  // code words per lane per level per chunk
  constexpr int COLS = 32 * WG * V;      // output columns per column block (256)
  constexpr int GC = 32 * WG;            // sub-vector columns per column block
  constexpr int NQ = V / 4;              // float4 per lane in the cross-warp reduction
  constexpr int RGB = GC * 16;           // bytes of one row group of a column block, per level
  constexpr int LEVB = (CR / RPL) * RGB; // bytes per level per full chunk (contiguous in GEMV_IL)
  constexpr bool SWITCH = TILE || GROUP; // the codebook changes inside a CTA's range
  constexpr int NBUF = SWITCH ? 2 : 1;   // codebook buffers
  // WIDE book layout (every code < 256 is in shared memory): entry e owns a 256-byte
  // row, half h = level (R == 2) or buffer (tile double buffering) holds its
  // replicas, so a lookup address is ONE PRMT of the code byte and the lane's
  // replica offset (the book base and the half fold into the LDS addressing).
  constexpr bool WIDE = !GTIER && R * NBUF <= 2;
  static_assert(LOADS >= 1, "bad tiling");
  static_assert(gemv_stages(R, CBYTES, WG, B, MMA) >= 3, "the ring refill lags two units");
  constexpr int STAGEB = R * LEVB;
  static_assert(STAGEB == stage_bytes(R, CBYTES, WG, B, MMA), "stage size");
  constexpr int XROWB = CR * 2;          // one batch row's activations per chunk
  constexpr int STG = stage_total(R, CBYTES, WG, B, MMA);
  constexpr int kStages = gemv_stages(R, CBYTES, WG, B, MMA);

  extern __shared__ __align__(1024) uint8_t smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint8_t* stages = smem;                                        // kStages x (codes | x)
  uint8_t* books_s = smem + kStages * STG;                       // WIDE: 256 x 256 B; else NBUF x R x n_sh x 128
  const size_t book_bytes = (size_t)R * a.n_sh * 128;
  const size_t book_region = WIDE ? 65536 : NBUF * book_bytes;
  float* red = reinterpret_cast<float*>(books_s + book_region);  // WM x COLS cross-warp partials
  constexpr int RED_ROWS = (B >= 2 && kGemvThreads >= 2 * COLS) ? 2 : 1;  // batch rows per epilogue pass
  uint64_t* bars = reinterpret_cast<uint64_t*>(red + RED_ROWS * WM * COLS);  // full[kStages], empty[kStages]
  const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + kStages);
  uint8_t* xres = reinterpret_cast<uint8_t*>(bars + 2 * kStages + 2);  // XF: the transformed x (M halves)

  const int U = GROUP ? a.total_units : a.n_cblk * a.n_chunks;
  const int u0 = (int)((int64_t)blockIdx.x * U / gridDim.x);
  const int u1 = (int)((int64_t)(blockIdx.x + 1) * U / gridDim.x);
  const int n = u1 - u0;

  // problem cursors: `fc` for the TMA feed (thread 0, runs kStages units ahead),
  // `cc` for the compute and epilogue
  auto load_prob = [&](ProbCursor& c, int i) {
    if constexpr (GROUP) {
      const GemvProblem& q = probs[i];
      c.codes = q.codes; c.level_bytes = q.level_bytes; c.books = q.books; c.x = q.x; c.y = q.y;
      c.M = q.M; c.N = q.N; c.n_cblk = q.n_cblk; c.n_chunks = q.n_chunks; c.base = q.unit_base;
    } else {
      c.codes = a.codes; c.level_bytes = a.level_bytes; c.books = a.books; c.x = a.x; c.y = a.y;
      c.M = a.M; c.N = a.N; c.n_cblk = a.n_cblk; c.n_chunks = a.n_chunks; c.base = 0;
    }
    c.end = c.base + c.n_cblk * c.n_chunks;
    c.idx = i;
    c.last_wb = (c.N / V) - (c.n_cblk - 1) * GC;
  };
  auto seek = [&](ProbCursor& c, int u) {
    if constexpr (GROUP) {
      while (u >= c.end) load_prob(c, c.idx + 1);
    }
  };
  auto first_prob = [&](int u) {
    int lo = 0;
    if constexpr (GROUP) {
      int hi = a.n_probs - 1;
      while (lo < hi) {  // last problem whose base <= u
        const int mid = (lo + hi + 1) >> 1;
        if (probs[mid].unit_base <= u) lo = mid; else hi = mid - 1;
      }
    }
    return lo;
  };
  ProbCursor cc, fc;
  load_prob(cc, first_prob(u0));
  fc = cc;
  // register tier (paper O2): the n_reg hottest entries of the (frequency-ordered,
  // whole-tensor) book live in registers of every thread; codes below n_reg are
  // served by a select chain instead of a shared-memory gather
  constexpr int kRegSlots = 4;
  uint4 hot[REGT ? kRegSlots : 1];
  const uint32_t nreg = REGT ? (uint32_t)min(a.n_reg, kRegSlots) : 0u;
  if constexpr (REGT) {
#pragma unroll
    for (int j = 0; j < kRegSlots; ++j)
      hot[j] = (j < (int)nreg) ? __ldg(reinterpret_cast<const uint4*>(cc.books) + j) : make_uint4(0u, 0u, 0u, 0u);
  }

  if (tid == 0) {
    trace_at(a.trace, 0);
    if (a.trace) {
      unsigned sm;
      asm volatile("mov.u32 %0, %smid;" : "=r"(sm));
      a.trace[blockIdx.x * 8 + 7] = sm;
    }
    for (int s = 0; s < kStages; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, kGemvWarps);
    }
    mbar_fence_init();
  }
  __syncthreads();
  pdl_launch_dependents();

  // ---- TMA feed (thread 0): a column block's chunk is contiguous in the
  // column-blocked GEMV_IL layout, so each unit is one bulk copy per level plus one
  // per activation row. Codes do not depend on the previous kernel and are
  // requested before griddepcontrol.wait; activations only after it.
  // rows of a unit (the last chunk of a column block may be partial) and the byte
  // width of one row group (the last column block may be narrower than 256 columns)
  auto unit_rows = [&](const ProbCursor& c, int u) {
    const int chunk = (u - c.base) % c.n_chunks;
    return chunk == c.n_chunks - 1 ? c.M - (c.n_chunks - 1) * CR : CR;
  };
  auto unit_rgb = [&](const ProbCursor& c, int u) {
    return ((u - c.base) / c.n_chunks == c.n_cblk - 1) ? c.last_wb * 16 : RGB;
  };
  auto expect = [&](int idx) {
    const int u = u0 + idx;
    seek(fc, u);
    const int rows = unit_rows(fc, u);
    mbar_arrive_expect_tx(full0 + 8 * (idx % kStages),
                          (uint32_t)(R * (rows / RPL) * unit_rgb(fc, u) + (XF ? 0 : B * rows * 2)));
  };
  auto issue_codes = [&](int idx) {
    const int s = idx % kStages, u = u0 + idx;
    seek(fc, u);
    const int cb = (u - fc.base) / fc.n_chunks, chunk = (u - fc.base) - cb * fc.n_chunks;
    const int rows = unit_rows(fc, u), rgb = unit_rgb(fc, u);
    const int64_t off = (int64_t)cb * GC * (fc.M / RPL) * 16 + (int64_t)chunk * (CR / RPL) * rgb;
#pragma unroll
    for (int r = 0; r < R; ++r)
      tma_load_1d_hint(smem_u32(stages + s * STG + r * LEVB), fc.codes + r * fc.level_bytes + off,
                  (uint32_t)((rows / RPL) * rgb), full0 + 8 * s, l2_evict_first());
  };
  auto issue_x = [&](ProbCursor& c, int idx) {
    if constexpr (XF) return;  // x is resident in shared memory
    const int s = idx % kStages, u = u0 + idx;
    seek(c, u);
    const int chunk = (u - c.base) % c.n_chunks;
    const int rows = unit_rows(c, u);
#pragma unroll
    for (int b = 0; b < B; ++b)
      tma_load_1d(smem_u32(stages + s * STG + STAGEB + b * XROWB), c.x + (int64_t)b * c.M + (int64_t)chunk * CR,
                  (uint32_t)(rows * 2), full0 + 8 * s);
  };
  const int pre = min(n, kStages);
  if (tid == 0)
    for (int idx = 0; idx < pre; ++idx) {
      expect(idx);
      issue_codes(idx);
    }

  // ===== codebook cache fill =====
  const int wm = warp / (WG * QS), wg = (warp / QS) % WG, wq = warp % QS;
  const uint32_t rep_off = (uint32_t)(lane % REP) * EB;
  const int g_local = wg * 32 + lane;

  constexpr int MAX_PER_THREAD = (1024 + kGemvThreads - 1) / kGemvThreads;  // n_sh * R <= 1024 entries
  auto book_issue = [&](const __half* books, int region, uint4 (&buf)[MAX_PER_THREAD]) {
#pragma unroll
    for (int k = 0; k < MAX_PER_THREAD; ++k) {
      const int idx = tid + k * kGemvThreads;
      if (idx < R * a.n_sh) {
        const int r = idx / a.n_sh, e = idx - r * a.n_sh;
        const uint8_t* src = reinterpret_cast<const uint8_t*>(books) +
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
      const int idx = tid + k * kGemvThreads;
      if (idx < R * a.n_sh) {
        const int r = idx / a.n_sh, e = idx - r * a.n_sh;
        uint8_t* row = WIDE ? books_s + (size_t)e * 256 + (R == 2 ? r : bufi) * 128
                            : books_s + bufi * book_bytes + ((size_t)r * a.n_sh + e) * 128;
#pragma unroll
        for (int q = 0; q < REP; ++q) {
          uint8_t* d = row + ((q + e) % REP) * EB;  // rotate so 8/16 threads hit distinct banks
          if constexpr (EB == 16) *reinterpret_cast<uint4*>(d) = buf[k];
          else *reinterpret_cast<uint2*>(d) = make_uint2(buf[k].x, buf[k].y);
        }
      }
    }
  };
  // region (codebook) of a unit: tile sharing (codec.py:135-177) changes books per
  // row tile and per column tile; whole-tensor sharing has one book
  auto region_of = [&](int u) {
    if constexpr (!TILE) return 0;
    const int cb = u / a.n_chunks, chunk = u - cb * a.n_chunks;  // TILE: single-problem launches only
    return (chunk * CR / a.tile_rows) * a.n_tc + (cb * COLS) / a.tile_cols;
  };

  {
    uint4 bb[MAX_PER_THREAD];
    book_issue(cc.books, region_of(u0), bb);
    book_commit(0, bb);
  }
  uint4 xf_wv[4];
  if constexpr (XF) gemv_xf_preload<kGemvThreads>(a, xf_wv);
  pdl_wait();  // x / y / the partial workspace may belong to the previous kernel
  // TP push: slot parity of this collective (the epoch the last finish kernel left)
  const int tp_par = a.tp_world ? (tp_epoch_of(a.tp_peer[a.tp_rank]) & 1) : 0;
  ProbCursor xc = cc;  // x cursor of the prologue (thread 0)
  if (tid == 0)
    for (int idx = 0; idx < pre; ++idx) issue_x(xc, idx);
  if constexpr (XF) gemv_xf_prologue<kGemvThreads>(a, xres, red, xf_wv);
  __syncthreads();
  if (tid == 0) trace_at(a.trace, 1);

  float acc[MMA ? 1 : B][V];
#pragma unroll
  for (int b = 0; b < (MMA ? 1 : B); ++b)
#pragma unroll
    for (int j = 0; j < V; ++j) acc[b][j] = 0.f;
  // MMA: D fragments (16 columns x 8 batch rows) of this warp's column pairs and batch tiles
  float cacc[MMA ? QW : 1][MMA ? NTL : 1][4];
#pragma unroll
  for (int q = 0; q < (MMA ? QW : 1); ++q)
#pragma unroll
    for (int t = 0; t < (MMA ? NTL : 1); ++t)
#pragma unroll
      for (int j = 0; j < 4; ++j) cacc[q][t][j] = 0.f;

  // SwiGLU epilogue staging (XF kernels, batch 1): a block's 256 finished sums
  float* swg = reinterpret_cast<float*>(xres + (XF ? (size_t)a.M * 2 : 0));
  // one finished output element: y, or (TP push) every rank's slot of this collective
  auto emit = [&](int b, int n, float v) {
    if (XF && a.swiglu) {
      swg[n & 255] = v;  // combined per column block after a barrier (swiglu_flush)
    } else if (a.tp_world == 0) {
      store_from_f32(cc.y, a.y_dtype, (int64_t)b * cc.N + n, v);
    } else {
      tp_push(a.tp_peer, a.tp_world, tp_slot_offset(a.tp_mode, tp_par, a.tp_world, a.tp_rank, a.tp_slot_elems,
                                                     b, n, cc.N), v);
    }
  };
  // silu(gate) * up of a finished column block, with the arithmetic of the unfused
  // path (fp16 gate_up output, then silu_mul_kernel): called by every thread after a
  // barrier that follows the block's emits
  auto swiglu_flush = [&](int cbk) {
    if constexpr (XF) {
      if (tid < 128) {
        const float g = __half2float(__float2half_rn(swg[tid]));
        const float u = __half2float(__float2half_rn(swg[tid + 128]));
        const __half sg = __float2half_rn(g / (1.0f + __expf(-g)));
        store_from_f32(cc.y, a.y_dtype, (int64_t)cbk * 128 + tid, __half2float(sg) * u);
      }
    }
  };
  int cur_buf = 0;
  int span_first = u0;  // first unit of the current span
  int cb = (u0 - cc.base) / cc.n_chunks;
  int span_end = min(u1, cc.base + (cb + 1) * cc.n_chunks);
  for (int u = u0, idx = 0; u < u1; ++u, ++idx) {
    const int s = idx % kStages;
    // refill the stage unit idx-2 used with unit idx-2+kStages (thread 0 only). Lagging
    // two units means every warp has long released that stage, so warp 0 rarely
    // waits (lagging one unit made it wait for the slowest warp every unit).
    if (idx >= 2 && idx - 2 + kStages < n) {
      if (tid == 0) {
        const int j = idx - 2 + kStages;
        mbar_wait(empty0 + 8 * (j % kStages), ((idx - 2) / kStages) & 1);
        expect(j);
        issue_codes(j);
        issue_x(fc, j);
      }
      __syncwarp();
    }
    uint4 nb[MAX_PER_THREAD];
    bool sw = false;
    if constexpr (TILE) {
      sw = (u + 1 < u1) && region_of(u + 1) != region_of(u);
      if (sw) book_issue(cc.books, region_of(u + 1), nb);
    } else if constexpr (GROUP) {
      sw = (u + 1 < u1) && (u + 1 >= cc.end);  // the next unit is the next linear's
      if (sw) book_issue(probs[cc.idx + 1].books, 0, nb);
    }
    mbar_wait(full0 + 8 * s, (idx / kStages) & 1);
    if (tid == 0 && idx == 0) trace_at(a.trace, 2);
    const uint8_t* st = stages + s * STG;
    // this warp's rows of the chunk's activations (XF: of the resident transformed x)
    const uint8_t* xs = XF ? xres + ((int64_t)((u - cc.base) % cc.n_chunks) * CR + wm * kSlabRows) * 2
                           : st + STAGEB + (wm * kSlabRows) * 2;
    const uint8_t* bsm = books_s + cur_buf * book_bytes + rep_off;
    const int region = region_of(u);
    const bool active = wm * kSlabRows < unit_rows(cc, u);  // the last chunk may be partial
    const int rgb = unit_rgb(cc, u);                        // row-group bytes (narrow last column block)
    const int wb = rgb >> 4;                                // sub-vector groups present
    if (MMA && active) {
      // per 16-row k-block: the activations' B fragment (lane: batch row lane/4, rows
      // 2(lane%4)+{0,1}, +8), then per column pair one ldmatrix.x4.trans whose 32 row
      // addresses are looked-up entries (lane: matrix lane/8 = (column half, k half),
      // row lane%8; replica lane%8 keeps each 8-lane phase conflict-free)
      const int j4 = lane >> 3, rr = lane & 7, bn = lane >> 2;
#pragma unroll
      for (int kb = 0; kb < kSlabRows / 16; ++kb) {
        uint32_t xb[NTL][2];
#pragma unroll
        for (int t = 0; t < NTL; ++t) {
          xb[t][0] = xb[t][1] = 0u;
          if (8 * t + bn < B) {
            const uint8_t* xr = xs + (8 * t + bn) * XROWB + (kb * 16 + 2 * (lane & 3)) * 2;
            xb[t][0] = *reinterpret_cast<const uint32_t*>(xr);
            xb[t][1] = *reinterpret_cast<const uint32_t*>(xr + 16);
          }
        }
        const int row = kb * 16 + (j4 >> 1) * 8 + rr;  // this lane's row of the slab
        const uint8_t* cbase = st + (wm * LOADS + row / RPL) * rgb + (row % RPL) * CBYTES + (j4 & 1) * 16;
        // software pipeline: the ldmatrix gathers of column-pair group g+1 are issued
        // before the MMAs of group g, so each MMA finds its A fragment landed instead of
        // waiting one shared-memory round trip per column pair
        // column pairs per group (the grouped kernel's problem cursors leave no registers
        // for a deeper pipeline: one pair at a time there)
        constexpr int QG0 = GROUP ? 1 : (R == 1 ? 4 : 2);
        constexpr int QG = QG0 < QW ? QG0 : QW;
        constexpr int NG = QW / QG;
        uint32_t af[2][QG][R][4];
        auto gather = [&](int g, uint32_t (&dst)[QG][R][4]) {
#pragma unroll
          for (int qq = 0; qq < QG; ++qq) {
            const int q = wq * QW + g * QG + qq;
#pragma unroll
            for (int r = 0; r < R; ++r) {
              const uint8_t* cp = cbase + r * LEVB + q * 32;
              // groups past a narrow last column block hold no codes: entry 0 (never stored)
              const uint32_t code = (2 * q + (j4 & 1) >= wb) ? 0u
                                    : CBYTES == 2 ? (uint32_t)*reinterpret_cast<const uint16_t*>(cp) & 0xffu
                                                  : (uint32_t)*cp;
              const uint32_t addr = WIDE ? smem_u32(books_s) + (code << 8) + (R == 2 ? r : cur_buf) * 128 + rep_off
                                         : smem_u32(bsm) + (uint32_t)(r * a.n_sh * 128) + (code << 7);
              asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
                           : "=r"(dst[qq][r][0]), "=r"(dst[qq][r][1]), "=r"(dst[qq][r][2]), "=r"(dst[qq][r][3])
                           : "r"(addr));
            }
          }
        };
        gather(0, af[0]);
#pragma unroll
        for (int g = 0; g < NG; ++g) {
          if (g + 1 < NG) gather(g + 1, af[(g + 1) & 1]);
#pragma unroll
          for (int qq = 0; qq < QG; ++qq) {
#pragma unroll
            for (int r = 0; r < R; ++r) {
              const uint32_t* f = af[g & 1][qq][r];
#pragma unroll
              for (int t = 0; t < NTL; ++t) {
                float (&c)[4] = cacc[g * QG + qq][t];
                asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, "
                             "{%8, %9}, {%0, %1, %2, %3};"
                             : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
                             : "r"(f[0]), "r"(f[1]), "r"(f[2]), "r"(f[3]), "r"(xb[t][0]), "r"(xb[t][1]));
              }
            }
          }
        }
      }
    } else if (active) {
      // code words of this warp's slab (LOADS x R 16-byte words per lane)
      uint4 cw[LOADS][R];
#pragma unroll
      for (int i = 0; i < LOADS; ++i)
#pragma unroll
        for (int r = 0; r < R; ++r)
          cw[i][r] = g_local < wb ? *reinterpret_cast<const uint4*>(st + r * LEVB + (wm * LOADS + i) * rgb + g_local * 16)
                                  : make_uint4(0u, 0u, 0u, 0u);
      auto lookup = [&](int k, int r) -> const uint8_t* {
        const int i = k / RPL, kr = k % RPL;
        if constexpr (WIDE) {
          // code byte -> bits 8..15, replica offset in bits 0..7: one PRMT
          const uint32_t w = (&cw[i][r].x)[CBYTES == 2 ? kr / 2 : kr / 4];
          const uint32_t byte = CBYTES == 2 ? (kr & 1) * 2 : (kr % 4);
          const uint32_t off = __byte_perm(w, rep_off, 0x5504 | (byte << 4));
          return books_s + off + (R == 2 ? r : cur_buf) * 128;
        }
        uint32_t code;
        if constexpr (CBYTES == 2) {
          const uint32_t w = (&cw[i][r].x)[kr / 2];
          code = (kr & 1) ? (w >> 16) : (w & 0xffff);
        } else {
          const uint32_t w = (&cw[i][r].x)[kr / 4];
          code = (w >> (8 * (kr % 4))) & 0xff;
        }
        bool in_smem = true;
        if constexpr (GTIER) in_smem = code < (uint32_t)a.n_sh;
        return in_smem ? bsm + (size_t)r * a.n_sh * 128 + ((size_t)code << 7)
                       : reinterpret_cast<const uint8_t*>(cc.books) +
                             (((int64_t)(r * a.n_regions + region) * a.K) + code) * EB;
      };
      if constexpr (B >= 4 && H2) {
        // large batch: an 8-row window's entries stay in registers while each batch
        // row runs its own fp16x2 window, so only one window accumulator is live
#pragma unroll
        for (int w8 = 0; w8 < kSlabRows / 8; ++w8) {
#pragma unroll
          for (int r = 0; r < R; ++r) {
            uint32_t ent[8][V / 2];
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
              const uint8_t* src = lookup(w8 * 8 + kk, r);
              if constexpr (EB == 16) {
                const uint4 q = *reinterpret_cast<const uint4*>(src);
                ent[kk][0] = q.x; ent[kk][1] = q.y; ent[kk][2] = q.z; ent[kk][3] = q.w;
              } else {
                const uint2 q = *reinterpret_cast<const uint2*>(src);
                ent[kk][0] = q.x; ent[kk][1] = q.y;
              }
            }
#pragma unroll
            for (int b = 0; b < B; ++b) {
              const uint4 xv = *reinterpret_cast<const uint4*>(xs + b * XROWB + w8 * 16);
              uint32_t hw[V / 2];
#pragma unroll
              for (int j = 0; j < V / 2; ++j) hw[j] = 0u;
#pragma unroll
              for (int kk = 0; kk < 8; ++kk) {
                const uint32_t xw = (&xv.x)[kk / 2];
#pragma unroll
                for (int j = 0; j < V / 2; ++j)
                  hw[j] = (kk & 1) ? hfma2_bcast<1>(ent[kk][j], xw, hw[j]) : hfma2_bcast<0>(ent[kk][j], xw, hw[j]);
              }
#pragma unroll
              for (int j = 0; j < V / 2; ++j) {
                acc[b][2 * j] = fma_h((uint16_t)(hw[j] & 0xffff), kHalfOne, acc[b][2 * j]);
                acc[b][2 * j + 1] = fma_h((uint16_t)(hw[j] >> 16), kHalfOne, acc[b][2 * j + 1]);
              }
            }
          }
        }
      } else {
      // lookups are issued LB rows at a time ahead of their FMAs (register budget:
      // 64 per thread at 1024 threads)
      constexpr int LB = (R == 2 || B >= 4) ? 4 : 8;
#pragma unroll
      for (int w8 = 0; w8 < kSlabRows / 8; ++w8) {  // 8-row fp16 windows
        uint32_t hw[B][V / 2];
#pragma unroll
        for (int b = 0; b < B; ++b)
#pragma unroll
          for (int j = 0; j < V / 2; ++j) hw[b][j] = 0u;
        uint4 xv[B];  // the window's 8 activations per batch row (shared-memory broadcast)
#pragma unroll
        for (int b = 0; b < B; ++b) xv[b] = *reinterpret_cast<const uint4*>(xs + b * XROWB + w8 * 16);
#pragma unroll
        for (int l0 = 0; l0 < 8; l0 += LB) {
        uint32_t ent[LB][R][V / 2];
#pragma unroll
        for (int kk = 0; kk < LB; ++kk)
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const uint8_t* src = lookup(w8 * 8 + l0 + kk, r);
            if constexpr (REGT) {
              // the code (16-bit or 8-bit) of row k; below n_reg -> registers
              const int k = w8 * 8 + l0 + kk, i = k / RPL, kr = k % RPL;
              uint32_t code;
              if constexpr (CBYTES == 2) {
                const uint32_t w = (&cw[i][r].x)[kr / 2];
                code = (kr & 1) ? (w >> 16) : (w & 0xffffu);
              } else {
                code = ((&cw[i][r].x)[kr / 4] >> (8 * (kr % 4))) & 0xffu;
              }
              uint4 q;
              if (code < nreg) {
                q = hot[0];
#pragma unroll
                for (int j = 1; j < kRegSlots; ++j)
                  if (code == (uint32_t)j) q = hot[j];
              } else {
                q = *reinterpret_cast<const uint4*>(src);
              }
              ent[kk][r][0] = q.x; ent[kk][r][1] = q.y; ent[kk][r][2] = q.z; ent[kk][r][3] = q.w;
            } else if constexpr (EB == 16) {
              const uint4 q = *reinterpret_cast<const uint4*>(src);
              ent[kk][r][0] = q.x; ent[kk][r][1] = q.y; ent[kk][r][2] = q.z; ent[kk][r][3] = q.w;
            } else {
              const uint2 q = *reinterpret_cast<const uint2*>(src);
              ent[kk][r][0] = q.x; ent[kk][r][1] = q.y;
            }
          }
#pragma unroll
        for (int kk = 0; kk < LB; ++kk) {
          const int k = w8 * 8 + l0 + kk;
#pragma unroll
          for (int r = 0; r < R; ++r) {
#pragma unroll
            for (int b = 0; b < B; ++b) {
              const uint32_t xw = (&xv[b].x)[(k % 8) / 2];  // packed pair holding row k
              if constexpr (H2) {
                // packed fp16x2 FMA into the 8-row window, activation broadcast by the
                // operand selector (full-rate HFMA2; mixed-precision FHFMA is quarter rate)
#pragma unroll
                for (int j = 0; j < V / 2; ++j)
                  hw[b][j] = (k & 1) ? hfma2_bcast<1>(ent[kk][r][j], xw, hw[b][j])
                                     : hfma2_bcast<0>(ent[kk][r][j], xw, hw[b][j]);
              } else {
                const uint16_t xh = (uint16_t)((k & 1) ? (xw >> 16) : (xw & 0xffff));
#pragma unroll
                for (int j = 0; j < V / 2; ++j) {
                  acc[b][2 * j] = fma_h((uint16_t)(ent[kk][r][j] & 0xffff), xh, acc[b][2 * j]);
                  acc[b][2 * j + 1] = fma_h((uint16_t)(ent[kk][r][j] >> 16), xh, acc[b][2 * j + 1]);
                }
              }
            }
          }
        }
        }
        if constexpr (H2) {  // flush the window into the fp32 accumulators (exact widening)
#pragma unroll
          for (int b = 0; b < B; ++b)
#pragma unroll
            for (int j = 0; j < V / 2; ++j) {
              acc[b][2 * j] = fma_h((uint16_t)(hw[b][j] & 0xffff), kHalfOne, acc[b][2 * j]);
              acc[b][2 * j + 1] = fma_h((uint16_t)(hw[b][j] >> 16), kHalfOne, acc[b][2 * j + 1]);
            }
        }
      }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty0 + 8 * s);
    if constexpr (SWITCH) {
      if (sw) {
        book_commit(cur_buf ^ 1, nb);  // the other buffer was released at the previous swap
        __syncthreads();
        cur_buf ^= 1;
      }
    }

    // ---- end of a span: reduce the WM row-slabs in a fixed order, then write y,
    // publish a partial, or finish a split column block
    if (u + 1 == span_end) {
      if (tid == 0 && u + 1 == u1) trace_at(a.trace, 3);
      const int cf = span_first - cc.base - cb * cc.n_chunks;  // first chunk of the span
      const int cl = u - cc.base - cb * cc.n_chunks;           // last chunk
      const bool whole = (cf == 0 && cl == cc.n_chunks - 1);
      const bool finisher = (cf == 0 && !whole);
      // with 512 threads each pass reduces two batch rows (thread half t / COLS takes
      // row b + half; a D fragment of the MMA path holds two rows anyway); keep[b] then
      // holds this thread's row b + half
      constexpr int BP = (B >= 2 && kGemvThreads >= 2 * COLS) ? 2 : 1;
      static_assert(!MMA || BP == 2, "the MMA epilogue writes two rows per pass");
      const int half = BP == 2 ? tid / COLS : 0;
      float keep[B];
#pragma unroll
      for (int b = 0; b < B; b += BP) {
        if constexpr (MMA) {
          // D fragment: lane holds columns 16q + lane/4 (+8) of batch rows 2(lane%4) + {0, 1}
          // (the column index goes through an opaque shift: nvcc otherwise folds
          // 4 * (lane >> 2) into lane - (b >> 1) under the predicate and emitted
          // misaligned stores for the batch-8 instance)
          uint32_t cq;
          asm("shr.b32 %0, %1, 2;" : "=r"(cq) : "r"((uint32_t)lane));
          float* rp = red + (size_t)wm * COLS + cq + 16 * wq * QW;
          if ((lane & 3) == ((b % 8) >> 1)) {
#pragma unroll
            for (int q = 0; q < QW; ++q) {
              rp[16 * q] = cacc[q][b / 8][0];
              rp[16 * q + 8] = cacc[q][b / 8][2];
              rp[WM * COLS + 16 * q] = cacc[q][b / 8][1];
              rp[WM * COLS + 16 * q + 8] = cacc[q][b / 8][3];
            }
          }
        } else {
        // partials stored [w][q][g][4]: each lane's float4 stores are conflict-free
#pragma unroll
        for (int h = 0; h < BP; ++h)
#pragma unroll
          for (int q = 0; q < NQ; ++q)
            *reinterpret_cast<float4*>(red + (size_t)(h * WM + wm) * COLS + (q * GC + g_local) * 4) =
                make_float4(acc[b + h][4 * q], acc[b + h][4 * q + 1], acc[b + h][4 * q + 2], acc[b + h][4 * q + 3]);
        }
        __syncthreads();
        keep[b] = 0.f;
        if (tid < BP * COLS) {
          const int o = tid % COLS, bb = b + half;
          float sum = 0.f;
#pragma unroll
          for (int w = 0; w < WM; ++w) sum += red[(size_t)(half * WM + w) * COLS + o];
          const int q = o / (GC * 4), g = (o / 4) % GC, c = o % 4;
          const int col = MMA ? o : g * V + q * 4 + c;
          if (whole) {
            if (cb * COLS + col < cc.N) emit(bb, cb * COLS + col, sum);
          }
          else if (finisher) keep[b] = sum;
          else st_relaxed_u64(a.part + ((int64_t)blockIdx.x * B + bb) * COLS + col, tag_partial(sum));
        }
        __syncthreads();
      }
      if (XF && a.swiglu && whole) {
        swiglu_flush(cb);
        __syncthreads();
      }
      if (finisher) {
        // the later spans of this column block are the first spans of the CTAs
        // k in (blockIdx.x, k_end); their tagged partials are polled in parallel,
        // summed in chunk order, and the slots zeroed for the next launch
        int k_end = blockIdx.x + 1;
        while (k_end < (int)gridDim.x && (int)((int64_t)k_end * U / gridDim.x) < cc.base + (cb + 1) * cc.n_chunks)
          ++k_end;
        const int n_later = k_end - blockIdx.x - 1;
        if (tid < BP * COLS) {
          const int o = tid % COLS;
          const int q = o / (GC * 4), g = (o / 4) % GC, c = o % 4;
          const int col = MMA ? o : g * V + q * 4 + c;
#pragma unroll
          for (int b0 = 0; b0 < B; b0 += BP) {
            const int b = b0 + half;
            float sum = keep[b0];
            constexpr int PF = 8;  // partial loads in flight
            for (int j0 = 0; j0 < n_later; j0 += PF) {
              unsigned long long pv[PF];
              unsigned long long* pp[PF];
#pragma unroll
              for (int j = 0; j < PF; ++j) {
                pp[j] = a.part + ((int64_t)(blockIdx.x + 1 + j0 + j) * B + b) * COLS + col;
                pv[j] = (j0 + j < n_later) ? ld_relaxed_u64(pp[j]) : (1ull << 32);
              }
              // re-poll every pending slot per round: one L2 round trip per round, not
              // one per slot (the publishers finish together, so a slot-by-slot wait
              // serialised up to PF round trips into the launch's tail)
              for (;;) {
                bool pending = false;
#pragma unroll
                for (int j = 0; j < PF; ++j) pending |= (pv[j] >> 32) == 0;
                if (!pending) break;
#pragma unroll
                for (int j = 0; j < PF; ++j)
                  if ((pv[j] >> 32) == 0) pv[j] = ld_relaxed_u64(pp[j]);
              }
#pragma unroll
              for (int j = 0; j < PF; ++j) {
                if (j0 + j < n_later) {
                  sum += __uint_as_float((uint32_t)pv[j]);
                  st_relaxed_u64(pp[j], 0ull);
                }
              }
            }
            if (cb * COLS + col < cc.N) emit(b, cb * COLS + col, sum);
          }
        }
        if (tid == 0) trace_at(a.trace, 5);
        if (XF && a.swiglu) {
          __syncthreads();
          swiglu_flush(cb);
          __syncthreads();
        }
      }
#pragma unroll
      for (int b = 0; b < (MMA ? 1 : B); ++b)
#pragma unroll
        for (int j = 0; j < V; ++j) acc[b][j] = 0.f;
#pragma unroll
      for (int q = 0; q < (MMA ? QW : 1); ++q)
#pragma unroll
        for (int t = 0; t < (MMA ? NTL : 1); ++t)
#pragma unroll
          for (int j = 0; j < 4; ++j) cacc[q][t][j] = 0.f;
      span_first = u + 1;
      if (u + 1 < u1) {
        seek(cc, u + 1);
        cb = (u + 1 - cc.base) / cc.n_chunks;
        span_end = min(u1, cc.base + (cb + 1) * cc.n_chunks);
      }
    }
  }
  if (tid == 0) trace_at(a.trace, 6);
  if (a.tp_world) tp_signal(a.tp_peer, a.tp_world, a.tp_rank, tp_par);
}

template <int V, int CBYTES, int R, int B, int WG, bool TILE, bool GTIER, int ACC, bool REGT = false, bool XF = false>
__global__ void __launch_bounds__(gemv_warps(B, ACC == 2) * 32, 1) gemv_fast_kernel(GemvFastArgs a) {
  gemv_fast_body<V, CBYTES, R, B, WG, TILE, GTIER, ACC, false, REGT, XF>(a, nullptr);
}

// grouped launch: the problem table travels as a __grid_constant__ kernel parameter
template <int V, int CBYTES, int R, int B, int WG, int ACC>
__global__ void __launch_bounds__(gemv_warps(B, ACC == 2) * 32, 1)
    gemv_group_kernel(GemvFastArgs a, const __grid_constant__ GemvTable t) {
  gemv_fast_body<V, CBYTES, R, B, WG, false, false, ACC, true>(a, t.p);
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

int gemv_tc_dispatch(const Geom& g, const VqbTensor* w, const void* x, int x_dtype, int rows, void* y, int y_dtype,
                     const VqbLaunch* L, void* ws, size_t ws_bytes, cudaStream_t st);
int64_t gemv_tc_ws_bytes(const Geom& g, const VqbTensor* w, int rows, const VqbLaunch* L);

// host-side description of a fused activation transform (vqb_gemv_xf)
struct GemvXf {
  int mode;  // VQB_XF_* (without the SWIGLU bit)
  int swiglu;
  const __half* add;
  const __half* res_in;
  __half* res_out;
  const __half* weight;
  float eps;
};

struct FastPlan {
  bool ok = false;
  int V = 0, cbytes = 0, R = 0, WG = 1;
  bool tile = false, gtier = true, h2 = true, mma = false;
  int n_sh = 0, n_cblk = 0, n_chunks = 0, threads = 0, n_reg = 0;
  size_t smem = 0;
};

static FastPlan plan_fast(const Geom& g, const VqbTensor* t, int rows, int x_dtype, const VqbLaunch* L) {
  FastPlan p;
  if (L && (L->flags & VQB_FLAG_FORCE_GENERIC)) return p;
  if (t->layout != VQB_LAYOUT_GEMV_IL || t->codebook_dtype != VQB_F16 || x_dtype != VQB_F16) return p;
  // batch 32 / 64 on mma.sync measured 1.5-4x slower than the tcgen05 GEMM (the legacy
  // HMMA path tops out near 50 TFLOP/s on sm_100): those batches take vqb_gemm
  if (!(rows == 1 || rows == 2 || rows == 4 || rows == 8 || rows == 16)) return p;
  if (!(g.v == 4 || g.v == 8) || g.R > 2) return p;
  if (!(g.bits == 8 || g.bits == 16)) return p;
  if (g.bits == 16 && g.R != 1) return p;
  p.V = g.v;
  p.cbytes = g.code_bytes;
  p.R = g.R;
  p.WG = (g.v == 4) ? 2 : 1;
  const int cols_per_cta = 32 * p.WG * g.v;
  const int CR = gemv_chunk_rows(p.WG, rows, p.cbytes);
  // the last column block may be narrower than 256 columns (TP shards such as
  // 22016 / 4 = 5504 columns): GEMV_IL stores it with its own row-group width
  if (g.rows % gemv_slab_rows(p.cbytes) != 0) return p;
  if (g.sharing == VQB_SHARE_TILE) {
    if (g.tile_rows % CR != 0 || g.tile_cols % cols_per_cta != 0) return p;
    p.tile = true;
  } else if (g.sharing != VQB_SHARE_WHOLE) {
    return p;
  }
  int n_sh = (L && L->n_shared > 0) ? L->n_shared : 256;
  n_sh = std::min(n_sh, g.K);
  n_sh = std::min(n_sh, 1024 / g.R);
  if (L && (L->flags & VQB_FLAG_NO_SHARED)) n_sh = 0;
  // every code of the stream is resident when the shared span covers the codebook
  // or the largest code; the WIDE (256-row) layout then drops the global tier
  const int span = g.K <= n_sh ? g.K : ((t->max_code >= 0 && t->max_code < n_sh) ? t->max_code + 1 : -1);
  p.gtier = !(span > 0 && span <= 256);
  if (!p.gtier) n_sh = std::min(n_sh, 256);
  p.n_sh = n_sh;
  p.h2 = !(L && (L->flags & VQB_FLAG_EXACT_ACCUM));
  // register tier: batch 1, one 16-bit/8-bit level of a whole-tensor book (REGT kernels)
  if (L && L->n_reg > 0 && rows == 1 && g.v == 8 && g.R == 1 && !p.tile && p.h2)
    p.n_reg = std::min(L->n_reg, std::min(4, g.K));
  // batch 4-8: tensor-core inner product (every entry resident in shared memory).
  // Measured (quip2 4096x12288 / 4096x4096): batch 8 22.0 / 13.7 us vs 28.1 / 20.1 on
  // CUDA cores, batch 4 about even, batch 2 slower (the mma path reads its codes with a
  // 2-way bank conflict per 16-row k-block of the GEMV_IL words).
  p.mma = p.h2 && !p.gtier && !p.tile && g.v == 8 && rows >= 4 && !(L && (L->flags & VQB_FLAG_NO_MMA));
  if (rows >= 16 && !p.mma) return FastPlan{};  // batch 16-64 exist only on the tensor-core path
  const int CRm = gemv_chunk_rows(p.WG, rows, p.cbytes, p.mma);
  p.n_cblk = (int)ceil_div(g.cols, cols_per_cta);
  p.n_chunks = (int)((g.rows + CRm - 1) / CRm);
  p.threads = gemv_warps(rows, p.mma) * 32;
  const int nst = gemv_stages(p.R, p.cbytes, p.WG, rows, p.mma);
  const int WM = gemv_warps(rows, p.mma) / p.WG;
  const bool wide = !p.gtier && p.R * (p.tile ? 2 : 1) <= 2;  // mirrors the kernel's WIDE layout
  p.smem = (size_t)nst * stage_total(p.R, p.cbytes, p.WG, rows, p.mma) +
           (wide ? (size_t)65536 : (size_t)(p.tile ? 2 : 1) * p.R * p.n_sh * 128) +
           (size_t)((rows >= 2 && p.threads >= 2 * cols_per_cta) ? 2 : 1) * WM * cols_per_cta * 4 +
           2 * nst * 8 + 16;
  p.ok = true;
  return p;
}


// workspace: the tagged partials (one B x COLS slot of 8-byte words per CTA) live
// in the self-resetting head
static int64_t fast_ws_bytes(const FastPlan& p, const Geom& g, int rows) {
  if (!p.ok) return VQB_WS_COUNTER_BYTES + 1024 * 64;  // (also the tcgen05 GEMV's partial slots)
  return VQB_WS_COUNTER_BYTES + 1024 * 64;  // tagged partials live in the head; + debug trace
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
      VQB_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, p.threads, p.smem));
      occ_cache[key] = occ;
    } else {
      occ = it->second;
    }
  }
  if (occ < 1) return set_error(VQB_ECAPACITY, "GEMV plan (n_shared=%d) does not fit one CTA per SM", p.n_sh);
  // one persistent CTA per SM: every CTA is resident (a finishing CTA polls the
  // partials of later CTAs) and the SM's second slot is left to the next kernel
  int grid = balanced_grid((int64_t)p.n_cblk * p.n_chunks, sm_count());
  // the planner's split of the reduction over M: each column block is shared by
  // ~split_factor CTAs of the stream-K schedule
  if (L && L->split_axis == 'M' && L->split_factor > 0) grid = std::max(1, std::min(grid, p.n_cblk * L->split_factor));
  if (L && L->grid_limit > 0) grid = std::min(grid, L->grid_limit);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(p.threads);
  cfg.dynamicSmemBytes = p.smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  cfg.attrs = attr;
  cfg.numAttrs = persistent_attrs(attr, L ? L->flags : 0);
  VQB_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kernel, a));
  set_kernel("gemv_fast");
  set_launch(grid, p.threads, p.n_sh, p.n_reg);
  return VQB_OK;
}

template <int V, int CBYTES, int R, int B, int WG, bool TILE>
static GemvKernel pick_acc(bool gtier, bool h2, bool mma, bool regt) {
  if constexpr (V == 8 && WG == 1 && !TILE && B == 1 && R == 1)
    if (regt && h2) return gtier ? gemv_fast_kernel<V, CBYTES, R, B, WG, TILE, true, 1, true>
                                 : gemv_fast_kernel<V, CBYTES, R, B, WG, TILE, false, 1, true>;
  if constexpr (V == 8 && WG == 1 && !TILE && B >= 2)
    if (mma && !gtier) return gemv_fast_kernel<V, CBYTES, R, B, WG, TILE, false, 2>;
  return gtier ? (h2 ? gemv_fast_kernel<V, CBYTES, R, B, WG, TILE, true, 1>
                     : gemv_fast_kernel<V, CBYTES, R, B, WG, TILE, true, 0>)
               : (h2 ? gemv_fast_kernel<V, CBYTES, R, B, WG, TILE, false, 1>
                     : gemv_fast_kernel<V, CBYTES, R, B, WG, TILE, false, 0>);
}

template <int V, int CBYTES, int R, int WG, bool TILE>
static GemvKernel pick_kernel(int rows, bool gtier, bool h2, bool mma, bool regt) {
  if constexpr (V == 8 && WG == 1 && !TILE) {
    if (rows == 16) return (mma && !gtier) ? gemv_fast_kernel<V, CBYTES, R, 16, WG, TILE, false, 2> : nullptr;
  }
  if (rows >= 16) return nullptr;
  switch (rows) {
    case 1: return pick_acc<V, CBYTES, R, 1, WG, TILE>(gtier, h2, mma, regt);
    case 2: return pick_acc<V, CBYTES, R, 2, WG, TILE>(gtier, h2, mma, regt);
    case 4: return pick_acc<V, CBYTES, R, 4, WG, TILE>(gtier, h2, mma, regt);
    default: return pick_acc<V, CBYTES, R, 8, WG, TILE>(gtier, h2, mma, regt);
  }
}

static GemvKernel fast_kernel_for(const FastPlan& p, int rows) {
  // (V, code bytes, R, WG, tile-shared) combinations covering the BASELINE configs
  if (p.V == 8 && p.cbytes == 2 && p.R == 1 && !p.tile) return pick_kernel<8, 2, 1, 1, false>(rows, p.gtier, p.h2, p.mma, p.n_reg > 0);
  if (p.V == 8 && p.cbytes == 1 && p.R == 2 && !p.tile) return pick_kernel<8, 1, 2, 1, false>(rows, p.gtier, p.h2, p.mma, p.n_reg > 0);
  if (p.V == 8 && p.cbytes == 1 && p.R == 1 && !p.tile) return pick_kernel<8, 1, 1, 1, false>(rows, p.gtier, p.h2, p.mma, p.n_reg > 0);
  if (p.V == 8 && p.cbytes == 1 && p.R == 1 && p.tile) return pick_kernel<8, 1, 1, 1, true>(rows, p.gtier, p.h2, p.mma, p.n_reg > 0);
  if (p.V == 4 && p.cbytes == 1 && p.R == 1 && p.tile) return pick_kernel<4, 1, 1, 2, true>(rows, p.gtier, p.h2, p.mma, p.n_reg > 0);
  if (p.V == 4 && p.cbytes == 1 && p.R == 1 && !p.tile) return pick_kernel<4, 1, 1, 2, false>(rows, p.gtier, p.h2, p.mma, p.n_reg > 0);
  return nullptr;
}

int gemv_cs_dispatch(const Geom& g, const VqbTensor* w, const void* x, int x_dtype, int rows, void* y, int y_dtype,
                     const VqbLaunch* L, cudaStream_t st);

int gemv_dispatch(const VqbTensor* w, const void* x, int x_dtype, int rows, void* y, int y_dtype,
                  const VqbLaunch* L, void* ws, size_t ws_bytes, cudaStream_t st, bool* used_fast,
                  const VqbPeerComm* tp, int tp_mode, const GemvXf* xf) {
  Geom g;
  int s = make_geom(w, &g);
  if (s) return s;
  if (g.ndim != 2) return set_error(VQB_ESHAPE, "quantized weight must be 2-D (M, N), got rank %d", g.ndim);
  if (rows < 1) return set_error(VQB_ESHAPE, "activation rows must be >= 1, got %d", rows);
  if (x_dtype < VQB_F32 || x_dtype > VQB_BF16 || y_dtype < VQB_F32 || y_dtype > VQB_BF16)
    return set_error(VQB_ECONFIG, "unknown activation/output dtype");
  if (!tp && !xf) {
    // batches 4-64: the tcgen05 decode GEMV (csrc/gemm.cu) where it covers the configuration
    const int t = gemv_tc_dispatch(g, w, x, x_dtype, rows, y, y_dtype, L, ws, ws_bytes, st);
    if (t <= 0) {
      if (used_fast && t == 0) *used_fast = true;
      return t;
    }
    // batch 1, 16 x 256-column outputs: the column-split kernel (csrc/gemv_cs.cu)
    const int c = gemv_cs_dispatch(g, w, x, x_dtype, rows, y, y_dtype, L, st);
    if (c <= 0) {
      if (used_fast && c == 0) *used_fast = true;
      return c;
    }
  }
  FastPlan p = plan_fast(g, w, rows, x_dtype, L);
  GemvKernel kernel = p.ok ? fast_kernel_for(p, rows) : nullptr;
  // the activations are TMA-staged: 16-byte aligned rows
  if (kernel && ((reinterpret_cast<uintptr_t>(x) & 15) != 0 || (g.rows % 8) != 0)) kernel = nullptr;
  if (xf) {
    // the fused-transform instances: batch 1, QuiP#-style VQ<8,16,1> / 8-bit whole-tensor
    // books resident in shared memory (every code < 256), fp16 windows
    const bool xf_ok = kernel && rows == 1 && p.V == 8 && p.R == 1 && !p.tile && !p.gtier && p.h2 && p.n_reg == 0 &&
                       (g.rows % 8) == 0;
    kernel = !xf_ok ? nullptr : (p.cbytes == 2 ? gemv_fast_kernel<8, 2, 1, 1, 1, false, false, 1, false, true>
                                               : gemv_fast_kernel<8, 1, 1, 1, 1, false, false, 1, false, true>);
    if (!kernel)
      return set_error(VQB_ECONFIG, "the fused-activation GEMV needs batch 1, v = 8, one level, whole-tensor "
                                    "books with every code < 256 and fp16 activations");
    p.smem += (size_t)g.rows * 2 + (xf->swiglu ? 1024 : 0);
    if (xf->swiglu && (g.cols % 256 != 0 || y_dtype != VQB_F16))
      return set_error(VQB_ECONFIG, "the SwiGLU epilogue needs N %% 256 == 0 ([gate 128 | up 128] blocks) and fp16 y");
  }
  if (used_fast) *used_fast = kernel != nullptr;
  if (tp && !kernel)
    return set_error(VQB_ECONFIG, "the tensor-parallel push GEMV needs the fast kernel's configuration");
  if (kernel) {
    const int64_t need = fast_ws_bytes(p, g, rows);
    if ((int64_t)ws_bytes < need || !ws)
      return set_error(VQB_ECAPACITY, "GEMV workspace too small: %zu < %lld", ws_bytes, (long long)need);
    const int64_t units = (int64_t)p.n_cblk * p.n_chunks;
    uint8_t* wsb = reinterpret_cast<uint8_t*>(ws);
    GemvFastArgs a = {};
    a.codes = reinterpret_cast<const uint8_t*>(w->d_codes);
    a.level_bytes = g.S * g.code_bytes;
    a.books = reinterpret_cast<const __half*>(w->d_codebooks);
    a.x = reinterpret_cast<const __half*>(x);
    a.y = y;
    a.y_dtype = y_dtype;
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
    a.n_reg = p.n_reg;
    const int grid = (int)std::min<int64_t>(units, sm_count());  // upper bound for the slot check
    // head layout: [0, 64 KB) split-arrival counters (attention), then the GEMV slots
    if ((int64_t)grid * rows * (32 * p.WG * p.V) * 8 > VQB_WS_COUNTER_BYTES - 2 * 65536)
      return set_error(VQB_ECAPACITY, "GEMV partial slots exceed the workspace head");
    a.part = reinterpret_cast<unsigned long long*>(wsb + 65536);
    a.trace = (L && (L->flags & 32)) ? reinterpret_cast<unsigned long long*>(wsb + VQB_WS_COUNTER_BYTES) : nullptr;
    if (xf) {
      a.xf_mode = xf->mode;
      a.swiglu = xf->swiglu;
      a.xf_add = xf->add;
      a.xf_res_in = xf->res_in;
      a.xf_res_out = xf->res_out;
      a.xf_w = xf->weight;
      a.xf_eps = xf->eps;
    }
    if (tp) {
      a.tp_world = tp->world;
      a.tp_rank = tp->rank;
      a.tp_mode = tp_mode;
      for (int i = 0; i < tp->world; ++i) a.tp_peer[i] = reinterpret_cast<char*>(tp->d_peer[i]);
      a.tp_slot_elems = tp->slot_elems;
    }
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

// ---------------------------------------------------------------------------
// grouped launch: every problem one GEMV of the same configuration

typedef void (*GemvGroupKernel)(GemvFastArgs, const GemvTable);

template <int CBYTES, int B>
static GemvGroupKernel group_kernel_acc(bool h2, bool mma) {
  if constexpr (B >= 4)
    if (mma) return gemv_group_kernel<8, CBYTES, 1, B, 1, 2>;
  return h2 ? gemv_group_kernel<8, CBYTES, 1, B, 1, 1> : gemv_group_kernel<8, CBYTES, 1, B, 1, 0>;
}

template <int CBYTES>
static GemvGroupKernel group_kernel_rows(int rows, bool h2, bool mma) {
  switch (rows) {
    case 1: return group_kernel_acc<CBYTES, 1>(h2, mma);
    case 2: return group_kernel_acc<CBYTES, 2>(h2, mma);
    case 4: return group_kernel_acc<CBYTES, 4>(h2, mma);
    default: return group_kernel_acc<CBYTES, 8>(h2, mma);
  }
}

int gemv_grouped_dispatch(const VqbTensor* ws_t, int n, const void* const* xs, int x_dtype, int rows,
                          void* const* ys, int y_dtype, const VqbLaunch* L, void* ws, size_t ws_bytes,
                          cudaStream_t st) {
  if (n < 1 || n > kMaxGroup) return set_error(VQB_ESHAPE, "grouped GEMV takes 1..%d problems, got %d", kMaxGroup, n);
  if (x_dtype != VQB_F16 || y_dtype < VQB_F32 || y_dtype > VQB_BF16)
    return set_error(VQB_ECONFIG, "grouped GEMV: fp16 activations, f32/f16/bf16 outputs");
  GemvTable table;
  FastPlan p0;
  int units = 0;
  for (int i = 0; i < n; ++i) {
    Geom g;
    int s = make_geom(&ws_t[i], &g);
    if (s) return s;
    if (g.ndim != 2) return set_error(VQB_ESHAPE, "grouped GEMV problem %d is not 2-D", i);
    FastPlan p = plan_fast(g, &ws_t[i], rows, x_dtype, L);
    if (!p.ok || p.tile || p.gtier || p.R != 1 || p.V != 8 || (reinterpret_cast<uintptr_t>(xs[i]) & 15) != 0)
      return set_error(VQB_ECONFIG,
                       "grouped GEMV problem %d: needs whole-tensor books with every code < 256, v = 8, R = 1, "
                       "GEMV_IL codes, fp16 books and 16-byte aligned activations", i);
    if (i == 0) {
      p0 = p;
    } else if (p.cbytes != p0.cbytes || p.mma != p0.mma || p.h2 != p0.h2 || p.n_sh != p0.n_sh ||
               ws_t[i].log2_entries != ws_t[0].log2_entries) {
      return set_error(VQB_ECONFIG, "grouped GEMV problem %d differs in configuration from problem 0", i);
    }
    GemvProblem& q = table.p[i];
    q.codes = reinterpret_cast<const uint8_t*>(ws_t[i].d_codes);
    q.level_bytes = g.S * g.code_bytes;
    q.books = reinterpret_cast<const __half*>(ws_t[i].d_codebooks);
    q.x = reinterpret_cast<const __half*>(xs[i]);
    q.y = ys[i];
    q.M = (int)g.rows;
    q.N = (int)g.cols;
    q.n_cblk = p.n_cblk;
    q.n_chunks = p.n_chunks;
    q.unit_base = units;
    q.pad = 0;
    if ((int64_t)units + (int64_t)p.n_cblk * p.n_chunks > (1LL << 30))
      return set_error(VQB_ESHAPE, "grouped GEMV: too many work units");
    units += p.n_cblk * p.n_chunks;
  }
  if ((int64_t)ws_bytes < (int64_t)VQB_WS_COUNTER_BYTES + 65536 || !ws)
    return set_error(VQB_ECAPACITY, "GEMV workspace too small: %zu", ws_bytes);
  GemvGroupKernel kernel = p0.cbytes == 2 ? group_kernel_rows<2>(rows, p0.h2, p0.mma)
                                          : group_kernel_rows<1>(rows, p0.h2, p0.mma);
  Geom g0;
  make_geom(&ws_t[0], &g0);
  GemvFastArgs a = {};
  a.y_dtype = y_dtype;
  a.K = g0.K;
  a.n_regions = 1;
  a.n_sh = p0.n_sh;
  a.total_units = units;
  a.n_probs = n;
  uint8_t* wsb = reinterpret_cast<uint8_t*>(ws);
  int grid = balanced_grid(units, sm_count());
  if (L && L->grid_limit > 0) grid = std::min(grid, L->grid_limit);
  if ((int64_t)grid * rows * 256 * 8 > VQB_WS_COUNTER_BYTES - 2 * 65536)
    return set_error(VQB_ECAPACITY, "GEMV partial slots exceed the workspace head");
  a.part = reinterpret_cast<unsigned long long*>(wsb + 65536);
  a.trace = (L && (L->flags & 32)) ? reinterpret_cast<unsigned long long*>(wsb + VQB_WS_COUNTER_BYTES) : nullptr;
  {
    static std::mutex mu;
    static std::unordered_map<const void*, int> done;
    std::lock_guard<std::mutex> lock(mu);
    int dev = 0;
    cudaGetDevice(&dev);
    const void* key = reinterpret_cast<const void*>(reinterpret_cast<uintptr_t>(kernel) ^ ((uintptr_t)dev << 56));
    if (!done.count(key)) {
      VQB_CUDA_CHECK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448));
      int occ = 0;
      VQB_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, p0.threads, p0.smem));
      done[key] = occ;
    }
    if (done[key] < 1) return set_error(VQB_ECAPACITY, "grouped GEMV plan does not fit one CTA per SM");
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(p0.threads);
  cfg.dynamicSmemBytes = p0.smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  cfg.attrs = attr;
  cfg.numAttrs = persistent_attrs(attr, L ? L->flags : 0);
  VQB_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kernel, a, table));
  set_kernel("gemv_group");
  set_launch(grid, p0.threads, p0.n_sh, 0);
  return VQB_OK;
}

int64_t gemv_ws_bytes(const VqbTensor* w, int64_t rows, const VqbLaunch* L) {
  Geom g;
  int s = make_geom(w, &g);
  if (s) return s;
  FastPlan p = plan_fast(g, w, (int)rows, VQB_F16, L);
  int64_t a = (p.ok && fast_kernel_for(p, (int)rows)) ? fast_ws_bytes(p, g, (int)rows) : 0;
  a = std::max(a, gemv_tc_ws_bytes(g, w, (int)rows, L));
  return std::max(a, generic_ws_bytes(g, (int)rows));
}

int gemv_usage(VqbUsage* u) {
  cudaFuncAttributes at;
  auto k = gemv_fast_kernel<8, 2, 1, 1, 1, false, false, true>;
  VQB_CUDA_CHECK(cudaFuncGetAttributes(&at, k));
  const int threads = gemv_warps(1) * 32;
  const int nst = gemv_stages(1, 2, 1, 1);
  const size_t smem = nst * stage_total(1, 2, 1, 1) + 65536 + (size_t)gemv_warps(1) * 256 * 4 + 2 * nst * 8 + 16;
  VQB_CUDA_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448));
  u->shared_bytes = (int)(at.sharedSizeBytes + smem);
  u->regs_per_thread = at.numRegs;
  u->threads_per_block = threads;
  int occ = 0;
  VQB_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, threads, smem));
  u->max_blocks_per_sm = occ;
  return VQB_OK;
}

}  // namespace vqb

extern "C" int vqb_gemv_grouped(const VqbTensor* w, int32_t n, const void* const* d_xs, int32_t x_dtype,
                                int32_t rows, void* const* d_ys, int32_t y_dtype, const VqbLaunch* launch, void* d_ws,
                                size_t ws_bytes, void* stream) {
  return vqb::gemv_grouped_dispatch(w, n, d_xs, x_dtype, rows, d_ys, y_dtype, launch, d_ws, ws_bytes,
                                    reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int vqb_gemv(const VqbTensor* w, const void* d_x, int32_t x_dtype, int32_t rows, void* d_y,
                        int32_t y_dtype, const VqbLaunch* launch, void* d_ws, size_t ws_bytes, void* stream) {
  return vqb::gemv_dispatch(w, d_x, x_dtype, rows, d_y, y_dtype, launch, d_ws, ws_bytes,
                            reinterpret_cast<cudaStream_t>(stream), nullptr, nullptr, 0, nullptr);
}

extern "C" int vqb_gemv_xf(const VqbTensor* w, const void* d_x, int32_t x_dtype, int32_t mode, const void* d_res_in,
                           void* d_res_out, const void* d_weight, float eps, void* d_y, int32_t y_dtype,
                           const VqbLaunch* launch, void* d_ws, size_t ws_bytes, void* stream) {
  const int swiglu = (mode & VQB_XF_SWIGLU_OUT) ? 1 : 0;
  mode &= ~VQB_XF_SWIGLU_OUT;
  if (mode != VQB_XF_RMSNORM && mode != VQB_XF_SILU_MUL) return vqb::set_error(VQB_ECONFIG, "unknown activation transform %d", mode);
  if (x_dtype != VQB_F16) return vqb::set_error(VQB_ECONFIG, "the fused-activation GEMV takes fp16 activations");
  if (mode == VQB_XF_RMSNORM && (!d_res_in || !d_weight))
    return vqb::set_error(VQB_ECONFIG, "RMSNorm transform needs the residual and the norm weight");
  if (mode == VQB_XF_SILU_MUL && !d_x) return vqb::set_error(VQB_ECONFIG, "SiLU transform needs the gate|up input");
  for (const void* ptr : {d_x, d_res_in, (const void*)d_res_out, d_weight})
    if (reinterpret_cast<uintptr_t>(ptr) & 15) return vqb::set_error(VQB_ECONFIG, "activation buffers must be 16-byte aligned");
  vqb::GemvXf xf{mode, swiglu, mode == VQB_XF_RMSNORM ? reinterpret_cast<const __half*>(d_x) : nullptr,
                 reinterpret_cast<const __half*>(d_res_in), reinterpret_cast<__half*>(d_res_out),
                 reinterpret_cast<const __half*>(d_weight), eps};
  // x is read only by the transform (never by the TMA ring in this mode): the plan
  // checks see the SiLU input or, for RMSNorm, the residual
  const void* xp = mode == VQB_XF_SILU_MUL ? d_x : d_res_in;
  int s = vqb::gemv_dispatch(w, xp, x_dtype, 1, d_y, y_dtype, launch, d_ws, ws_bytes,
                             reinterpret_cast<cudaStream_t>(stream), nullptr, nullptr, 0, &xf);
  if (s) return s;
  vqb::set_kernel(mode == VQB_XF_RMSNORM ? "gemv_rmsnorm" : "gemv_silu");
  return VQB_OK;
}
