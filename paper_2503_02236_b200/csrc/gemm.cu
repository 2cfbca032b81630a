// gemm.cu — prefill GEMM with VQ dequantisation fused into the tcgen05 operand
// pipeline: Y(rows, N) = X(rows, M) @ dequant(W)(M, N).
//
// Replaces SimMachine._matmul/_mm_block (pkg/src/vqforge/sim.py:697-775) for
// ComputeOp.gemm (dataflow.py:68-71); oracle reference_compute `a @ w`
// (sim.py:136-144).
//
// B200 design. One CTA computes a 256 x 128 tile of Y with
// two 128 x 128 fp32 accumulators in TMEM (256 of the 512 columns):
//  * warp 0 — TMA producer: X tiles (256 rows x 64 K, fp16/bf16) are loaded with
//    cp.async.bulk.tensor (SWIZZLE_128B) into a 4-stage ring; this is exactly the
//    UMMA K-major SW128 canonical layout, so no reshuffle is needed.
//  * warps 2-9 — dequantisation producers (the paper's "shared" fusion level:
//    tcgen05 reads operands only from shared memory / TMEM): each lane takes one
//    16-byte code word (8 K-rows of one 8-column sub-vector group, GEMV_IL layout),
//    looks each code up in the replicated, bank-conflict-free shared codebook
//    (csrc/gemv.cu) and stores the 16-byte fp16 entry straight into the UMMA
//    MN-major SW128 layout of the W tile: one LDS.128 -> one STS.128 per code,
//    both conflict-free. A proxy fence then hands the tile to the async proxy.
//  * warp 1 — a single thread issues tcgen05.mma.cta_group::1.kind::f16
//    (M=128, N=128, K=16) for both accumulators and commits each stage back to
//    the producers through an mbarrier; the final commit releases the epilogue.
//  * epilogue (the producer warps again, two per TMEM lane quarter): tcgen05.ld 32x32b,
//    convert, store.
#include <cuda.h>

#include <mutex>
#include <type_traits>

#include "common.cuh"

namespace vqb {

int gemv_dispatch(const VqbTensor* w, const void* x, int x_dtype, int rows, void* y, int y_dtype,
                  const VqbLaunch* L, void* ws, size_t ws_bytes, cudaStream_t st, bool* used_fast,
                  const VqbPeerComm* tp, int tp_mode, const struct GemvXf* xf);

constexpr int kProdWarps = 16;      // dequantisation producer warps (2..17)
constexpr int kGemmThreads = 64 + kProdWarps * 32;  // + TMA warp + MMA warp
constexpr int kTileM = 256;         // rows (two 128-row accumulators)
constexpr int kTileN = 128;         // output columns (16 sub-vector groups of 8)
constexpr int kTileK = 64;          // reduction rows per stage (one 128-byte swizzle span)
__host__ __device__ constexpr int gemm_stages(int R) { return R == 1 ? 4 : 3; }  // ring depth (smem)
constexpr int kABytes = kTileM * kTileK * 2;   // 32 KB
constexpr int kBBytes = kTileK * kTileN * 2;   // 16 KB
constexpr int kBookEntries = 256;              // shared tier (replicated, 128 B per entry)
constexpr int kBookBytes = kBookEntries * 128; // per level

struct GemmArgs {
  const uint8_t* codes;  // GEMV_IL (8 rows of u16 codes / 16 rows of u8 codes per 16-byte word)
  int64_t level_bytes;
  const uint16_t* books; // (R, K, 8) fp16 or bf16
  void* y;
  int y_dtype;
  int rows, M, N, G, K, n_sh;
  int splits;            // split-K factor (CTAs per output tile); > 1 writes fp32 partials
  float* part;           // (splits, rows, N) fp32 partials when splits > 1
};

// ---- tcgen05 / TMA PTX wrappers ----------------------------------------------

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  // SM100 shared-memory matrix descriptor (cute::UMMA::SmemDescriptor): start>>4 [0,14),
  // LBO>>4 [16,30), SBO>>4 [32,46), version 1 [46,48), SWIZZLE_128B (2) [61,64)
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3fff);
  d |= (uint64_t)((lbo >> 4) & 0x3fff) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3fff) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

__device__ __forceinline__ void umma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

// Calls f(integral_constant<I * STEP>) for the runtime index idx in [0, N), so the
// callee can index register arrays with a compile-time row offset.
template <int I, int N, int STEP, typename F>
__device__ __forceinline__ void dispatch_rows(int idx, F&& f) {
  if constexpr (I < N) {
    if (idx == I) f(std::integral_constant<int, I * STEP>{});
    else dispatch_rows<I + 1, N, STEP>(idx, f);
  }
}

template <typename OutT>
__device__ __forceinline__ void store_row32(void* y, int y_dtype, int64_t off, const uint32_t (&v)[32]) {
  (void)y_dtype;
  if constexpr (sizeof(OutT) == 4) {
    float4* p = reinterpret_cast<float4*>(reinterpret_cast<float*>(y) + off);
#pragma unroll
    for (int i = 0; i < 8; ++i)
      p[i] = make_float4(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1]), __uint_as_float(v[4 * i + 2]),
                         __uint_as_float(v[4 * i + 3]));
  } else {
    uint4* p = reinterpret_cast<uint4*>(reinterpret_cast<OutT*>(y) + off);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint32_t w[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float lo = __uint_as_float(v[8 * i + 2 * j]), hi = __uint_as_float(v[8 * i + 2 * j + 1]);
        if constexpr (std::is_same<OutT, __half>::value) {
          const __half2 h = __floats2half2_rn(lo, hi);
          w[j] = *reinterpret_cast<const uint32_t*>(&h);
        } else {
          const __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
          w[j] = *reinterpret_cast<const uint32_t*>(&h);
        }
      }
      p[i] = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
}

template <int CBYTES, int R, bool BF16, typename OutT>
__global__ void __launch_bounds__(kGemmThreads, 1) gemm_tc_kernel(const __grid_constant__ CUtensorMap tmap_x,
                                                                  GemmArgs a) {
  constexpr int RPL = 16 / CBYTES;          // K-rows per 16-byte code word
  constexpr int WORDS = (kTileK / RPL) * (kTileN / 8);  // code words per level per stage
  constexpr int STG = gemm_stages(R);
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* book = smem;                                      // R x 256 entries x 128 B (replicated)
  uint8_t* sa = smem + R * kBookBytes;                       // STG x 32 KB (A)
  uint8_t* sb = sa + STG * kABytes;                  // STG x 16 KB (B)
  uint64_t* bars = reinterpret_cast<uint64_t*>(sb + STG * kBBytes);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * STG + 1);
  const uint32_t full_a0 = smem_u32(bars), full_b0 = smem_u32(bars + STG);
  const uint32_t empty0 = smem_u32(bars + 2 * STG), tmem_full = smem_u32(bars + 3 * STG);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n_tiles_n = a.N / kTileN;
  // split-K (small row counts): CTA (tile, ks) reduces K stages [it_lo, it_hi) of its tile
  const int tile = blockIdx.x / a.splits, ks = blockIdx.x % a.splits;
  const int tile_n = tile % n_tiles_n, tile_m = tile / n_tiles_n;
  const int row0 = tile_m * kTileM, n0 = tile_n * kTileN;
  const int k_total = a.M / kTileK;
  const int it_lo = ks * k_total / a.splits, it_hi = (ks + 1) * k_total / a.splits;
  const int k_iters = it_hi - it_lo;  // stages of this CTA; local stage j = it - it_lo

  // ---- setup: barriers, TMEM, replicated shared codebook
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STG; ++s) {
      mbar_init(full_a0 + 8 * s, 1);
      mbar_init(full_b0 + 8 * s, kProdWarps);  // one arrive per dequant warp
      mbar_init(empty0 + 8 * s, 1);   // tcgen05.commit
    }
    mbar_init(tmem_full, 1);
    mbar_fence_init();
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_x)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int idx = tid; idx < R * a.n_sh; idx += kGemmThreads) {
    const int r = idx / a.n_sh, e = idx - r * a.n_sh;
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(a.books + ((int64_t)r * a.K + e) * 8));
    uint8_t* row = book + ((size_t)r * kBookEntries + e) * 128;
#pragma unroll
    for (int q = 0; q < 8; ++q) *reinterpret_cast<uint4*>(row + ((q + e) & 7) * 16) = v;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ===== TMA producer (X tiles) =====
    if (lane == 0) {
      for (int it = 0; it < k_iters; ++it) {
        const int s = it % STG;
        mbar_wait(empty0 + 8 * s, ((it / STG) & 1) ^ 1);
        mbar_arrive_expect_tx(full_a0 + 8 * s, kABytes);
        tma_load_2d(smem_u32(sa + s * kABytes), &tmap_x, (it_lo + it) * kTileK, row0, full_a0 + 8 * s);
      }
    }
  } else if (warp == 1) {
    // ===== MMA issuer =====
    // kind::f16, D fp32, A K-major, B MN-major, N = 128, M = 128
    const uint32_t fmt = BF16 ? 1u : 0u;
    const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | (0u << 15) | (1u << 16) |
                           ((uint32_t)(kTileN >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    if (lane == 0) {
      for (int it = 0; it < k_iters; ++it) {
        const int s = it % STG;
        const uint32_t ph = (it / STG) & 1;
        mbar_wait(full_a0 + 8 * s, ph);
        mbar_wait(full_b0 + 8 * s, ph);
        tc_fence_after();
        const uint32_t a_base = smem_u32(sa + s * kABytes), b_base = smem_u32(sb + s * kBBytes);
#pragma unroll
        for (int k = 0; k < kTileK / 16; ++k) {
          // B: MN-major SW128, atoms of 8 K-rows x 64 columns (1 KB); LBO = column-atom
          // stride (1 KB), SBO = 8-row-group stride (2 KB); K=16 spans two row groups.
          const uint64_t bdesc = umma_desc(b_base + k * 4096, 1024, 2048);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (h == 1 && row0 + 128 >= a.rows) break;  // the second 128-row half is all padding
            // A: K-major SW128 rows of 128 B; SBO = 8-row-group stride (1 KB); K step = 32 B
            const uint64_t adesc = umma_desc(a_base + h * 16384 + k * 32, 16, 1024);
            umma_f16(tmem_base + h * kTileN, adesc, bdesc, idesc, (it | k) != 0);
          }
        }
        umma_commit(empty0 + 8 * s);  // frees the stage once these MMAs completed
      }
      umma_commit(tmem_full);
    }
  } else {
    // ===== dequantisation producers (warps 2..2+kProdWarps) =====
    const int dw = warp - 2;
    const int dtid = dw * 32 + lane;  // 0..kProdWarps*32-1
    // code words are prefetched PF stages ahead into a register ring, so the global
    // load latency overlaps the dequantisation of the previous stages
    // 256 producer threads share the stage's 64 K-rows x 16 groups evenly: a thread
    // owns one code word (8 rows of u16 codes / 16 rows of u8) and KROWS of its rows,
    // so every thread dequantises 4 rows x R levels
    constexpr int NPT = kProdWarps * 32;
    static_assert(WORDS * RPL % NPT == 0 && NPT % WORDS == 0, "producer split");
    constexpr int NW = 1;
    constexpr int KROWS = WORDS * RPL / NPT;  // rows per thread per word
    const int my_item = dtid % WORDS;
    const int k_off = (dtid / WORDS) * KROWS;
    constexpr int PF = 3;
    uint4 ring[PF][R][NW];
    auto fetch = [&](int it, uint4 (&cw)[R][NW]) {
#pragma unroll
      for (int i = 0; i < NW; ++i) {
        const int item = my_item;
        if (it < k_iters) {
          const int grp = item % (kTileN / 8), blk = item / (kTileN / 8);
          // column-blocked GEMV_IL: 32 groups (256 columns) per block, blocks of M/RPL row groups
          const int gg = n0 / 8 + grp, cb = gg / 32, gi = gg % 32, wb = min(32, a.G - cb * 32);
          const int64_t word =
              ((int64_t)cb * 32 * (a.M / RPL) + (int64_t)((it_lo + it) * kTileK / RPL + blk) * wb + gi) * 16;
#pragma unroll
          for (int r = 0; r < R; ++r) cw[r][i] = ldg_stream(a.codes + r * a.level_bytes + word);
        }
      }
    };
#pragma unroll
    for (int p = 0; p < PF; ++p) fetch(p, ring[p]);
    for (int it0 = 0; it0 < k_iters; it0 += PF)
#pragma unroll
    for (int pp = 0; pp < PF; ++pp) {
      const int it = it0 + pp;
      if (it >= k_iters) break;
      const int s = it % STG;
      uint4 cw[R][NW];
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int i = 0; i < NW; ++i) cw[r][i] = ring[pp][r][i];
      fetch(it + PF, ring[pp]);
      mbar_wait(empty0 + 8 * s, ((it / STG) & 1) ^ 1);
      uint8_t* btile = sb + s * kBBytes;
#pragma unroll
      for (int i = 0; i < NW; ++i) {
        const int item = my_item;
        {
          const int grp = item % (kTileN / 8), blk = item / (kTileN / 8);
          const int c = grp & 7, nb = grp >> 3;  // 16-byte chunk and 64-column atom
          // the row offset must be a compile-time constant for cw[] to stay in registers
          auto rows = [&](auto ko) {
            constexpr int KO = decltype(ko)::value;
#pragma unroll
          for (int kk = 0; kk < KROWS; ++kk) {
            const int k = KO + kk;  // compile-time: the code word stays in registers
            uint4 e;
#pragma unroll
            for (int r = 0; r < R; ++r) {
              uint32_t code;
              if constexpr (CBYTES == 2) {
                const uint32_t w = (&cw[r][i].x)[k / 2];
                code = (k & 1) ? (w >> 16) : (w & 0xffff);
              } else {
                const uint32_t w = (&cw[r][i].x)[k / 4];
                code = (w >> (8 * (k % 4))) & 0xff;
              }
              const uint4 q = code < (uint32_t)a.n_sh
                                  ? *reinterpret_cast<const uint4*>(book + ((size_t)r * kBookEntries + code) * 128 +
                                                                     (lane & 7) * 16)
                                  : __ldg(reinterpret_cast<const uint4*>(a.books + ((int64_t)r * a.K + code) * 8));
              if (r == 0) {
                e = q;
              } else {
                // residual level: packed fp16x2 / bf16x2 add, a single rounding of the
                // exact two-term sum (the fp32 dequant rounds it to fp32 first; both
                // agree unless that rounding creates an fp16 tie — within the GEMM
                // tolerance, never observed on the parity sets)
                uint32_t* ew = &e.x;
                const uint32_t* qw = &q.x;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                  if constexpr (BF16) {
                    const __nv_bfloat162 h = __hadd2(*reinterpret_cast<const __nv_bfloat162*>(&ew[j]),
                                                     *reinterpret_cast<const __nv_bfloat162*>(&qw[j]));
                    ew[j] = *reinterpret_cast<const uint32_t*>(&h);
                  } else {
                    const __half2 h = __hadd2(*reinterpret_cast<const __half2*>(&ew[j]),
                                              *reinterpret_cast<const __half2*>(&qw[j]));
                    ew[j] = *reinterpret_cast<const uint32_t*>(&h);
                  }
                }
              }
            }
            const int r = blk * RPL + k;  // K-row within the stage
            uint8_t* dst = btile + ((r >> 3) * (kTileN / 64) + nb) * 1024 + (r & 7) * 128 + ((c ^ (r & 7)) << 4);
            *reinterpret_cast<uint4*>(dst) = e;
          }
          };
          dispatch_rows<0, RPL / KROWS, KROWS>(k_off / KROWS, rows);
        }
      }
      fence_proxy_async();  // generic-proxy stores -> visible to the tensor core (async proxy)
      __syncwarp();
      if (lane == 0) mbar_arrive(full_b0 + 8 * s);
    }

    // ===== epilogue: TMEM -> registers -> global =====
    mbar_wait(tmem_full, 0);
    tc_fence_after();
    const int quarter = warp & 3;  // TMEM lane quarter this warp may access
    constexpr int CPW = (kTileN / 32) / (kProdWarps / 4);  // 32-column chunks per warp
    const int cc0 = ((warp - 2) / 4) * CPW;                  // warps sharing a quarter split the columns
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (h == 1 && row0 + 128 >= a.rows) break;  // never computed: padding rows only
      const int row = row0 + h * 128 + quarter * 32 + lane;
#pragma unroll
      for (int c2 = 0; c2 < CPW; ++c2) {
        const int cc = cc0 + c2;
        uint32_t v[32];
        const uint32_t taddr = tmem_base + ((uint32_t)(quarter * 32) << 16) + h * kTileN + cc * 32;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
              "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
              "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
              "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (row < a.rows) {
          if (a.splits == 1) store_row32<OutT>(a.y, a.y_dtype, (int64_t)row * a.N + n0 + cc * 32, v);
          else store_row32<float>(a.part + (int64_t)ks * a.rows * a.N, VQB_F32, (int64_t)row * a.N + n0 + cc * 32, v);
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(256));
  }
}

// ---------------------------------------------------------------------------
// CTA-pair GEMM (tcgen05.mma.cta_group::2): a cluster of two CTAs on one TPC
// computes a 256 x NT output tile with UMMA M = 256. Each CTA holds its 128 rows of
// the X tile (TMA) and dequantises HALF of the W tile (NT / 2 columns) into its own
// shared memory; the leader CTA's single thread issues one MMA per K=16 step that
// reads A and B from both CTAs and writes each CTA's 128 x NT accumulator into its
// own TMEM. Per SM and K stage that is 16 KB of A + NT / 2 x 64 x 2 B of B read by
// the tensor core plus the same B bytes of dequantisation stores/gathers — half the
// B-side shared-memory traffic per flop of the one-CTA kernel, whose 256 x 128 tile
// reads its B tile once per 128-row half. Barriers: the leader's "full" barriers
// count both CTAs' X bytes (cta_group::2 TMA) and both CTAs' dequant-warp arrivals
// (remote mbarrier arrive through mapa); tcgen05.commit multicasts "empty" and the
// final "TMEM full" to both CTAs.

// Remote arrive on the leader's barrier. Default (.release.cta) semantics like
// CUTLASS's 2-SM transform pipeline: the data is consumed by the pair's tensor core
// (async proxy), ordered by the preceding fence.proxy.async; a .release.cluster arrive
// costs a cluster-scope memory barrier per stage (measured: the dominant stall).
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAITC_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAITC_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d_pair(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                                 uint32_t leader_bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(leader_bar)
      : "memory");
}
__device__ __forceinline__ void umma_f16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit_pair(uint32_t bar) {
  asm volatile(
      "{\n.reg .b16 m;\nmov.b16 m, 3;\n"
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n}" ::"r"(bar)
      : "memory");
}

constexpr int kPairRowsCta = 128;                  // X rows per CTA (UMMA M = 256 per pair)
constexpr int kPairABytes = kPairRowsCta * kTileK * 2;  // 16 KB
__host__ __device__ constexpr int pair_stages(int R) { return R == 1 ? 5 : 4; }
__host__ __device__ constexpr size_t pair_smem(int R, int NT) {
  return (size_t)R * kBookBytes + (size_t)pair_stages(R) * (kPairABytes + kTileK * (NT / 2) * 2) +
         (3 * pair_stages(R) + 1) * 8 + 16;
}

template <int CBYTES, int R, bool BF16, typename OutT, int NT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kGemmThreads, 1)
    gemm_pair_kernel(const __grid_constant__ CUtensorMap tmap_x, GemmArgs a) {
  constexpr int CN = NT / 2;                        // W columns this CTA dequantises
  constexpr int BBYTES = kTileK * CN * 2;
  constexpr int RPL = 16 / CBYTES;
  constexpr int WORDS = (kTileK / RPL) * (CN / 8);  // code words per level per stage (this CTA)
  constexpr int STG = pair_stages(R);
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* book = smem;
  uint8_t* sa = smem + R * kBookBytes;
  uint8_t* sb = sa + STG * kPairABytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sb + STG * BBYTES);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * STG + 1);
  const uint32_t full_a0 = smem_u32(bars), full_b0 = smem_u32(bars + STG);
  const uint32_t empty0 = smem_u32(bars + 2 * STG), tmem_full = smem_u32(bars + 3 * STG);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t rank = cluster_ctarank();
  const int pair = blockIdx.x >> 1;
  const int n_tiles_n = a.N / NT;
  const int tile_n = pair % n_tiles_n, tile_m = pair / n_tiles_n;
  const int row0 = tile_m * 2 * kPairRowsCta + (int)rank * kPairRowsCta;  // this CTA's X rows
  const int n0 = tile_n * NT + (int)rank * CN;                            // this CTA's W columns
  const int k_iters = a.M / kTileK;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STG; ++s) {
      mbar_init(full_a0 + 8 * s, 1);               // the leader's expect_tx (both CTAs' bytes)
      mbar_init(full_b0 + 8 * s, 2 * kProdWarps);  // every dequant warp of the pair
      mbar_init(empty0 + 8 * s, 1);                // multicast tcgen05.commit
    }
    mbar_init(tmem_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_x)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(NT));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  for (int idx = tid; idx < R * a.n_sh; idx += kGemmThreads) {
    const int r = idx / a.n_sh, e = idx - r * a.n_sh;
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(a.books + ((int64_t)r * a.K + e) * 8));
    uint8_t* row = book + ((size_t)r * kBookEntries + e) * 128;
#pragma unroll
    for (int q = 0; q < 8; ++q) *reinterpret_cast<uint4*>(row + ((q + e) & 7) * 16) = v;
  }
  tc_fence_before();
  cluster_sync_all();  // barriers initialised and TMEM allocated in both CTAs
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ===== TMA producer: this CTA's 128 X rows; bytes counted on the leader's barrier
    if (lane == 0) {
      for (int it = 0; it < k_iters; ++it) {
        const int s = it % STG;
        mbar_wait(empty0 + 8 * s, ((it / STG) & 1) ^ 1);
        if (rank == 0) mbar_arrive_expect_tx(full_a0 + 8 * s, 2 * kPairABytes);
        tma_load_2d_pair(smem_u32(sa + s * kPairABytes), &tmap_x, it * kTileK, row0,
                         mapa_rank(full_a0 + 8 * s, 0));
      }
    }
  } else if (warp == 1) {
    // ===== MMA issuer (leader CTA, one thread): UMMA 256 x NT x 16 over both CTAs
    const uint32_t fmt = BF16 ? 1u : 0u;
    const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | (0u << 15) | (1u << 16) |
                           ((uint32_t)(NT >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
    if (rank == 0 && lane == 0) {
      for (int it = 0; it < k_iters; ++it) {
        const int s = it % STG;
        const uint32_t ph = (it / STG) & 1;
        mbar_wait(full_a0 + 8 * s, ph);
        mbar_wait(full_b0 + 8 * s, ph);
        tc_fence_after();
        const uint32_t a_base = smem_u32(sa + s * kPairABytes), b_base = smem_u32(sb + s * BBYTES);
#pragma unroll
        for (int k = 0; k < kTileK / 16; ++k) {
          // B: this CTA's CN columns, MN-major SW128 atoms (8 K-rows x 64 columns, 1 KB);
          // LBO = column-atom stride (1 KB), SBO = 8-row-group stride (CN / 64 KB)
          const uint64_t bdesc = umma_desc(b_base + k * 2 * (CN / 64) * 1024, 1024, (CN / 64) * 1024);
          const uint64_t adesc = umma_desc(a_base + k * 32, 16, 1024);
          umma_f16_pair(tmem_base, adesc, bdesc, idesc, (it | k) != 0);
        }
        umma_commit_pair(empty0 + 8 * s);  // frees the stage in both CTAs
      }
      umma_commit_pair(tmem_full);
    }
  } else {
    // ===== dequantisation producers: this CTA's CN columns of the W tile
    const int dw = warp - 2;
    const int dtid = dw * 32 + lane;
    constexpr int NPT = kProdWarps * 32;
    static_assert(WORDS * RPL % NPT == 0 && NPT % WORDS == 0, "producer split");
    constexpr int KROWS = WORDS * RPL / NPT;
    const int my_item = dtid % WORDS;
    const int k_off = (dtid / WORDS) * KROWS;
    const uint32_t full_b_leader = mapa_rank(full_b0, 0);
    constexpr int PF = 6;  // code words requested 6 stages ahead (3: latency-bound)
    uint4 ring[PF][R];
    const int grp = my_item % (CN / 8), blk = my_item / (CN / 8);
    const int gg = n0 / 8 + grp, cb = gg / 32, gi = gg % 32, wb = min(32, a.G - cb * 32);
    auto fetch = [&](int it, uint4 (&cw)[R]) {
      if (it < k_iters) {
        const int64_t word = ((int64_t)cb * 32 * (a.M / RPL) + (int64_t)(it * kTileK / RPL + blk) * wb + gi) * 16;
#pragma unroll
        for (int r = 0; r < R; ++r) cw[r] = ldg_stream(a.codes + r * a.level_bytes + word);
      }
    };
#pragma unroll
    for (int p = 0; p < PF; ++p) fetch(p, ring[p]);
    const int c = grp & 7, nb = grp >> 3;  // 16-byte chunk and 64-column atom
    for (int it0 = 0; it0 < k_iters; it0 += PF)
#pragma unroll
      for (int pp = 0; pp < PF; ++pp) {
        const int it = it0 + pp;
        if (it >= k_iters) break;
        const int s = it % STG;
        uint4 cw[R];
#pragma unroll
        for (int r = 0; r < R; ++r) cw[r] = ring[pp][r];
        fetch(it + PF, ring[pp]);
        mbar_wait(empty0 + 8 * s, ((it / STG) & 1) ^ 1);
        uint8_t* btile = sb + s * BBYTES;
        auto rows = [&](auto ko) {
          constexpr int KO = decltype(ko)::value;
#pragma unroll
          for (int kk = 0; kk < KROWS; ++kk) {
            const int k = KO + kk;
            uint4 e;
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
              const uint4 q = code < (uint32_t)a.n_sh
                                  ? *reinterpret_cast<const uint4*>(book + ((size_t)r * kBookEntries + code) * 128 +
                                                                     (lane & 7) * 16)
                                  : __ldg(reinterpret_cast<const uint4*>(a.books + ((int64_t)r * a.K + code) * 8));
              if (r == 0) {
                e = q;
              } else {
                uint32_t* ew = &e.x;
                const uint32_t* qw = &q.x;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                  if constexpr (BF16) {
                    const __nv_bfloat162 h = __hadd2(*reinterpret_cast<const __nv_bfloat162*>(&ew[j]),
                                                     *reinterpret_cast<const __nv_bfloat162*>(&qw[j]));
                    ew[j] = *reinterpret_cast<const uint32_t*>(&h);
                  } else {
                    const __half2 h = __hadd2(*reinterpret_cast<const __half2*>(&ew[j]),
                                              *reinterpret_cast<const __half2*>(&qw[j]));
                    ew[j] = *reinterpret_cast<const uint32_t*>(&h);
                  }
                }
              }
            }
            const int kr = blk * RPL + k;  // K-row within the stage
            uint8_t* dst = btile + ((kr >> 3) * (CN / 64) + nb) * 1024 + (kr & 7) * 128 + ((c ^ (kr & 7)) << 4);
            *reinterpret_cast<uint4*>(dst) = e;
          }
        };
        dispatch_rows<0, RPL / KROWS, KROWS>(k_off / KROWS, rows);
        fence_proxy_async();  // generic stores -> async proxy (the pair's tensor core)
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(full_b_leader + 8 * s);
      }

    // ===== epilogue: this CTA's 128 rows x NT columns of TMEM
    mbar_wait(tmem_full, 0);
    tc_fence_after();
    const int quarter = warp & 3;
    constexpr int CPW = (NT / 32) / (kProdWarps / 4);
    const int cc0 = ((warp - 2) / 4) * CPW;
    const int row = row0 + quarter * 32 + lane;
    const int ncol0 = tile_n * NT;
#pragma unroll
    for (int c2 = 0; c2 < CPW; ++c2) {
      const int cc = cc0 + c2;
      uint32_t v[32];
      const uint32_t taddr = tmem_base + ((uint32_t)(quarter * 32) << 16) + cc * 32;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
          "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
            "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
            "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
            "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (row < a.rows) store_row32<OutT>(a.y, a.y_dtype, (int64_t)row * a.N + ncol0 + cc * 32, v);
    }
  }

  tc_fence_before();
  cluster_sync_all();  // both CTAs are done with the pair's shared memory and TMEM
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(NT));
  }
}

// ---------------------------------------------------------------------------
// Decode GEMV on tcgen05 (batches 4-64): the roles of the GEMM swapped so the batch is
// the UMMA N dimension — D[n_out, b] = W^T[n_out, k] x X^T[k, b] with M = 128 output
// columns per UMMA (two halves of a 256-column GEMV_IL block), N = the batch padded to
// 8..64, K = 16. A CTA owns one column block and a contiguous range of its 64-row
// chunks (split-K sized to one wave); the chunk's code words arrive by one bulk copy
// per level, 16 producer warps look them up in the replicated shared codebook and
// write the W^T tile in the UMMA MN-major SW128 layout (A operand, transposed), X
// arrives by TMA as the K-major B operand (rows past the batch zero-filled), the fp32
// accumulator lives in TMEM. Split partials go to the workspace as plain fp32 and an
// ordered reduce kernel sums them (deterministic). This replaces mma.sync for the
// batches where the legacy HMMA path (~50 TFLOP/s on sm_100) made the GEMV compute-bound.
constexpr int kGemvTcMinRows = 5;                // default from 5 rows: at 4 the mma.sync GEMV is faster (measured)
constexpr int kGtProd = 16;                       // dequantisation producer warps (2..17)
constexpr int kGtEpi = 4;                         // epilogue warps (18..21)
constexpr int kGtThreads = (2 + kGtProd + kGtEpi) * 32;
// producer groups: the 16 dequantisation warps form gt_stages(R) groups that work on
// consecutive stages concurrently (one group's latency chain — code LDS, gathers, STS,
// proxy fence, barrier — no longer serialises the stages); the A / X ring has one slot
// per group
// K rows per stage: 128 for one level (fewer, fatter stages: the per-stage hand-off
// chain, not any one resource, bounds this kernel), 64 for two (shared-memory budget)
__host__ __device__ constexpr int gt_k(int R) { return R == 1 ? 128 : 64; }
__host__ __device__ constexpr int gt_stages(int R) { return 2; }
__host__ __device__ constexpr int gt_code_stages(int BN) { return 4; }                     // code-word ring
__host__ __device__ constexpr int gt_x_stages(int R, int BN) { return R == 1 && BN > 32 ? 2 : 4; }  // X ring
__host__ __device__ constexpr int gt_a_bytes(int R) { return 256 * gt_k(R) * 2; }       // W^T tile, two halves

struct GemvTcArgs {
  const uint8_t* codes;  // GEMV_IL, N % 256 == 0
  int64_t level_bytes;
  const uint16_t* books;  // (R, K, 8) fp16
  void* y;
  int y_dtype;
  int B, M, N, K, n_sh;
  int n_cblk, n_chunks, splits;  // 256-column blocks, 64-row chunks, CTAs per block
  float* part;                    // (splits, B, N) fp32 partials when splits > 1
};

__host__ __device__ constexpr int gt_code_bytes(int cbytes, int R) { return R * (gt_k(R) / (16 / cbytes)) * 512; }
__host__ __device__ constexpr size_t gt_smem(int cbytes, int R, int BN) {
  return 1024 + (size_t)R * kBookBytes + (size_t)gt_stages(R) * gt_a_bytes(R) +
         (size_t)gt_x_stages(R, BN) * BN * 2 * gt_k(R) + (size_t)gt_code_stages(BN) * gt_code_bytes(cbytes, R) +
         (2 * gt_stages(R) + 2 * gt_x_stages(R, BN) + 2 * gt_code_stages(BN) + 4) * 8 + 16;
}

template <int CBYTES, int R, int BN>
__global__ void __launch_bounds__(kGtThreads, 1)
    gemv_tc_kernel(const __grid_constant__ CUtensorMap tmap_x, GemvTcArgs a) {
  constexpr int RPL = 16 / CBYTES;
  constexpr int CODEB = gt_code_bytes(CBYTES, R) / R;  // one level's code bytes per stage
  constexpr int GK = gt_k(R);
  constexpr int ABYTES = gt_a_bytes(R);
  constexpr int XB = BN * 2 * GK;                       // X tile bytes (GK / 64 SW128 boxes of BN rows)
  constexpr int STG = gt_stages(R);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  constexpr int CST = gt_code_stages(BN), XST = gt_x_stages(R, BN);
  uint8_t* sa = smem;                                   // STG x 32 KB (A: W^T tiles)
  uint8_t* sx = sa + STG * ABYTES;                   // XST x XB (B: X tiles)
  uint8_t* sc = sx + XST * XB;                          // CST x R x CODEB (code words)
  uint8_t* book = sc + CST * R * CODEB;                 // R x 256 entries x 128 B (replicated)
  uint64_t* bars = reinterpret_cast<uint64_t*>(book + R * kBookBytes);
  // afull[s] (A written), empty[s] (MMA done with A slot s), full[x] (X landed),
  // xempty[x] (MMA done with X slot x), cfull[c] (code words landed), cempty[c]
  // (producers read them), tfull (accumulator done)
  constexpr int NGRP = STG >= 2 ? STG / 2 : 1;  // producer groups, two A slots each (fill one while the MMA reads the other)
  constexpr int GW = kGtProd / NGRP;           // warps per producer group
  const uint32_t afull0 = smem_u32(bars), empty0 = smem_u32(bars + STG);
  const uint32_t full0 = smem_u32(bars + 2 * STG), xempty0 = smem_u32(bars + 2 * STG + XST);
  const uint32_t cfull0 = smem_u32(bars + 2 * STG + 2 * XST), cempty0 = smem_u32(bars + 2 * STG + 2 * XST + CST);
  const uint32_t tfull = smem_u32(bars + 2 * STG + 2 * XST + 2 * CST);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STG + 2 * XST + 2 * CST + 2);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cb = blockIdx.x / a.splits, ks = blockIdx.x % a.splits;
  const int c_lo = ks * a.n_chunks / a.splits, c_hi = (ks + 1) * a.n_chunks / a.splits;
  const int n = c_hi - c_lo;

  if (tid == 0) {
    for (int s = 0; s < STG; ++s) {
      mbar_init(afull0 + 8 * s, GW);
      mbar_init(empty0 + 8 * s, 1);
    }
    for (int x = 0; x < XST; ++x) {
      mbar_init(full0 + 8 * x, 1);
      mbar_init(xempty0 + 8 * x, 1);
    }
    for (int c = 0; c < CST; ++c) {
      mbar_init(cfull0 + 8 * c, 1);
      mbar_init(cempty0 + 8 * c, GW);
    }
    mbar_init(tfull, 1);
    mbar_fence_init();
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_x)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(2 * BN < 32 ? 32 : 2 * BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int idx = tid; idx < R * a.n_sh; idx += kGtThreads) {
    const int r = idx / a.n_sh, e = idx - r * a.n_sh;
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(a.books + ((int64_t)r * a.K + e) * 8));
    uint8_t* row = book + ((size_t)r * kBookEntries + e) * 128;
#pragma unroll
    for (int q = 0; q < 8; ++q) *reinterpret_cast<uint4*>(row + ((q + e) & 7) * 16) = v;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_launch_dependents();

  if (warp == 0) {
    // ===== TMA, two independent streams: lane 0 keeps CST chunks of code words in
    // flight (one bulk copy per level; codes do not depend on the previous kernel, so
    // the first ones go before griddepcontrol.wait), lane 1 the X tiles (the previous
    // kernel's output) STG chunks ahead of the MMA
    if (lane == 0) {
      for (int i = 0; i < n; ++i) {
        const int c = i % CST, ch = c_lo + i;
        if (i >= CST) mbar_wait(cempty0 + 8 * c, ((i / CST) & 1) ^ 1);
        mbar_arrive_expect_tx(cfull0 + 8 * c, (uint32_t)(R * CODEB));
        const int64_t off = (int64_t)cb * 32 * (a.M / RPL) * 16 + (int64_t)ch * (GK / RPL) * 512;
#pragma unroll
        for (int r = 0; r < R; ++r)
          tma_load_1d_hint(smem_u32(sc + (c * R + r) * CODEB), a.codes + r * a.level_bytes + off, CODEB, cfull0 + 8 * c, l2_evict_first());
      }
    } else if (lane == 1) {
      pdl_wait();
      for (int i = 0; i < n; ++i) {
        const int x = i % XST;
        if (i >= XST) mbar_wait(xempty0 + 8 * x, ((i / XST) & 1) ^ 1);
        mbar_arrive_expect_tx(full0 + 8 * x, (uint32_t)XB);
#pragma unroll
        for (int bx = 0; bx < GK / 64; ++bx)
          tma_load_2d(smem_u32(sx + x * XB + bx * BN * 128), &tmap_x, (c_lo + i) * GK + bx * 64, 0, full0 + 8 * x);
      }
    }
  } else if (warp == 1) {
    // ===== MMA issuer: per stage 2 halves x 4 K-steps of UMMA 128 x BN x 16
    // idesc: D f32, A/B f16, A MN-major (transposed), B K-major, N = BN, M = 128
    const uint32_t idesc = (1u << 4) | (1u << 15) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    if (lane == 0) {
      for (int i = 0; i < n; ++i) {
        const int s = i % STG, x = i % XST;
        mbar_wait(full0 + 8 * x, (i / XST) & 1);
        mbar_wait(afull0 + 8 * s, (i / STG) & 1);
        tc_fence_after();
        const uint32_t a_base = smem_u32(sa + s * ABYTES), x_base = smem_u32(sx + x * XB);
#pragma unroll
        for (int k = 0; k < GK / 16; ++k) {
          // X: K-step k lies in SW128 box k / 4 (BN rows x 128 B), 32 B per K-step inside it
          const uint64_t bdesc = umma_desc(x_base + (k >> 2) * BN * 128 + (k & 3) * 32, 16, 1024);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint64_t adesc = umma_desc(a_base + h * (ABYTES / 2) + k * 4096, 1024, 2048);
            umma_f16(tmem_base + h * BN, adesc, bdesc, idesc, (i | k) != 0);
          }
        }
        umma_commit(empty0 + 8 * s);
        umma_commit(xempty0 + 8 * x);
      }
      umma_commit(tfull);
    }
  } else if (warp < 2 + kGtProd) {
    // ===== dequantisation producers: a stage is 64 K-rows x 32 sub-vector groups;
    // group grp takes stages grp, grp + NGRP, ... (two A slots of its own)
    const int pw = warp - 2, grp = pw / GW;
    const int gtid = (pw % GW) * 32 + lane;
    constexpr int NPT = GW * 32;
    constexpr int WORDS = (GK / RPL) * 32;          // code words per level per stage
    constexpr int TPW = NPT >= WORDS ? NPT / WORDS : 1;  // threads per word
    constexpr int WPT = NPT >= WORDS ? 1 : WORDS / NPT;  // words per thread
    constexpr int KR = RPL / TPW;                   // rows per thread per word
    const uint32_t rep = (uint32_t)(lane & 7) * 16;
    for (int i = grp; i < n; i += NGRP) {
      const int s = i % STG, cs = i % CST;
      mbar_wait(cfull0 + 8 * cs, (i / CST) & 1);  // code words landed
      uint4 cw[WPT][R];
#pragma unroll
      for (int ww = 0; ww < WPT; ++ww) {
        const int w = (gtid + ww * NPT) % WORDS;
#pragma unroll
        for (int r = 0; r < R; ++r) cw[ww][r] = *reinterpret_cast<const uint4*>(sc + (cs * R + r) * CODEB + w * 16);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(cempty0 + 8 * cs);  // the code slot may be refilled
      if (i >= STG) mbar_wait(empty0 + 8 * s, ((i / STG) & 1) ^ 1);  // the MMA is done with A slot s
#pragma unroll
      for (int ww = 0; ww < WPT; ++ww) {
        const int idx = gtid + ww * NPT;
        const int w = idx % WORDS, part = (idx / WORDS) % TPW;
        const int gi = w % 32, rg = w / 32;
        const int h = gi >> 4, g16 = gi & 15, nb = g16 >> 3, c = g16 & 7;
        uint8_t* at = sa + s * ABYTES + h * (ABYTES / 2);
#pragma unroll
        for (int kk = 0; kk < KR; ++kk) {
          const int k = part * KR + kk;  // row within the word
          uint4 e;
#pragma unroll
          for (int r = 0; r < R; ++r) {
            uint32_t code;
            if constexpr (CBYTES == 2) {
              const uint32_t x = (&cw[ww][r].x)[k / 2];
              code = (k & 1) ? (x >> 16) : (x & 0xffffu);
            } else {
              code = ((&cw[ww][r].x)[k / 4] >> (8 * (k % 4))) & 0xffu;
            }
            const uint4 q = *reinterpret_cast<const uint4*>(book + ((size_t)r * kBookEntries + code) * 128 + rep);
            if (r == 0) {
              e = q;
            } else {
              uint32_t* ew = &e.x;
              const uint32_t* qw = &q.x;
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const __half2 hs = __hadd2(*reinterpret_cast<const __half2*>(&ew[j]), *reinterpret_cast<const __half2*>(&qw[j]));
                ew[j] = *reinterpret_cast<const uint32_t*>(&hs);
              }
            }
          }
          const int kr = rg * RPL + k;  // K-row within the stage
          *reinterpret_cast<uint4*>(at + ((kr >> 3) * 2 + nb) * 1024 + (kr & 7) * 128 + ((c ^ (kr & 7)) << 4)) = e;
        }
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(afull0 + 8 * s);
    }
  } else {
    // ===== epilogue: TMEM lanes = output columns, columns = batch rows (8 at a time);
    // y / the partials may still be read by the previous kernel
    pdl_wait();
    const int quarter = warp & 3;
    mbar_wait(tfull, 0);
    tc_fence_after();
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const int64_t ncol = (int64_t)cb * 256 + hh * 128 + quarter * 32 + lane;
      const uint32_t taddr = tmem_base + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(hh * BN);
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 8) {
        uint32_t r8[8];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(r8[0]), "=r"(r8[1]), "=r"(r8[2]), "=r"(r8[3]), "=r"(r8[4]), "=r"(r8[5]), "=r"(r8[6]),
                       "=r"(r8[7])
                     : "r"(taddr + c0));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int b = c0 + j;
          if (b < a.B) {
            const float v = __uint_as_float(r8[j]);
            if (a.splits == 1) store_from_f32(a.y, a.y_dtype, (int64_t)b * a.N + ncol, v);
            else a.part[((int64_t)ks * a.B + b) * a.N + ncol] = v;
          }
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(2 * BN < 32 ? 32 : 2 * BN));
  }
}

// ---------------------------------------------------------------------------
// Two-phase prefill (dequantise, then a dense tcgen05 GEMM). At prefill sizes the
// fused kernels above are shared-memory-bound: every W element costs an LDS gather
// and an STS into the UMMA layout on top of the tensor core's own operand traffic,
// and with AQLM's two levels (R = 2) the producers do twice the gathers. Written
// once to HBM as fp16 (the RN cast of the bit-exact fp32 dequantisation) and read
// back by TMA, the dequantised W costs 2 x M x N x 2 bytes of HBM traffic, which at
// rows >= 512 is cheaper than the fused producers' shared-memory time (DESIGN.md
// §3 GEMM; measured in bench.py's c3 / gemm_c2 keys).

// W (M, N) -> fp16/bf16 row-major straight from the GEMV_IL stream (N % 256 == 0, so
// 16-byte code word w of a level sits at byte 16 w and holds rows rg*RPL .. +RPL of
// sub-vector group cb*32 + gi, w = (cb * M/RPL + rg) * 32 + gi): one coalesced word
// load per level, then per row the summed entries (fp32, level order, one RN cast)
// as one 16-byte store; the 32 lanes of a warp cover one 512-byte row span
template <typename CB, int CBYTES, int R>
__global__ void __launch_bounds__(256) dequant_rows_kernel(const uint8_t* __restrict__ codes, int64_t level_bytes,
                                                           const CB* __restrict__ books, int K, int M, int N,
                                                           CB* __restrict__ out) {
  constexpr int RPL = 16 / CBYTES;
  pdl_launch_dependents();
  pdl_wait();
  const int64_t words = (int64_t)M / RPL * (N / 8);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int rgs = M / RPL;
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < words; w += stride) {
    const int gi = (int)(w & 31);
    const int64_t t = w >> 5;
    const int rg = (int)(t % rgs), cb = (int)(t / rgs);
    uint4 cw[R];
#pragma unroll
    for (int r = 0; r < R; ++r) cw[r] = ldg_stream(codes + r * level_bytes + w * 16);
    CB* o = out + (int64_t)rg * RPL * N + (int64_t)(cb * 32 + gi) * 8;
#pragma unroll
    for (int k = 0; k < RPL; ++k) {
      float acc[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] = 0.0f;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        uint32_t code;
        if constexpr (CBYTES == 2) {
          const uint32_t x = (&cw[r].x)[k / 2];
          code = (k & 1) ? (x >> 16) : (x & 0xffffu);
        } else {
          code = ((&cw[r].x)[k / 4] >> (8 * (k % 4))) & 0xffu;
        }
        const uint4 e = __ldg(reinterpret_cast<const uint4*>(books + ((int64_t)r * K + code) * 8));
        const CB* ep = reinterpret_cast<const CB*>(&e);
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] = __fadd_rn(acc[j], to_f32<CB>(ep[j]));
      }
      uint4 v;
      CB* vp = reinterpret_cast<CB*>(&v);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if constexpr (std::is_same<CB, __half>::value) vp[j] = __float2half_rn(acc[j]);
        else vp[j] = __float2bfloat16_rn(acc[j]);
      }
      *reinterpret_cast<uint4*>(o + (int64_t)k * N) = v;
    }
  }
}

// Dense CTA-pair GEMM: Y(rows, N) = X(rows, M) @ W(M, N) with both operands by TMA.
// UMMA 256 x 256 x 16 over the pair (each CTA: 128 X rows, 128 W columns as two
// 64-column SWIZZLE_128B boxes = the MN-major SW128 canonical layout). Tiles are
// ordered row-tile fastest, so the pairs working on one W column strip run together
// and the strip is read from HBM once (L2 serves the other row tiles).
constexpr int kDenseStages = 5;
constexpr int kDenseBBytes = kTileK * 128 * 2;  // this CTA's 128 columns x 64 K
constexpr size_t dense_smem() {
  return (size_t)kDenseStages * (kPairABytes + kDenseBBytes) + (2 * kDenseStages + 1) * 8 + 16 + 1024;
}

template <bool BF16, typename OutT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kGemmThreads, 1)
    gemm_dense_pair_kernel(const __grid_constant__ CUtensorMap tmap_x, const __grid_constant__ CUtensorMap tmap_w,
                           GemmArgs a) {
  constexpr int NT = 256, CN = 128, STG = kDenseStages;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sa = smem;
  uint8_t* sb = sa + STG * kPairABytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sb + STG * kDenseBBytes);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STG + 1);
  const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + STG), tmem_full = smem_u32(bars + 2 * STG);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t rank = cluster_ctarank();
  const int pair = blockIdx.x >> 1;
  const int n_tiles_m = (a.rows + 2 * kPairRowsCta - 1) / (2 * kPairRowsCta);
  const int tile_m = pair % n_tiles_m, tile_n = pair / n_tiles_m;
  const int row0 = tile_m * 2 * kPairRowsCta + (int)rank * kPairRowsCta;
  const int n0 = tile_n * NT + (int)rank * CN;
  const int k_iters = a.M / kTileK;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STG; ++s) {
      mbar_init(full0 + 8 * s, 1);   // the leader's expect_tx (both CTAs' A and B bytes)
      mbar_init(empty0 + 8 * s, 1);  // multicast tcgen05.commit
    }
    mbar_init(tmem_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_x)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_w)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(NT));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_launch_dependents();
  pdl_wait();  // W was dequantised by the preceding kernel

  if (warp == 0) {
    if (lane == 0) {
      const uint32_t bar_l = mapa_rank(full0, 0);
      for (int it = 0; it < k_iters; ++it) {
        const int s = it % STG;
        mbar_wait(empty0 + 8 * s, ((it / STG) & 1) ^ 1);
        if (rank == 0) mbar_arrive_expect_tx(full0 + 8 * s, 2 * (kPairABytes + kDenseBBytes));
        tma_load_2d_pair(smem_u32(sa + s * kPairABytes), &tmap_x, it * kTileK, row0, bar_l + 8 * s);
        tma_load_2d_pair(smem_u32(sb + s * kDenseBBytes), &tmap_w, n0, it * kTileK, bar_l + 8 * s);
        tma_load_2d_pair(smem_u32(sb + s * kDenseBBytes + kDenseBBytes / 2), &tmap_w, n0 + 64, it * kTileK,
                         bar_l + 8 * s);
      }
    }
  } else if (warp == 1) {
    const uint32_t fmt = BF16 ? 1u : 0u;
    const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | (0u << 15) | (1u << 16) |
                           ((uint32_t)(NT >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
    if (rank == 0 && lane == 0) {
      for (int it = 0; it < k_iters; ++it) {
        const int s = it % STG;
        mbar_wait(full0 + 8 * s, (it / STG) & 1);
        tc_fence_after();
        const uint32_t a_base = smem_u32(sa + s * kPairABytes), b_base = smem_u32(sb + s * kDenseBBytes);
#pragma unroll
        for (int k = 0; k < kTileK / 16; ++k) {
          // B: two 64-column boxes (8 KB apart = LBO), 8-row groups 1 KB apart (SBO)
          const uint64_t bdesc = umma_desc(b_base + k * 2 * 1024, kDenseBBytes / 2, 1024);
          const uint64_t adesc = umma_desc(a_base + k * 32, 16, 1024);
          umma_f16_pair(tmem_base, adesc, bdesc, idesc, (it | k) != 0);
        }
        umma_commit_pair(empty0 + 8 * s);
      }
      umma_commit_pair(tmem_full);
    }
  } else {
    // epilogue: this CTA's 128 rows x 256 columns of TMEM
    mbar_wait(tmem_full, 0);
    tc_fence_after();
    const int quarter = warp & 3;
    constexpr int CPW = (NT / 32) / (kProdWarps / 4);
    const int cc0 = ((warp - 2) / 4) * CPW;
    const int row = row0 + quarter * 32 + lane;
    const int ncol0 = tile_n * NT;
#pragma unroll
    for (int c2 = 0; c2 < CPW; ++c2) {
      const int cc = cc0 + c2;
      uint32_t v[32];
      const uint32_t taddr = tmem_base + ((uint32_t)(quarter * 32) << 16) + cc * 32;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
          "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
            "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
            "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
            "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (row < a.rows) store_row32<OutT>(a.y, a.y_dtype, (int64_t)row * a.N + ncol0 + cc * 32, v);
    }
  }

  tc_fence_before();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(NT));
  }
}

// ---------------------------------------------------------------------------
// host

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

static size_t gemm_smem(int R) {
  return (size_t)R * kBookBytes + gemm_stages(R) * (kABytes + kBBytes) + (3 * gemm_stages(R) + 1) * 8 + 16;
}

// split-K epilogue: y = sum over splits of the fp32 partials, in split order
__global__ void __launch_bounds__(256) gemm_splitk_reduce_kernel(const float* __restrict__ part, int splits,
                                                                 int64_t n_out, void* __restrict__ y, int y_dtype) {
  pdl_launch_dependents();
  pdl_wait();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < n_out; o += stride) {
    float acc = 0.f;
    for (int k = 0; k < splits; ++k) acc += part[(int64_t)k * n_out + o];
    store_from_f32(y, y_dtype, o, acc);
  }
}

// K splits for a grid of `tiles` output tiles (one CTA per SM): minimise the waves a
// split grid needs per unit of work, ceil(tiles * s / SMs) / s, at least 4 stages per
// split; ties to the smaller split (fewer partials)
// split-K factor minimising the wave-quantised time. Only for a single row tile
// (decode batches up to 256 rows): there the fp32 partials are small, while at
// prefill sizes they would cost more HBM traffic than the quantisation saves.
static int gemm_splits(int tiles, int k_total) {
  const int sms = sm_count();
  if (tiles >= 2 * sms) return 1;
  int best = 1;
  double best_t = 1e30;
  for (int sp = 1; sp <= std::min(16, std::max(1, k_total / 4)); ++sp) {
    const double t = (double)((tiles * sp + sms - 1) / sms) / sp;
    if (t < best_t - 1e-9) { best_t = t; best = sp; }
  }
  return best;
}

// the two-phase prefill path (dequantise to an fp16 scratch, dense CTA-pair GEMM):
// forced by VQB_FLAG_GEMM_TWO_PHASE, else the default for AQLM-style two-level
// codes at prefill sizes (measured faster than the fused producers)
static bool gemm_two_phase(const Geom& g, const VqbTensor* w, int64_t rows, const VqbLaunch* L) {
  if (g.ndim != 2 || g.v != 8 || g.cols % 256 != 0 || g.rows % kTileK != 0 || rows <= kTileM) return false;
  if (w->codebook_dtype == VQB_F32 || w->layout != VQB_LAYOUT_GEMV_IL || g.sharing != VQB_SHARE_WHOLE) return false;
  const int flags = L ? L->flags : 0;
  if (flags & (VQB_FLAG_FORCE_GENERIC | VQB_FLAG_NO_PAIR | VQB_FLAG_PAIR_N128 | VQB_FLAG_GEMM_FUSED)) return false;
  if (flags & VQB_FLAG_GEMM_TWO_PHASE) return true;
  return g.R == 2 && rows >= 512;
}

static int64_t a1k(int64_t x) { return (x + 1023) & ~int64_t(1023); }

int64_t gemm_ws_bytes(const VqbTensor* w, int64_t rows, const VqbLaunch* L) {
  Geom g;
  if (make_geom(w, &g)) return 0;
  if (gemm_two_phase(g, w, rows, L)) return VQB_WS_COUNTER_BYTES + a1k(g.rows * g.cols * 2);
  const int tiles = (int)(ceil_div(rows, kTileM) * (g.cols / kTileN));
  const int sp = g.cols % kTileN == 0 && g.rows % kTileK == 0 && rows <= kTileM
                     ? gemm_splits(std::max(tiles, 1), (int)(g.rows / kTileK))
                     : 1;
  return sp > 1 ? VQB_WS_COUNTER_BYTES + (int64_t)sp * rows * g.cols * 4 : 0;
}

static bool gemm_fast_ok(const Geom& g, const VqbTensor* w, int x_dtype, const VqbLaunch* L) {
  if (L && (L->flags & VQB_FLAG_FORCE_GENERIC)) return false;
  if (w->layout != VQB_LAYOUT_GEMV_IL || g.v != 8 || g.sharing != VQB_SHARE_WHOLE) return false;
  if (!(g.R == 1 || g.R == 2)) return false;
  if (!(g.bits == 8 || (g.bits == 16 && g.R == 1))) return false;
  if (!((w->codebook_dtype == VQB_F16 && x_dtype == VQB_F16) || (w->codebook_dtype == VQB_BF16 && x_dtype == VQB_BF16)))
    return false;
  if (g.rows % kTileK != 0 || g.cols % kTileN != 0) return false;
  return true;
}

template <int CBYTES, int R, bool BF16, typename OutT>
static int launch_gemm_t(const CUtensorMap& map, const GemmArgs& a, int grid, cudaStream_t st) {
  auto kern = gemm_tc_kernel<CBYTES, R, BF16, OutT>;
  const size_t smem = gemm_smem(R);
  // the attribute is per device: one guard per device ordinal
  static std::once_flag once[64];
  static cudaError_t attr_err[64] = {};
  int dev = 0;
  VQB_CUDA_CHECK(cudaGetDevice(&dev));
  dev &= 63;
  std::call_once(once[dev], [&] {
    attr_err[dev] = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  });
  if (attr_err[dev] != cudaSuccess) return cuda_error(attr_err[dev], "cudaFuncSetAttribute(gemm_tc_kernel)");
  kern<<<grid, kGemmThreads, smem, st>>>(map, a);
  VQB_LAUNCH_CHECK("gemm_tc_kernel");
  set_launch(grid, kGemmThreads, 256, 0);
  if (a.splits > 1) {
    const int64_t n_out = (int64_t)a.rows * a.N;
    const int blocks = (int)std::min<int64_t>(ceil_div(n_out, 256), (int64_t)sm_count() * 4);
    VQB_CUDA_CHECK(launch_pdl(gemm_splitk_reduce_kernel, dim3(blocks), dim3(256), 0, st,
                              static_cast<const float*>(a.part), a.splits, n_out, a.y, a.y_dtype));
  }
  set_kernel("gemm_tc");
  return VQB_OK;
}

template <int CBYTES, int R, bool BF16, typename OutT, int NT>
static int launch_pair_t(const CUtensorMap& map, const GemmArgs& a, int grid, cudaStream_t st) {
  auto kern = gemm_pair_kernel<CBYTES, R, BF16, OutT, NT>;
  const size_t smem = pair_smem(R, NT);
  static std::once_flag once[64];
  static cudaError_t attr_err[64] = {};
  int dev = 0;
  VQB_CUDA_CHECK(cudaGetDevice(&dev));
  dev &= 63;
  std::call_once(once[dev], [&] {
    attr_err[dev] = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  });
  if (attr_err[dev] != cudaSuccess) return cuda_error(attr_err[dev], "cudaFuncSetAttribute(gemm_pair_kernel)");
  kern<<<grid, kGemmThreads, smem, st>>>(map, a);  // cluster dims (2, 1, 1) from __cluster_dims__
  VQB_LAUNCH_CHECK("gemm_pair_kernel");
  set_launch(grid, kGemmThreads, 256, 0);
  set_kernel("gemm_tc2");
  return VQB_OK;
}

template <int CBYTES, int R, bool BF16, int NT>
static int launch_pair_out(const CUtensorMap& map, const GemmArgs& a, int grid, cudaStream_t st) {
  if (a.y_dtype == VQB_F32) return launch_pair_t<CBYTES, R, BF16, float, NT>(map, a, grid, st);
  if (a.y_dtype == VQB_F16) return launch_pair_t<CBYTES, R, BF16, __half, NT>(map, a, grid, st);
  return launch_pair_t<CBYTES, R, BF16, __nv_bfloat16, NT>(map, a, grid, st);
}

template <int CBYTES, int R, bool BF16>
static int launch_pair_nt(const CUtensorMap& map, const GemmArgs& a, int nt, cudaStream_t st) {
  const int grid = 2 * (int)(ceil_div(a.rows, 2 * kPairRowsCta) * (a.N / nt));
  return nt == 256 ? launch_pair_out<CBYTES, R, BF16, 256>(map, a, grid, st)
                   : launch_pair_out<CBYTES, R, BF16, 128>(map, a, grid, st);
}

template <int CBYTES, int R, bool BF16>
static int launch_gemm_out(const CUtensorMap& map, const GemmArgs& a, int grid, cudaStream_t st) {
  if (a.y_dtype == VQB_F32) return launch_gemm_t<CBYTES, R, BF16, float>(map, a, grid, st);
  if (a.y_dtype == VQB_F16) return launch_gemm_t<CBYTES, R, BF16, __half>(map, a, grid, st);
  return launch_gemm_t<CBYTES, R, BF16, __nv_bfloat16>(map, a, grid, st);
}

template <bool BF16, typename OutT>
static int launch_dense_pair(const CUtensorMap& mx, const CUtensorMap& mw, const GemmArgs& a, cudaStream_t st) {
  auto kern = gemm_dense_pair_kernel<BF16, OutT>;
  const size_t smem = dense_smem();
  static std::once_flag once[64];
  static cudaError_t attr_err[64] = {};
  int dev = 0;
  VQB_CUDA_CHECK(cudaGetDevice(&dev));
  dev &= 63;
  std::call_once(once[dev], [&] {
    attr_err[dev] = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  });
  if (attr_err[dev] != cudaSuccess) return cuda_error(attr_err[dev], "cudaFuncSetAttribute(gemm_dense_pair_kernel)");
  const int grid = 2 * (int)(ceil_div(a.rows, 2 * kPairRowsCta) * (a.N / 256));
  VQB_CUDA_CHECK(launch_pdl(kern, dim3(grid), dim3(kGemmThreads), smem, st, mx, mw, a));
  VQB_LAUNCH_CHECK("gemm_dense_pair_kernel");
  set_launch(grid, kGemmThreads, 0, 0);
  set_kernel("gemm_2phase");
  return VQB_OK;
}

// dequantise W into the scratch (fp16/bf16 row-major), then the dense pair GEMM
static int launch_two_phase(const Geom& g, const VqbTensor* w, const void* d_x, int x_dtype, const GemmArgs& a,
                            void* scratch, cudaStream_t st) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return set_error(VQB_ECUDA, "cuTensorMapEncodeTiled unavailable");
  const bool bf = w->codebook_dtype == VQB_BF16;
  const CUtensorMapDataType dt = bf ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  const cuuint32_t estr[2] = {1, 1};
  CUtensorMap mx, mw;
  const cuuint64_t xd[2] = {(cuuint64_t)g.rows, (cuuint64_t)a.rows};
  const cuuint64_t xs[1] = {(cuuint64_t)g.rows * 2};
  const cuuint32_t xb[2] = {(cuuint32_t)kTileK, (cuuint32_t)kPairRowsCta};
  CUresult cr = enc(&mx, dt, 2, const_cast<void*>(d_x), xd, xs, xb, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) return set_error(VQB_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)cr);
  const cuuint64_t wd[2] = {(cuuint64_t)g.cols, (cuuint64_t)g.rows};
  const cuuint64_t wsd[1] = {(cuuint64_t)g.cols * 2};
  const cuuint32_t wb[2] = {64u, (cuuint32_t)kTileK};
  cr = enc(&mw, dt, 2, scratch, wd, wsd, wb, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) return set_error(VQB_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)cr);
  (void)x_dtype;
  const int64_t words = g.rows / (16 / g.code_bytes) * (g.cols / 8);
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(ceil_div(words, 256), (int64_t)sm_count() * 8));
  const uint8_t* cp = reinterpret_cast<const uint8_t*>(w->d_codes);
  const int64_t lb = g.S * g.code_bytes;
  const int M = (int)g.rows, N = (int)g.cols, K = g.K;
#define VQB_DQ(CB, CBY, RR)                                                                                       \
  VQB_CUDA_CHECK(launch_pdl(dequant_rows_kernel<CB, CBY, RR>, dim3((unsigned)blocks), dim3(256), 0, st, cp, lb,   \
                            reinterpret_cast<const CB*>(w->d_codebooks), K, M, N, reinterpret_cast<CB*>(scratch)))
  if (bf) {
    if (g.code_bytes == 2) VQB_DQ(__nv_bfloat16, 2, 1);
    else if (g.R == 1) VQB_DQ(__nv_bfloat16, 1, 1);
    else VQB_DQ(__nv_bfloat16, 1, 2);
  } else {
    if (g.code_bytes == 2) VQB_DQ(__half, 2, 1);
    else if (g.R == 1) VQB_DQ(__half, 1, 1);
    else VQB_DQ(__half, 1, 2);
  }
#undef VQB_DQ
  VQB_LAUNCH_CHECK("dequant_rows_kernel");
  if (a.y_dtype == VQB_F32) return bf ? launch_dense_pair<true, float>(mx, mw, a, st) : launch_dense_pair<false, float>(mx, mw, a, st);
  if (a.y_dtype == VQB_F16) return bf ? launch_dense_pair<true, __half>(mx, mw, a, st) : launch_dense_pair<false, __half>(mx, mw, a, st);
  return bf ? launch_dense_pair<true, __nv_bfloat16>(mx, mw, a, st) : launch_dense_pair<false, __nv_bfloat16>(mx, mw, a, st);
}

template <int CBYTES, int R, int BN>
static int launch_gemv_tc_t(const CUtensorMap& mx, const GemvTcArgs& a, cudaStream_t st, int flags) {
  auto kern = gemv_tc_kernel<CBYTES, R, BN>;
  const size_t smem = gt_smem(CBYTES, R, BN);
  static std::once_flag once[64];
  static cudaError_t attr_err[64] = {};
  int dev = 0;
  VQB_CUDA_CHECK(cudaGetDevice(&dev));
  dev &= 63;
  std::call_once(once[dev], [&] {
    attr_err[dev] = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  });
  if (attr_err[dev] != cudaSuccess) return cuda_error(attr_err[dev], "cudaFuncSetAttribute(gemv_tc_kernel)");
  const int grid = a.n_cblk * a.splits;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kGtThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (flags & VQB_FLAG_NO_PDL) ? 0 : 1;
  VQB_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, mx, a));
  if (a.splits > 1) {
    const int64_t n_out = (int64_t)a.B * a.N;
    const int blocks = (int)std::min<int64_t>(ceil_div(n_out, 256), (int64_t)sm_count() * 4);
    VQB_CUDA_CHECK(launch_pdl(gemm_splitk_reduce_kernel, dim3(blocks), dim3(256), 0, st,
                              static_cast<const float*>(a.part), a.splits, n_out, a.y, a.y_dtype));
  }
  set_kernel("gemv_tc");
  set_launch(grid, kGtThreads, a.n_sh, 0);
  return VQB_OK;
}

// K splits of the tcgen05 GEMV: one wave of CTAs over the column blocks
static int gemv_tc_splits(int n_cblk, int n_chunks, int rows, int64_t N) {
  // modelled time: waves x chunks per CTA x ~0.75 us per 64-row chunk, plus (split) the
  // fp32 partials written and read back (~5 TB/s) and the reduce launch (~2 us)
  const int sms = sm_count();
  int best = 1;
  double best_t = 1e30;
  for (int sp = 1; sp <= std::max(1, n_chunks / 4); ++sp) {
    const double waves = (double)((n_cblk * sp + sms - 1) / sms);
    double t = waves * (double)((n_chunks + sp - 1) / sp) * 0.75;
    if (sp > 1) t += (double)sp * rows * N * 8 / 5e6 + 2.0;
    if (t < best_t - 1e-9) { best_t = t; best = sp; }
  }
  return best;
}

static bool gemv_tc_covers(const Geom& g, const VqbTensor* w, int x_dtype, int rows, const VqbLaunch* L) {
  const int flags = L ? L->flags : 0;
  if (flags & (VQB_FLAG_FORCE_GENERIC | VQB_FLAG_NO_GEMV_TC)) return false;
  if (rows < 2 || rows > 64 || x_dtype != VQB_F16 || w->codebook_dtype != VQB_F16) return false;
  if (w->layout != VQB_LAYOUT_GEMV_IL || g.v != 8 || g.sharing != VQB_SHARE_WHOLE || g.ndim != 2) return false;
  if (!(g.R == 1 || g.R == 2) || !(g.bits == 8 || (g.bits == 16 && g.R == 1))) return false;
  if (g.cols % 256 != 0 || g.rows % gt_k(g.R) != 0) return false;
  // every code must be resident in the 256-entry shared table
  if (!(g.K <= 256 || (w->max_code >= 0 && w->max_code < 256))) return false;
  // default: batches from kGemvTcMinRows, and every batch the CUDA-core / mma.sync
  // kernels do not cover (3, 5-7)
  return (flags & VQB_FLAG_GEMV_TC) || rows >= kGemvTcMinRows || !(rows == 1 || rows == 2 || rows == 4 || rows == 8);
}

int64_t gemv_tc_ws_bytes(const Geom& g, const VqbTensor* w, int rows, const VqbLaunch* L) {
  if (!gemv_tc_covers(g, w, VQB_F16, rows, L)) return 0;
  const int sp = gemv_tc_splits((int)(g.cols / 256), (int)(g.rows / gt_k(g.R)), rows, g.cols);
  return VQB_WS_COUNTER_BYTES + (sp > 1 ? (int64_t)sp * rows * g.cols * 4 : 0);
}

// Decode GEMV on tcgen05 for batches 4-64 (gemv.cu dispatches here). Returns 1 when
// the configuration is not covered (the caller keeps its own kernels).
int gemv_tc_dispatch(const Geom& g, const VqbTensor* w, const void* x, int x_dtype, int rows, void* y, int y_dtype,
                     const VqbLaunch* L, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (!gemv_tc_covers(g, w, x_dtype, rows, L) || (reinterpret_cast<uintptr_t>(x) & 15)) return 1;
  const int flags = L ? L->flags : 0;
  const int BN = rows <= 8 ? 8 : rows <= 16 ? 16 : rows <= 32 ? 32 : 64;
  GemvTcArgs a;
  a.n_cblk = (int)(g.cols / 256);
  a.n_chunks = (int)(g.rows / gt_k(g.R));
  a.splits = gemv_tc_splits(a.n_cblk, a.n_chunks, rows, g.cols);
  const int64_t need = VQB_WS_COUNTER_BYTES + (a.splits > 1 ? (int64_t)a.splits * rows * g.cols * 4 : 0);
  if (!ws || (int64_t)ws_bytes < need)
    return set_error(VQB_ECAPACITY, "tcgen05 GEMV workspace too small: %zu < %lld", ws_bytes, (long long)need);
  EncodeTiledFn enc = encode_fn();
  if (!enc) return set_error(VQB_ECUDA, "cuTensorMapEncodeTiled unavailable");
  CUtensorMap mx;
  const cuuint64_t dims[2] = {(cuuint64_t)g.rows, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)g.rows * 2};
  const cuuint32_t box[2] = {64u, (cuuint32_t)BN};
  const cuuint32_t estr[2] = {1, 1};
  CUresult cr = enc(&mx, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(x), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) return set_error(VQB_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)cr);
  a.codes = reinterpret_cast<const uint8_t*>(w->d_codes);
  a.level_bytes = g.S * g.code_bytes;
  a.books = reinterpret_cast<const uint16_t*>(w->d_codebooks);
  a.y = y;
  a.y_dtype = y_dtype;
  a.B = rows;
  a.M = (int)g.rows;
  a.N = (int)g.cols;
  a.K = g.K;
  a.n_sh = std::min(g.K, kBookEntries);
  a.part = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ws) + VQB_WS_COUNTER_BYTES);
#define VQB_GT(CBY, RR)                                                     \
  switch (BN) {                                                             \
    case 8: return launch_gemv_tc_t<CBY, RR, 8>(mx, a, st, flags);           \
    case 16: return launch_gemv_tc_t<CBY, RR, 16>(mx, a, st, flags);         \
    case 32: return launch_gemv_tc_t<CBY, RR, 32>(mx, a, st, flags);         \
    default: return launch_gemv_tc_t<CBY, RR, 64>(mx, a, st, flags);         \
  }
  if (g.code_bytes == 2) { VQB_GT(2, 1) }
  if (g.R == 1) { VQB_GT(1, 1) }
  VQB_GT(1, 2)
#undef VQB_GT
}

int gemm_usage(VqbUsage* u) {
  cudaFuncAttributes at;
  auto k = gemm_tc_kernel<2, 1, false, float>;
  VQB_CUDA_CHECK(cudaFuncGetAttributes(&at, k));
  u->shared_bytes = (int)(at.sharedSizeBytes + gemm_smem(1));
  u->regs_per_thread = at.numRegs;
  u->threads_per_block = kGemmThreads;
  u->max_blocks_per_sm = 1;
  return VQB_OK;
}

}  // namespace vqb

using namespace vqb;

extern "C" int vqb_gemm(const VqbTensor* w, const void* d_x, int32_t x_dtype, int32_t rows, void* d_y,
                        int32_t y_dtype, const VqbLaunch* launch, void* d_ws, size_t ws_bytes, void* stream) {
  Geom g;
  int s = make_geom(w, &g);
  if (s) return s;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (g.ndim == 2 && rows >= 1 && y_dtype >= VQB_F32 && y_dtype <= VQB_BF16 && gemm_fast_ok(g, w, x_dtype, launch)) {
    EncodeTiledFn enc = encode_fn();
    if (!enc) return set_error(VQB_ECUDA, "cuTensorMapEncodeTiled unavailable");
    CUtensorMap map;
    const cuuint64_t dims[2] = {(cuuint64_t)g.rows, (cuuint64_t)rows};          // {K = M, rows}
    const cuuint64_t strides[1] = {(cuuint64_t)g.rows * 2};                      // bytes between rows
    const cuuint32_t box[2] = {(cuuint32_t)kTileK, (cuuint32_t)kTileM};
    const cuuint32_t estr[2] = {1, 1};
    CUresult cr = enc(&map, x_dtype == VQB_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2,
                      const_cast<void*>(d_x), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) return set_error(VQB_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)cr);
    GemmArgs a;
    a.codes = reinterpret_cast<const uint8_t*>(w->d_codes);
    a.level_bytes = g.S * g.code_bytes;
    a.books = reinterpret_cast<const uint16_t*>(w->d_codebooks);
    a.y = d_y;
    a.y_dtype = y_dtype;
    a.rows = rows;
    a.M = (int)g.rows;
    a.N = (int)g.cols;
    a.G = (int)g.gpr;
    a.K = g.K;
    a.n_sh = std::min(g.K, kBookEntries);
    const int tiles = (int)(ceil_div(rows, kTileM) * (g.cols / kTileN));
    a.splits = rows <= kTileM ? gemm_splits(tiles, (int)(g.rows / kTileK)) : 1;
    a.part = nullptr;
    if (a.splits > 1) {
      const int64_t need = VQB_WS_COUNTER_BYTES + (int64_t)a.splits * rows * g.cols * 4;
      if (!d_ws || (int64_t)ws_bytes < need) {
        a.splits = 1;  // no room for partials: one CTA per tile
      } else {
        a.part = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(d_ws) + VQB_WS_COUNTER_BYTES);
      }
    }
    const bool bf = w->codebook_dtype == VQB_BF16;
    if (a.splits == 1 && gemm_two_phase(g, w, rows, launch)) {
      const int64_t need = VQB_WS_COUNTER_BYTES + a1k(g.rows * g.cols * 2);
      if (!d_ws || (int64_t)ws_bytes < need)
        return set_error(VQB_ECAPACITY, "two-phase GEMM workspace too small: %zu < %lld", ws_bytes, (long long)need);
      void* scratch = reinterpret_cast<uint8_t*>(d_ws) + VQB_WS_COUNTER_BYTES;
      return launch_two_phase(g, w, d_x, x_dtype, a, scratch, st);
    }
    // prefill sizes (no split-K): the CTA-pair kernel with 256 x 256 tiles
    // (VQB_FLAG_NO_PAIR keeps the one-CTA kernel)
    // (measured: the pair kernel's 256 x 128 tiles run at ~500 TFLOP/s, latency-bound
    // on the per-stage cross-CTA handshake with only 256 MMA cycles per stage, so
    // they are used only where 256-wide tiles do not divide N; VQB_FLAG_PAIR_N128
    // forces them)
    const bool pair_ok = a.splits == 1 && g.cols % 128 == 0 && !(launch && (launch->flags & VQB_FLAG_NO_PAIR));
    const bool force128 = launch && (launch->flags & VQB_FLAG_PAIR_N128);
    if (pair_ok && (g.cols % 256 == 0 || force128)) {
      const int nt = (g.cols % 256 == 0 && !force128) ? 256 : 128;
      CUtensorMap map2;
      const cuuint32_t box2[2] = {(cuuint32_t)kTileK, (cuuint32_t)kPairRowsCta};
      cr = enc(&map2, x_dtype == VQB_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2,
               const_cast<void*>(d_x), dims, strides, box2, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (cr != CUDA_SUCCESS) return set_error(VQB_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)cr);
      if (g.bits == 16) return bf ? launch_pair_nt<2, 1, true>(map2, a, nt, st) : launch_pair_nt<2, 1, false>(map2, a, nt, st);
      if (g.R == 1) return bf ? launch_pair_nt<1, 1, true>(map2, a, nt, st) : launch_pair_nt<1, 1, false>(map2, a, nt, st);
      return bf ? launch_pair_nt<1, 2, true>(map2, a, nt, st) : launch_pair_nt<1, 2, false>(map2, a, nt, st);
    }
    const int grid = tiles * a.splits;
    if (g.bits == 16) return bf ? launch_gemm_out<2, 1, true>(map, a, grid, st) : launch_gemm_out<2, 1, false>(map, a, grid, st);
    if (g.R == 1) return bf ? launch_gemm_out<1, 1, true>(map, a, grid, st) : launch_gemm_out<1, 1, false>(map, a, grid, st);
    return bf ? launch_gemm_out<1, 2, true>(map, a, grid, st) : launch_gemm_out<1, 2, false>(map, a, grid, st);
  }
  VqbLaunch l = launch ? *launch : VqbLaunch{};
  l.flags |= VQB_FLAG_FORCE_GENERIC;
  return gemv_dispatch(w, d_x, x_dtype, rows, d_y, y_dtype, &l, d_ws, ws_bytes, st, nullptr, nullptr, 0, nullptr);
}
