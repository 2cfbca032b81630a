// attn.cu — fused decode attention over a VQ-compressed (CQ) KV cache.
//
// Replaces SimMachine._attention / _attention_naive / _attention_centric
// (pkg/src/vqforge/sim.py:491-693) for ComputeOp.attention_decode
// (dataflow.py:77-82). Oracle: reference_compute (sim.py:145-155):
//   logits = (q . K_t) / sqrt(C); p = softmax(logits); out = sum_t p_t V_t.
//
// Fast kernel (channel-group sharing with group_width == v, one residual level,
// u8 codes, fp16 codebooks, KV_IL layout, C/v in {32, 64}, T % 32 == 0):
//  * codebook-centric dataflow: work units (h, b, 512-token chunk) are ordered
//    head-major and dealt out as contiguous ranges to persistent CTAs (one per
//    SM), so a CTA loads the K and V codebooks of a head once (CQ books are per
//    head, shared by all batch rows and tokens, codec.py:161-165) and reuses
//    them for every batch row of that head.
//  * K side as a lookup table: q is fixed per (b, h), so the CTA builds
//    LUT[e][g] = log2(e)/sqrt(C) * <q_g, K_book_g[e]> once per (b, h); a token's
//    logit is sum_g LUT[code_g][g]: one LDS.32 + FADD per code, no dequantise.
//  * bank-conflict-free by construction: lane (h, ll) = (lane / 8, lane % 8) owns
//    channel groups g = ll + 8 (j ^ h); the LUT and the V book are stored
//    [entry][group], so in every shared load the 32 lanes hit 32 distinct banks
//    (g mod 32) whatever their codes are. With a 256-byte row the shared address is
//    a single PRMT of the code byte and the lane's column (plus the region base).
//  * select-free logit reduction: in the KV_IL layout a set of 8 lanes spans a token's
//    groups and lane (h, ll) stores token 8h + (i ^ ll) in slot i, so the 8x8
//    transpose-reduction inside each set is 7 shuffle+add pairs with no selects,
//    leaving lane l with token l's logit (24 fewer shuffles per 32 tokens than
//    spanning the groups over the whole warp).
//  * online softmax (flash-decode) in the exp2 domain; V is dequantised in
//    registers and fused into fp32 accumulators with fma.rn.f32.f16.
//  * the next 32-token batch's K codes load during the V phase, its V codes during
//    the next K phase (one register set, 16 warps), with L2 bulk prefetch ahead.
//  * split-T partials (m, l, acc) of a (b, h) cut across CTAs travel as tagged
//    64-bit words (no fence, no counter) to the CTA holding its first chunk, which
//    merges them in T order (deterministic), like the reference's split reduction
//    (sim.py:604-620).
// Generic path: dequantise K and V to fp32 (vqb_dequant) and run a plain fp32
// decode attention; covers every other configuration.
#include <cfloat>

#include "common.cuh"

namespace vqb {

int launch_dequant(const Geom& g, const VqbTensor* t, void* out, int out_dtype, cudaStream_t st);

constexpr int kAttnWarps = 16;  // 16 x 32 threads: 128 registers with one code register set per stream
constexpr int kAttnThreads = kAttnWarps * 32;
constexpr int kAttnChunk = 512;  // tokens per work unit
constexpr int64_t kAttnSlotOffset = 65536;  // tagged span slots in the self-resetting workspace head

struct AttnArgs {
  const uint8_t* kc;
  const uint8_t* vc;
  const __half* kb;
  const __half* vb;
  const __half* kbt;  // optional per-head [H][256][G][V] copies: one bulk copy per head
  const __half* vbt;
  const void* q;
  int q_dtype;
  void* out;
  int out_dtype;
  unsigned long long* slots;  // (grid, C + 2) tagged {m, l, acc} of a CTA's leading partial span; zero between launches
  int B, H, T, NT;       // valid tokens and 512-token chunks (when len_ptr is null)
  int T_cap, NT_cap;      // cache capacity (layout stride) and its chunk count
  const int* len_ptr;     // optional device-resident valid length (decode loops in CUDA graphs)
  float scale_log2;
  unsigned long long* trace;  // debug (VqbLaunch.flags & 32): per-CTA phase timestamps, 8 per CTA
  // fused decode front end (vqb_attn_decode_append): q, k, v come raw from the fused qkv
  // projection (B, 3*H*C); q is roped by every CTA of its (b, h), and the CTA whose span
  // holds position len-1 ropes k and quantizes the new K and V rows against the books
  // it already has in shared memory (the qkv_rope_append arithmetic), writing the codes
  // into the caches before it streams that token
  const __half* qkv;
  float log2_theta;
  uint8_t* kc_w;
  uint8_t* vc_w;
};

// per-CTA phase sums: slot 2 prologue (books + LUT), 3 streaming, 4 merge, 6 spans
struct AttnPhase {
  unsigned long long t = 0, sum[3] = {0, 0, 0};
  int spans = 0;
  __device__ __forceinline__ void mark(const AttnArgs& a, int phase) {
    if (a.trace && threadIdx.x == 0) {
      const unsigned long long n = gtimer();
      if (phase >= 0) sum[phase] += n - t;
      else ++spans;
      t = n;
    }
  }
  __device__ __forceinline__ void flush(const AttnArgs& a) {
    if (a.trace && threadIdx.x == 0) {
      for (int i = 0; i < 3; ++i) a.trace[blockIdx.x * 8 + 2 + i] = sum[i];
      a.trace[blockIdx.x * 8 + 6] = spans;
    }
  }
};

__device__ __forceinline__ void attn_trace(const AttnArgs& a, int slot) {
  if (a.trace && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    a.trace[blockIdx.x * 8 + slot] = t;
  }
}

template <int V, int GPL>
struct AttnSmem {
  static constexpr int G = 32 * GPL;
  static constexpr int C = G * V;
  static constexpr int EPB = 2 * V;                        // fp16 entry bytes
  // The LUT ([256][G] fp32) and the V book ([256][G] x V halves) each sit in a
  // 64 KB region starting at a 64 KB-aligned *shared-window* address, so a shared
  // address is one PRMT of (column, code, region high bytes). The dynamic base is
  // only known at run time (1 KB on B200), hence the slack of one region.
  static constexpr size_t region = 65536;
  // merge scratch, then each warp's 32 token probabilities (fp16, the V phase's
  // broadcast), then the book mbarrier
  static constexpr size_t pbuf_off = ((((size_t)kAttnWarps * (C + 2) + C + 1) * 4) + 63) & ~(size_t)63;
  static constexpr size_t scratch_bytes = pbuf_off + (size_t)kAttnWarps * 64 + 16;
  static constexpr size_t total = 3 * region + scratch_bytes;
  static_assert(256 * G * 4 <= region && 256 * G * EPB <= region, "region overflow");
};

// RoPE (rotate-half) of channel c at position pos, fp32 angle like the HF rotary
// embedding — the arithmetic of decode.cu's rope kernels
__device__ __forceinline__ float rope_channel_attn(const __half* x, int c, int C, float log2_theta, int pos) {
  const int half = C / 2;
  const int i = c < half ? c : c - half;
  const float inv_freq = exp2f(-log2_theta * (2.0f * i) / (float)C);
  float sn, cs;
  sincosf((float)pos * inv_freq, &sn, &cs);
  const float x0 = __half2float(x[i]), x1 = __half2float(x[i + half]);
  return c < half ? x0 * cs - x1 * sn : x1 * cs + x0 * sn;
}

__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}

// Shared address of row `code` (byte k of `w`) in a table with ROWB-byte rows,
// at column `col` of a region starting at `base`. With 256-byte rows and a
// 64 KB-aligned base this is ONE prmt: [col, code, base>>16 (2 bytes)].
template <int ROWB, bool PRMT>
__device__ __forceinline__ uint32_t row_addr(uint32_t w, int k, uint32_t colbase, uint32_t col, uint32_t base) {
  if constexpr (PRMT && ROWB == 256) {
    return prmt(w, colbase, 0x7604u | ((uint32_t)k << 4));
  } else {
    const uint32_t code = (w >> (8 * k)) & 0xffu;
    return base + code * ROWB + col;
  }
}

// A warp's 32-token batch of K and V codes (KV_IL: 2*GPL 16-byte words per lane each).
// (the batch holding a token appended by this kernel is read from L2 with ld.global.cg:
// the non-coherent streaming path may not see the kernel's own writes)
template <int V, int GPL>
__device__ __forceinline__ void attn_load_batch(const AttnArgs& a, int bh, int t0, uint4 (&kc)[2 * GPL],
                                                uint4 (&vc)[2 * GPL], bool fresh = false) {
  constexpr int G = 32 * GPL;
  const int lane = threadIdx.x & 31;
  const int64_t base = (int64_t)bh * a.T_cap * G + (int64_t)(t0 / 32) * 32 * G + lane * 16;
#pragma unroll
  for (int q = 0; q < 2 * GPL; ++q) {
    if (fresh) {
      kc[q] = __ldcg(reinterpret_cast<const uint4*>(a.kc + base + q * 512));
      vc[q] = __ldcg(reinterpret_cast<const uint4*>(a.vc + base + q * 512));
    } else {
      kc[q] = ldg_stream(a.kc + base + q * 512);
      vc[q] = ldg_stream(a.vc + base + q * 512);
    }
  }
}

template <int V, int GPL, bool PRMT, bool APPEND>
__device__ __forceinline__ void attn_stream_span(const AttnArgs& a, int T, int bh, int tok0, int tok1, uint32_t lut_base,
                                                 uint32_t vbook_base, float& m_w, float& l_lane,
                                                 float (&acc)[32 * GPL / kKvLanes][V], uint4 (&ka)[2 * GPL],
                                                 uint4 (&va)[2 * GPL], int fresh_t0, uint32_t pbuf) {
  using SM = AttnSmem<V, GPL>;
  constexpr int G = SM::G, EPB = SM::EPB;
  constexpr int Q = 2 * GPL;    // 16-byte loads per lane per 32-token batch
  constexpr int LPT = kKvLanes;  // lanes spanning one token's G groups (KV_IL)
  constexpr int NS = LPT;        // slots (tokens) per lane per 32-token batch
  constexpr int GPH = G / LPT;   // groups per lane
  static_assert(GPH * 32 / LPT >= 32 / LPT && (GPH & (GPH - 1)) == 0 && GPH >= 32 / LPT, "KV_IL lane sets");
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int hh = lane / LPT, ll = lane % LPT;
  const int64_t TG = (int64_t)a.T_cap * G;
  const uint8_t* kbase = a.kc + (int64_t)bh * TG;
  const uint8_t* vbase = a.vc + (int64_t)bh * TG;
  // per-lane columns (and, for the single-prmt form, the region's high address bytes)
  uint32_t colK[GPH], colV[GPH], cbK[GPH], cbV[GPH];
#pragma unroll
  for (int j = 0; j < GPH; ++j) {
    colK[j] = (uint32_t)(ll + LPT * (j ^ hh)) * 4;
    colV[j] = (uint32_t)(ll + LPT * (j ^ hh)) * EPB;
    cbK[j] = (lut_base & 0xffff0000u) | colK[j];
    cbV[j] = (vbook_base & 0xffff0000u) | colV[j];
  }
  // L2 prefetch of a later batch (one bulk prefetch of each 2*GPL x 512-byte run):
  // the register set alone keeps too few bytes in flight to cover the HBM latency,
  // so the batches PF_AHEAD strides ahead are pulled into L2 meanwhile
  auto prefetch = [&](int t0) {
    if (lane == 0 && t0 < tok1) {
      const int64_t off = (int64_t)(t0 / 32) * 32 * G;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(kbase + off), "r"(Q * 512) : "memory");
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(vbase + off), "r"(Q * 512) : "memory");
    }
  };
  // K phase + online-softmax update of one 32-token batch; lane l stores token l's
  // probability (fp16) in the warp's pbuf for the V phase
  auto kphase = [&](const uint4 (&kc)[Q], int tb) {
    // lane partial logits for its NS slots (slot i = token LPT hh + (i ^ ll))
    auto partial = [&](int i) {
      float acc_s = 0.f;
#pragma unroll
      for (int j = 0; j < GPH; ++j) {
        const int byte = i * GPH + j;
        const uint32_t w = (&kc[byte / 16].x)[(byte % 16) / 4];
        const float lv = lds_f32(row_addr<G * 4, PRMT>(w, byte % 4, cbK[j], colK[j], lut_base));
        acc_s = (j == 0) ? lv : acc_s + lv;
      }
      return acc_s;
    };
    // select-free transpose-reduction inside each lane set: afterwards s[0] on lane l
    // is token l's logit. The first (offset NS/2) step is fused into the partial
    // computation so only NS/2 partial logits are ever live; NS-1 shuffles per batch.
    float s[NS / 2];
#pragma unroll
    for (int i = 0; i < NS / 2; ++i) {
      const float lo = partial(i), hi = partial(i + NS / 2);
      s[i] = lo + __shfl_xor_sync(0xffffffffu, hi, NS / 2);
    }
#pragma unroll
    for (int off = NS / 4; off >= 1; off >>= 1)
#pragma unroll
      for (int i = 0; i < off; ++i) s[i] += __shfl_xor_sync(0xffffffffu, s[i + off], off);
    // tokens past the valid length (a partial last batch) get p = 0
    const float z = (tb + lane < T) ? s[0] : -INFINITY;
    // the running max moves only when some logit exceeds it (rarer as the span goes
    // on): one vote instead of the 5-level max tree and the rescale. Bit-identical —
    // the skipped path would compute corr = exp2(0) = 1.
    float corr = 1.f;
    if (__any_sync(0xffffffffu, z > m_w)) {
      float mb = z;
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) mb = fmaxf(mb, __shfl_xor_sync(0xffffffffu, mb, off));
      const float m_new = fmaxf(m_w, mb);
      corr = fast_exp2(m_w - m_new);
      m_w = m_new;
#pragma unroll
      for (int j = 0; j < GPH; ++j)
#pragma unroll
        for (int c = 0; c < V; ++c) acc[j][c] *= corr;
    }
    const float p = fast_exp2(z - m_w);
    l_lane = l_lane * corr + p;
    __syncwarp();  // every lane has read the previous batch's probabilities
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(pbuf + lane * 2), "h"(__half_as_ushort(__float2half_rn(p))) : "memory");
    __syncwarp();
  };
  // V phase: slot i holds token LPT hh + (i ^ ll). Slots 4k..4k+3 hold tokens
  // LPT hh + 4(k ^ (ll >> 2)) + (r ^ (ll & 3)), so one 8-byte broadcast read of pbuf
  // serves four slots and a PRMT (per-lane selector of half r ^ (ll & 3)) makes each
  // slot's (p, p) pair: NS/4 LDS instead of NS shuffles per batch — the MIO pipe
  // (shared loads and shuffles) is what bounds this kernel.
  // p * V accumulates in packed fp16x2 windows of 8 tokens (HFMA2, full rate; the
  // mixed-precision fp32 FMA is quarter rate), flushed into the fp32 accumulators
  // with an exact widening FMA — the GEMV's windowing, at attention's 2e-3 bound.
  uint32_t psel[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const uint32_t h2 = 2u * (uint32_t)(r ^ (lane & 3));
    psel[r] = h2 | ((h2 + 1) << 4) | (h2 << 8) | ((h2 + 1) << 12);
  }
  const uint32_t pb_lane = pbuf + (uint32_t)hh * (2 * LPT) + (uint32_t)(ll >> 2) * 8;  // pbuf is 64-byte aligned
  auto vphase = [&](const uint4 (&vc)[Q]) {
    constexpr int HW = V / 2;  // fp16x2 words per entry
    uint2 pv = make_uint2(0u, 0u);
#pragma unroll
    for (int w8 = 0; w8 < NS / 8; ++w8) {
      uint32_t hw[GPH][HW];
#pragma unroll
      for (int j = 0; j < GPH; ++j)
#pragma unroll
        for (int c = 0; c < HW; ++c) hw[j][c] = 0u;
#pragma unroll
      for (int ii = 0; ii < 8; ++ii) {
        const int i = w8 * 8 + ii;
        if ((i & 3) == 0) pv = lds64(pb_lane ^ (uint32_t)((i >> 2) * 8));
        const uint32_t pp = prmt(pv.x, pv.y, psel[i & 3]);
#pragma unroll
        for (int j = 0; j < GPH; ++j) {
          const int byte = i * GPH + j;
          const uint32_t w = (&vc[byte / 16].x)[(byte % 16) / 4];
          const uint32_t addr = row_addr<G * EPB, PRMT>(w, byte % 4, cbV[j], colV[j], vbook_base);
          if constexpr (V == 2) {
            const uint32_t e = lds32(addr);
            asm("fma.rn.f16x2 %0, %1, %2, %0;" : "+r"(hw[j][0]) : "r"(e), "r"(pp));
          } else {
            const uint2 e = lds64(addr);
            asm("fma.rn.f16x2 %0, %1, %2, %0;" : "+r"(hw[j][0]) : "r"(e.x), "r"(pp));
            asm("fma.rn.f16x2 %0, %1, %2, %0;" : "+r"(hw[j][1]) : "r"(e.y), "r"(pp));
          }
        }
      }
#pragma unroll
      for (int j = 0; j < GPH; ++j)
#pragma unroll
        for (int c = 0; c < HW; ++c) {
          acc[j][2 * c] = fma_h((uint16_t)(hw[j][c] & 0xffff), (uint16_t)0x3C00, acc[j][2 * c]);
          acc[j][2 * c + 1] = fma_h((uint16_t)(hw[j][c] >> 16), (uint16_t)0x3C00, acc[j][2 * c + 1]);
        }
    }
  };
  auto load_k = [&](uint4 (&kc)[Q], int t0) {
    const int64_t off = (int64_t)(t0 / 32) * 32 * G + lane * 16;
#pragma unroll
    for (int q = 0; q < Q; ++q)
      kc[q] = (APPEND && t0 == fresh_t0) ? __ldcg(reinterpret_cast<const uint4*>(kbase + off + q * 512))
                                         : ldg_stream(kbase + off + q * 512);
  };
  auto load_v = [&](uint4 (&vc)[Q], int t0) {
    const int64_t off = (int64_t)(t0 / 32) * 32 * G + lane * 16;
#pragma unroll
    for (int q = 0; q < Q; ++q)
      vc[q] = (APPEND && t0 == fresh_t0) ? __ldcg(reinterpret_cast<const uint4*>(vbase + off + q * 512))
                                         : ldg_stream(vbase + off + q * 512);
  };
  // warp w takes 32-token batches w, w+kAttnWarps, ... of the span. One register set
  // per stream: the next batch's K codes load during this batch's V phase and its V
  // codes during the next K phase (the first batch (ka, va) was loaded by the caller).
  int t0 = tok0 + warp * 32;
  if (t0 >= tok1) return;
  constexpr int STRIDE = kAttnWarps * 32;
  constexpr int PF_AHEAD = 2;
  for (int p = 1; p <= PF_AHEAD; ++p) prefetch(t0 + p * STRIDE);
  for (; t0 < tok1; t0 += STRIDE) {
    const int tn = t0 + STRIDE;
    prefetch(t0 + (PF_AHEAD + 1) * STRIDE);
    kphase(ka, t0);
    if (tn < tok1) load_k(ka, tn);
    vphase(va);
    if (tn < tok1) load_v(va, tn);
  }
}

// Nearest of the 256 fp16 pairs book[e] (e at byte offset e * stride) to p = (p0, p1),
// found by a team of TS consecutive lanes (lane `split` of the team scans entries
// split, split + TS, ...): fp32 screen keeping the best and second-best distance, then
// float64 rescoring of the entries inside the fp32 error band — the reference quantize's
// float64 argmin with the lowest index on ties (V/codec.py:239-253), the arithmetic of
// qkv_rope_append_cq_kernel (csrc/decode.cu). Returns the code on every lane of the team.
template <int TS>
__device__ __forceinline__ int cq_nearest_team(const uint8_t* book, int stride, float p0, float p1, int split) {
  const float m0 = -2.f * p0, m1 = -2.f * p1;
  float d1 = FLT_MAX, d2 = FLT_MAX, cmax2 = 0.f;
  int e1 = 0x7fffffff;
#pragma unroll 4
  for (int e = split; e < 256; e += TS) {
    const uint32_t w = *reinterpret_cast<const uint32_t*>(book + e * stride);
    const float c0 = __half2float(__ushort_as_half((unsigned short)(w & 0xffff)));
    const float c1 = __half2float(__ushort_as_half((unsigned short)(w >> 16)));
    const float cn = c0 * c0 + c1 * c1;
    cmax2 = fmaxf(cmax2, cn);
    const float d = fmaf(m0, c0, fmaf(m1, c1, cn));
    // branch-free best / second best (equal distances keep the earlier, lower index)
    d2 = fminf(d2, fmaxf(d, d1));
    e1 = d < d1 ? e : e1;
    d1 = fminf(d1, d);
  }
#pragma unroll
  for (int o = 1; o < TS; o <<= 1) {
    const float od1 = __shfl_xor_sync(0xffffffffu, d1, o), od2 = __shfl_xor_sync(0xffffffffu, d2, o);
    const int oe1 = __shfl_xor_sync(0xffffffffu, e1, o);
    cmax2 = fmaxf(cmax2, __shfl_xor_sync(0xffffffffu, cmax2, o));
    d2 = fminf(fmaxf(d1, od1), fminf(d2, od2));
    if (od1 < d1 || (od1 == d1 && oe1 < e1)) {
      d1 = od1;
      e1 = oe1;
    }
  }
  const float tol = 2e-5f * (cmax2 + p0 * p0 + p1 * p1) + 1e-30f;
  const bool need64 = d2 - d1 <= tol;  // uniform over a team, not over the warp:
  if (!__any_sync(0xffffffffu, need64)) return e1;  // every lane takes the shuffles below
  const double r0 = p0, r1 = p1;
  const double pn = __dadd_rn(__dmul_rn(r0, r0), __dmul_rn(r1, r1));
  double best = DBL_MAX;
  int be = 0x7fffffff;
  for (int e = split; e < 256; e += TS) {
    const uint32_t w = *reinterpret_cast<const uint32_t*>(book + e * stride);
    const float c0 = __half2float(__ushort_as_half((unsigned short)(w & 0xffff)));
    const float c1 = __half2float(__ushort_as_half((unsigned short)(w >> 16)));
    if (need64 && fmaf(m0, c0, fmaf(m1, c1, c0 * c0 + c1 * c1)) <= d1 + tol) {
      const double a0 = c0, a1 = c1;
      const double dot = __dadd_rn(__dmul_rn(r0, a0), __dmul_rn(r1, a1));
      const double cnd = __dadd_rn(__dmul_rn(a0, a0), __dmul_rn(a1, a1));
      const double d = __dadd_rn(__dadd_rn(__dmul_rn(dot, -2.0), cnd), pn);
      if (d < best) {  // entries ascend within a lane: the first minimum is the lowest index
        best = d;
        be = e;
      }
    }
  }
#pragma unroll
  for (int o = 1; o < TS; o <<= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int oe = __shfl_xor_sync(0xffffffffu, be, o);
    if (ob < best || (ob == best && oe < be)) {
      best = ob;
      be = oe;
    }
  }
  return need64 ? be : e1;
}

template <int V, int GPL, bool APPEND = false>
__global__ void __launch_bounds__(kAttnThreads, 1) attn_cq_kernel(AttnArgs a) {
  using SM = AttnSmem<V, GPL>;
  constexpr int G = SM::G, C = SM::C, EPB = SM::EPB;

  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t dyn_base = smem_u32(smem);
  const uint32_t lut_off = ((dyn_base + 0xffffu) & ~0xffffu) - dyn_base;  // first 64 KB-aligned region
  const uint32_t scratch_off = lut_off >= SM::scratch_bytes ? 0u : lut_off + 2 * (uint32_t)SM::region;
  uint8_t* vbook_s = smem + lut_off + SM::region;
  float* lut_s = reinterpret_cast<float*>(smem + lut_off);
  float* scratch = reinterpret_cast<float*>(smem + scratch_off);
  const uint32_t pbuf = smem_u32(smem + scratch_off + SM::pbuf_off) + (uint32_t)(threadIdx.x >> 5) * 64;
  // mbarrier for the bulk-copied books (8-byte aligned slot at the end of the scratch)
  const uint32_t book_bar = smem_u32(smem + ((scratch_off + SM::scratch_bytes - 8) & ~7u));
  const bool bulk_books = (V == 2) && a.kbt != nullptr && a.vbt != nullptr;
  uint32_t book_phase = 0;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (bulk_books && threadIdx.x == 0) {
    mbar_init(book_bar, 1);
    mbar_fence_init();
  }
  pdl_launch_dependents();
  attn_trace(a, 0);
  if (threadIdx.x < 2) {
    // L2 prefetch of the first unit's K / V codes while the preceding kernel drains (the
    // work split depends on the device length, read speculatively: a stale value only
    // misdirects a hint)
    const int Ts = a.len_ptr ? max(1, min(*(volatile const int*)a.len_ptr, a.T_cap)) : a.T;
    const int NTs = (Ts + kAttnChunk - 1) / kAttnChunk, Us = a.H * a.B * NTs;
    const int GEs = min((int)gridDim.x, Us);
    if ((int)blockIdx.x < GEs) {
      const int u = (int)((int64_t)blockIdx.x * Us / GEs);
      const int hh = u / (a.B * NTs), bb = (u / NTs) % a.B, tc = u % NTs;
      const int64_t off = ((int64_t)(bb * a.H + hh) * a.T_cap + (int64_t)tc * kAttnChunk) * G;
      const uint32_t bytes = (uint32_t)min(kAttnChunk, Ts - tc * kAttnChunk) * G;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"((threadIdx.x ? a.vc : a.kc) + off),
                   "r"((bytes + 15) & ~15u) : "memory");
    }
  }
  pdl_wait();  // q, the fresh KV codes and the length come from the preceding kernels
  attn_trace(a, 1);
  const uint32_t lut_base = smem_u32(lut_s);
  const uint32_t vbook_base = smem_u32(vbook_s);
  constexpr bool aligned = true;  // by construction: single-prmt addressing
  // valid length: the host's, or read on the device (a graph-replayed decode step)
  const int T = a.len_ptr ? max(1, min(__ldg(a.len_ptr), a.T_cap)) : a.T;
  const int NT = (T + kAttnChunk - 1) / kAttnChunk;
  const int BNT = a.B * NT;
  const int U = a.H * BNT;
  // The grid is sized from the capacity; a shorter device length leaves fewer units
  // than CTAs. Only the first GE = min(grid, U) CTAs take part, so every
  // participating CTA owns at least one unit and publishes the partial a finisher
  // counts on (an empty range would never publish: the finisher would spin forever).
  const int GE = min((int)gridDim.x, U);
  if ((int)blockIdx.x >= GE) return;
  const int u0 = (int)((int64_t)blockIdx.x * U / GE);
  const int u1 = (int)((int64_t)(blockIdx.x + 1) * U / GE);

  int cur_h = -1;
  bool books_inflight = false;
  auto issue_books = [&](int hh, bool with_v) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    const uint32_t bytes = 256u * G * EPB;
    mbar_arrive_expect_tx(book_bar, with_v ? 2 * bytes : bytes);
    tma_load_1d(smem_u32(lut_s), a.kbt + (int64_t)hh * 256 * G * V, bytes, book_bar);
    if (with_v) tma_load_1d(smem_u32(vbook_s), a.vbt + (int64_t)hh * 256 * G * V, bytes, book_bar);
  };
  AttnPhase ph;
  for (int u = u0; u < u1;) {
    ph.mark(a, -1);
    const int h = u / BNT;
    const int b = (u / NT) % a.B;
    const int tc0 = u % NT;
    const int span_end = min(u1, (u / NT + 1) * NT);
    const int tc1 = tc0 + (span_end - u);
    const int bh = b * a.H + h;
    const int tok0 = tc0 * kAttnChunk;
    const int tok1 = min(tc1 * kAttnChunk, T);

    // ---- span prologue. The query and K-book reads for the LUT are issued before
    // waiting for the previous span to release shared memory.
    constexpr int EPL = 16 / EPB;  // entries per 16-byte read
    constexpr int VITEMS = G * (256 / EPL);
    constexpr int VPER = (VITEMS + kAttnThreads - 1) / kAttnThreads;
    constexpr int KSTEP = kAttnThreads / G;
    constexpr int KPER = (256 / EPL + KSTEP - 1) / KSTEP;
    const bool switch_h = (h != cur_h);
    const int g = tid % G;  // constant per thread since kAttnThreads % G == 0
    float qv[V];
    if (APPEND) {
      // fused front end: q roped here (fp16-rounded like the separate rope kernel)
      const __half* qr = a.qkv + (int64_t)b * 3 * a.H * C + (int64_t)h * C;
#pragma unroll
      for (int j = 0; j < V; ++j)
        qv[j] = __half2float(__float2half_rn(rope_channel_attn(qr, g * V + j, C, a.log2_theta, T - 1))) * a.scale_log2;
    } else {
#pragma unroll
      for (int j = 0; j < V; ++j) qv[j] = load_as_f32(a.q, a.q_dtype, (int64_t)bh * C + g * V + j) * a.scale_log2;
    }
    const int pos = T - 1;  // the new token of a fused decode step
    const bool append_here = APPEND && tok0 <= pos && pos < tok1;
    if (bulk_books) {
      // ---- books by bulk copy: the head's K book lands in the LUT region and its V
      // book in the V-book region, both already [e][g]; the LUT is then computed in
      // place (an fp16 pair and its fp32 logit term occupy the same 4 bytes). After
      // the first span the copies were issued at the end of the previous span.
      if (!books_inflight) {
        __syncthreads();  // previous span finished with books / LUT / scratch
        if (tid == 0) issue_books(h, switch_h);
      }
      cur_h = h;
      mbar_wait(book_bar, book_phase);
      book_phase ^= 1;
      if constexpr (APPEND && V == 2 && GPL == 2 && kAttnThreads == 512) if (append_here) {
        // the new K row (roped) and V row of (b, h): nearest centroids against the books in
        // shared memory ([e][g] fp16 pairs), teams of 4 lanes per group, K on threads
        // 0..255 and V on 256..511; codes written into the caches (KV_IL, token pos)
        const bool is_k = tid < 256;
        const int gg = (tid & 255) >> 2, split = tid & 3;
        const __half* row = a.qkv + (int64_t)b * 3 * a.H * C + (int64_t)((is_k ? a.H : 2 * a.H) + h) * C;
        float p[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int c = gg * 2 + j;
          p[j] = is_k ? __half2float(__float2half_rn(rope_channel_attn(row, c, C, a.log2_theta, pos)))
                      : __half2float(row[c]);
        }
        const uint8_t* bk = is_k ? reinterpret_cast<const uint8_t*>(lut_s) : vbook_s;
        const int code = cq_nearest_team<4>(bk + gg * 4, G * 4, p[0], p[1], split);
        if (split == 0) (is_k ? a.kc_w : a.vc_w)[(int64_t)bh * a.T_cap * G + kvil_offset(pos, gg, G)] = (uint8_t)code;
        __syncthreads();  // the codes are in global memory before any warp loads that batch
      }
      uint32_t* lw = reinterpret_cast<uint32_t*>(lut_s);
      for (int idx = tid; idx < 256 * G; idx += kAttnThreads) {  // idx % G == g for every idx of a thread
        const uint32_t w = lw[idx];
        const float k0 = __half2float(__ushort_as_half((unsigned short)(w & 0xffff)));
        const float k1 = __half2float(__ushort_as_half((unsigned short)(w >> 16)));
        lut_s[idx] = fmaf(qv[1], k1, qv[0] * k0);
      }
      __syncthreads();
    } else {
    const __half* kbk = a.kb + (int64_t)(h * G + g) * 256 * V;
    uint4 wk[KPER];
#pragma unroll
    for (int k = 0; k < KPER; ++k) {
      const int ec = tid / G + k * KSTEP;
      if (ec < 256 / EPL) wk[k] = __ldg(reinterpret_cast<const uint4*>(kbk + ec * EPL * V));
    }
    __syncthreads();  // previous span finished with books / LUT / scratch
    if (switch_h) {
      uint4 wv[VPER];
#pragma unroll
      for (int k = 0; k < VPER; ++k) {
        const int item = tid + k * kAttnThreads;
        if (item < VITEMS) {
          const int gg = item % G, ec = item / G;
          wv[k] = __ldg(reinterpret_cast<const uint4*>(a.vb + ((int64_t)(h * G + gg) * 256 + ec * EPL) * V));
        }
      }
      // ---- Switch/Load: the V codebooks of head h, transposed to [e][g]
#pragma unroll
      for (int k = 0; k < VPER; ++k) {
        const int item = tid + k * kAttnThreads;
        if (item < VITEMS) {
          const int gg = item % G, ec = item / G;
          const uint32_t* wp = &wv[k].x;
#pragma unroll
          for (int i = 0; i < EPL; ++i) {
            uint8_t* d = vbook_s + ((size_t)(ec * EPL + i) * G + gg) * EPB;
            if constexpr (V == 2) *reinterpret_cast<uint32_t*>(d) = wp[i];
            else *reinterpret_cast<uint2*>(d) = make_uint2(wp[2 * i], wp[2 * i + 1]);
          }
        }
      }
      cur_h = h;
    }
    // ---- LUT for (b, h): LUT[e][g] = scale_log2 * <q_g, Kbook_g[e]>; lanes own
    // groups so the stores are bank-conflict free.
#pragma unroll
    for (int k = 0; k < KPER; ++k) {
      const int ec = tid / G + k * KSTEP;
      if (ec < 256 / EPL) {
        const __half* ent = reinterpret_cast<const __half*>(&wk[k]);
#pragma unroll
        for (int i = 0; i < EPL; ++i) {
          float s = 0.f;
#pragma unroll
          for (int j = 0; j < V; ++j) s = fmaf(qv[j], __half2float(ent[i * V + j]), s);
          lut_s[(ec * EPL + i) * G + g] = s;
        }
      }
    }
    __syncthreads();
    }
    ph.mark(a, 0);
    float m_w = -INFINITY, l_lane = 0.f;
    constexpr int GPH = G / kKvLanes;
    float acc[GPH][V];  // lane (h, ll): groups ll + kKvLanes (j ^ h), j < GPH
#pragma unroll
    for (int j = 0; j < GPH; ++j)
#pragma unroll
      for (int i = 0; i < V; ++i) acc[j][i] = 0.f;
    uint4 ka[2 * GPL], va[2 * GPL];
    const int fresh_t0 = append_here ? (pos & ~31) : -1;  // the batch holding the appended token
    if (tok0 + warp * 32 < tok1) attn_load_batch<V, GPL>(a, bh, tok0 + warp * 32, ka, va, APPEND && tok0 + warp * 32 == fresh_t0);
    if (aligned)
      attn_stream_span<V, GPL, true, APPEND>(a, T, bh, tok0, tok1, lut_base, vbook_base, m_w, l_lane, acc, ka, va,
                                              fresh_t0, pbuf);
    else
      attn_stream_span<V, GPL, false, APPEND>(a, T, bh, tok0, tok1, lut_base, vbook_base, m_w, l_lane, acc, ka, va,
                                               fresh_t0, pbuf);

    ph.mark(a, 1);
    // ---- merge the warps of this span
    float l_w = l_lane;
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) l_w += __shfl_xor_sync(0xffffffffu, l_w, off);
    float* my = scratch + warp * (C + 2);
    if (lane == 0) {
      my[0] = m_w;
      my[1] = l_w;
    }
    // the lane sets hold the same groups for different tokens: a butterfly over the
    // sets (set h's slot j is group ll + kKvLanes (j ^ h)) leaves set 0 with the sums
#pragma unroll
    for (int o = kKvLanes; o < 32; o <<= 1) {
      float nx[GPH][V];
#pragma unroll
      for (int j = 0; j < GPH; ++j)
#pragma unroll
        for (int i = 0; i < V; ++i) nx[j][i] = acc[j][i] + __shfl_xor_sync(0xffffffffu, acc[j ^ (o / kKvLanes)][i], o);
#pragma unroll
      for (int j = 0; j < GPH; ++j)
#pragma unroll
        for (int i = 0; i < V; ++i) acc[j][i] = nx[j][i];
    }
    if (lane < kKvLanes)
#pragma unroll
      for (int j = 0; j < GPH; ++j)
#pragma unroll
        for (int i = 0; i < V; ++i) my[2 + (lane + kKvLanes * j) * V + i] = acc[j][i];
    __syncthreads();
    // every warp is done with the LUT and the V book: fetch the next span's books now,
    // so the copy overlaps this span's merge
    books_inflight = bulk_books && span_end < u1;
    if (books_inflight && tid == 0) issue_books(span_end / BNT, span_end / BNT != h);
    const bool whole = (tc0 == 0 && tc1 == NT);
    // A (b, h) split across CTAs is finished by the CTA holding its chunk 0 (for that
    // CTA it is the last span of its range); the later parts are the first spans of
    // the following CTAs, which publish {m, l, acc} as tagged 64-bit words in their
    // own slot — no fence, no counter, no extra launch (the GEMV's scheme).
    const bool finisher = (tc0 == 0 && !whole);
    unsigned long long* slots = a.slots;
    float M = -INFINITY, val = 0.f;
    if (tid <= C) {
#pragma unroll
      for (int w = 0; w < kAttnWarps; ++w) M = fmaxf(M, scratch[w * (C + 2)]);
      for (int w = 0; w < kAttnWarps; ++w) {
        const float mw = scratch[w * (C + 2)];
        const float sc = (mw == -INFINITY) ? 0.f : fast_exp2(mw - M);
        val += sc * (tid < C ? scratch[w * (C + 2) + 2 + tid] : scratch[w * (C + 2) + 1]);
      }
      if (whole || finisher) {
        scratch[kAttnWarps * (C + 2) + tid] = val;
      } else {
        unsigned long long* my_slot = slots + (int64_t)blockIdx.x * (C + 2);
        if (tid < C) {
          st_relaxed_u64(my_slot + 2 + tid, tag_partial(val));
        } else {
          st_relaxed_u64(my_slot, tag_partial(M));
          st_relaxed_u64(my_slot + 1, tag_partial(val));
        }
      }
    }
    __syncthreads();
    if (whole) {
      if (tid < C) {
        const float L = scratch[kAttnWarps * (C + 2) + C];
        store_from_f32(a.out, a.out_dtype, (int64_t)bh * C + tid, scratch[kAttnWarps * (C + 2) + tid] / L);
      }
    } else if (finisher) {
      // the CTAs after this one whose ranges start inside (b, h)
      const int bh_end = u - tc0 + NT;  // first unit past this (b, h)
      int k_end = blockIdx.x + 1;
      while (k_end < GE && (int)((int64_t)k_end * U / GE) < bh_end) ++k_end;
      const int n_later = k_end - blockIdx.x - 1;
      if (tid < C) {
        float Mr = M, L = scratch[kAttnWarps * (C + 2) + C], A = scratch[kAttnWarps * (C + 2) + tid];
        constexpr int PF = 4;  // slots in flight
        for (int j0 = 0; j0 < n_later; j0 += PF) {
          unsigned long long wm[PF], wl[PF], wa[PF];
#pragma unroll
          for (int j = 0; j < PF; ++j) {
            const unsigned long long* sp = slots + (int64_t)(blockIdx.x + 1 + j0 + j) * (C + 2);
            wm[j] = wl[j] = wa[j] = 1ull << 32;
            if (j0 + j < n_later) {
              wm[j] = ld_relaxed_u64(sp);
              wl[j] = ld_relaxed_u64(sp + 1);
              wa[j] = ld_relaxed_u64(sp + 2 + tid);
            }
          }
          for (;;) {  // re-poll every pending word per round (one L2 round trip per round)
            bool pending = false;
#pragma unroll
            for (int j = 0; j < PF; ++j) pending |= ((wm[j] >> 32) == 0) | ((wl[j] >> 32) == 0) | ((wa[j] >> 32) == 0);
            if (!pending) break;
#pragma unroll
            for (int j = 0; j < PF; ++j) {
              const unsigned long long* sp = slots + (int64_t)(blockIdx.x + 1 + j0 + j) * (C + 2);
              if ((wm[j] >> 32) == 0) wm[j] = ld_relaxed_u64(sp);
              if ((wl[j] >> 32) == 0) wl[j] = ld_relaxed_u64(sp + 1);
              if ((wa[j] >> 32) == 0) wa[j] = ld_relaxed_u64(sp + 2 + tid);
            }
          }
#pragma unroll
          for (int j = 0; j < PF; ++j) {
            if (j0 + j < n_later) {
              unsigned long long* sp = slots + (int64_t)(blockIdx.x + 1 + j0 + j) * (C + 2);
              const float mj = __uint_as_float((uint32_t)wm[j]);
              const float Mn = fmaxf(Mr, mj);
              const float s0 = fast_exp2(Mr - Mn);
              const float s1 = (mj == -INFINITY) ? 0.f : fast_exp2(mj - Mn);
              L = L * s0 + __uint_as_float((uint32_t)wl[j]) * s1;
              A = A * s0 + __uint_as_float((uint32_t)wa[j]) * s1;
              Mr = Mn;
              st_relaxed_u64(sp + 2 + tid, 0ull);  // slots reset for the next launch
            }
          }
        }
        store_from_f32(a.out, a.out_dtype, (int64_t)bh * C + tid, A / L);
      }
      __syncthreads();  // every thread has read m and l
      for (int j = tid; j < n_later; j += kAttnThreads) {
        unsigned long long* sp = slots + (int64_t)(blockIdx.x + 1 + j) * (C + 2);
        st_relaxed_u64(sp, 0ull);
        st_relaxed_u64(sp + 1, 0ull);
      }
    }
    ph.mark(a, 2);
    u = span_end;
  }
  attn_trace(a, 5);
  ph.flush(a);
}

// ---------------------------------------------------------------------------
// generic path: dense fp32 K/V in the workspace

__global__ void __launch_bounds__(256) attn_dense_kernel(const float* __restrict__ k, const float* __restrict__ v,
                                                         const void* __restrict__ q, int q_dtype, int T, int T_cap,
                                                         int C,
                                                         float* __restrict__ logits, void* __restrict__ out,
                                                         int out_dtype) {
  const int bh = blockIdx.x;
  const float* kb = k + (int64_t)bh * T_cap * C;
  const float* vb = v + (int64_t)bh * T_cap * C;
  float* lg = logits + (int64_t)bh * T_cap;
  __shared__ float red[256];
  const float inv = 1.0f / sqrtf((float)C);
  float mx = -INFINITY;
  for (int t = threadIdx.x; t < T; t += blockDim.x) {
    float s = 0.f;
    for (int c = 0; c < C; ++c) s = fmaf(load_as_f32(q, q_dtype, (int64_t)bh * C + c), kb[(int64_t)t * C + c], s);
    s *= inv;
    lg[t] = s;
    mx = fmaxf(mx, s);
  }
  red[threadIdx.x] = mx;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] = fmaxf(red[threadIdx.x], red[threadIdx.x + o]);
    __syncthreads();
  }
  mx = red[0];
  __syncthreads();
  float sum = 0.f;
  for (int t = threadIdx.x; t < T; t += blockDim.x) {
    const float p = expf(lg[t] - mx);
    lg[t] = p;
    sum += p;
  }
  red[threadIdx.x] = sum;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  sum = red[0];
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    float acc = 0.f;
    for (int t = 0; t < T; ++t) acc = fmaf(lg[t], vb[(int64_t)t * C + c], acc);
    store_from_f32(out, out_dtype, (int64_t)bh * C + c, acc / sum);
  }
}

// ---------------------------------------------------------------------------
// dispatch

// the per-tensor half of the fast-path test (K and V are checked separately)
static bool attn_fast_tensor_ok(const Geom& g, const VqbTensor* t) {
  if (t->layout != VQB_LAYOUT_KV_IL || t->codebook_dtype != VQB_F16) return false;
  if (g.sharing != VQB_SHARE_CHANNEL_GROUP || g.group_width != g.v || g.R != 1 || g.bits != 8) return false;
  if (!(g.v == 2 || g.v == 4) || !(g.gpr == 32 || g.gpr == 64)) return false;
  if (g.v * g.gpr > 128) return false;  // C <= 128: books fit the 64 KB regions
  return g.ndim == 4 && g.dims[2] % 32 == 0;
}

static bool attn_fast_ok(const Geom& gk, const Geom& gv, const VqbTensor* k, const VqbTensor* v, int T,
                         const VqbLaunch* L) {
  if (L && (L->flags & VQB_FLAG_FORCE_GENERIC)) return false;
  if (!attn_fast_tensor_ok(gk, k) || !attn_fast_tensor_ok(gv, v)) return false;
  if (gk.v != gv.v || T % 32 != 0) return false;
  return kAttnSlotOffset + (int64_t)sm_count() * (gk.cols + 2) * 8 <= VQB_WS_COUNTER_BYTES;
}

static int64_t a256(int64_t x) { return (x + 255) & ~int64_t(255); }

static int64_t attn_generic_ws(const Geom& g, int64_t BH) {
  const int64_t T = g.dims[2], C = g.cols;
  return VQB_WS_COUNTER_BYTES + a256(2 * BH * T * C * 4) + BH * T * 4;
}

// Path-aware: the fast kernel needs only the self-resetting counter/slot head; the
// generic path dense fp32 K + V + logits. Sized from K (V is expected in the same
// format; a mismatching V that forces the generic path fails with ECAPACITY).
int64_t attn_ws_bytes(const VqbTensor* k, int64_t BH, const VqbLaunch* L) {
  Geom g;
  int s = make_geom(k, &g);
  if (s) return s;
  const bool fast = !(L && (L->flags & VQB_FLAG_FORCE_GENERIC)) && attn_fast_tensor_ok(g, k) &&
                    kAttnSlotOffset + (int64_t)sm_count() * (g.cols + 2) * 8 <= VQB_WS_COUNTER_BYTES;
  return fast ? (int64_t)VQB_WS_COUNTER_BYTES : attn_generic_ws(g, BH);
}

template <int V, int GPL>
static int launch_attn_t(AttnArgs& a, cudaStream_t st, int grid_limit, int flags) {
  auto kern = a.qkv ? attn_cq_kernel<V, GPL, true> : attn_cq_kernel<V, GPL, false>;
  constexpr size_t smem = AttnSmem<V, GPL>::total;
  static bool configured[2][64] = {};  // per kernel (plain / fused append) and device
  int dev = 0;
  cudaGetDevice(&dev);
  const int which = a.qkv ? 1 : 0;
  if (!configured[which][dev & 63]) {
    VQB_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured[which][dev & 63] = true;
  }
  const int U = a.B * a.H * (a.len_ptr ? a.NT_cap : a.NT);  // a device length is bounded by the capacity
  int grid = balanced_grid(U, sm_count());
  if (grid_limit > 0) grid = std::min(grid, grid_limit);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kAttnThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  cfg.attrs = attr;
  cfg.numAttrs = persistent_attrs(attr, flags);
  VQB_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, a));
  set_kernel(a.qkv ? "attn_cq_append" : "attn_cq");
  set_launch(grid, kAttnThreads, 256, 0);
  return VQB_OK;
}

int attn_dispatch(const VqbTensor* k, const VqbTensor* v, const void* q, int q_dtype, int B, int H, int T, int C,
                  const int* d_len, void* out, int out_dtype, const VqbLaunch* L, void* ws, size_t ws_bytes,
                  cudaStream_t st, bool* used_fast, const __half* qkv = nullptr, float log2_theta = 0.f) {
  Geom gk, gv;
  int s = make_geom(k, &gk);
  if (s) return s;
  s = make_geom(v, &gv);
  if (s) return s;
  // T is the number of valid tokens: a prefix of the cache's capacity dims[2]
  if (gk.ndim != 4 || gv.ndim != 4 || gk.dims[0] != B || gk.dims[1] != H || T < 1 || gk.dims[2] < T ||
      gk.dims[3] != C)
    return set_error(VQB_ESHAPE, "quantized KV shape does not match op axes (%d, %d, %d, %d)", B, H, T, C);
  const int T_cap = (int)gk.dims[2];
  for (int i = 0; i < 4; ++i)
    if (gv.dims[i] != gk.dims[i]) return set_error(VQB_ESHAPE, "K and V shapes differ");
  if (q_dtype < VQB_F32 || q_dtype > VQB_BF16 || out_dtype < VQB_F32 || out_dtype > VQB_BF16)
    return set_error(VQB_ECONFIG, "unknown query/output dtype");
  const int64_t BH = (int64_t)B * H;
  const bool fast = attn_fast_ok(gk, gv, k, v, T_cap, L);
  const int64_t need = fast ? (int64_t)VQB_WS_COUNTER_BYTES : attn_generic_ws(gk, BH);
  if ((int64_t)ws_bytes < need || !ws)
    return set_error(VQB_ECAPACITY, "attention workspace too small: %zu < %lld", ws_bytes, (long long)need);
  if (used_fast) *used_fast = fast;
  if (!fast && d_len)
    return set_error(VQB_ECONFIG, "a device-resident KV length needs the fast attention configuration");
  if (qkv && (!fast || !d_len || !k->d_codebooks_t || !v->d_codebooks_t || gk.v != 2 || gk.gpr != 64 ||
              k->layout != VQB_LAYOUT_KV_IL || v->layout != VQB_LAYOUT_KV_IL || k->codebook_dtype != VQB_F16))
    return set_error(VQB_ECONFIG, "the fused rope + KV append attention needs the CQ-4 fast configuration (v = 2, "
                                  "C = 128, KV_IL caches with per-head books) and a device length");
  if (fast) {
    AttnArgs a;
    a.kc = reinterpret_cast<const uint8_t*>(k->d_codes);
    a.vc = reinterpret_cast<const uint8_t*>(v->d_codes);
    a.kb = reinterpret_cast<const __half*>(k->d_codebooks);
    a.vb = reinterpret_cast<const __half*>(v->d_codebooks);
    a.kbt = reinterpret_cast<const __half*>(k->d_codebooks_t);
    a.vbt = reinterpret_cast<const __half*>(v->d_codebooks_t);
    a.q = q;
    a.q_dtype = q_dtype;
    a.out = out;
    a.out_dtype = out_dtype;
    a.slots = reinterpret_cast<unsigned long long*>(reinterpret_cast<uint8_t*>(ws) + kAttnSlotOffset);
    a.B = B;
    a.H = H;
    a.T = T;
    a.NT = (int)ceil_div(T, kAttnChunk);
    a.T_cap = T_cap;
    a.NT_cap = (int)ceil_div(T_cap, kAttnChunk);
    a.len_ptr = d_len;
    a.trace = (L && (L->flags & 32)) ? reinterpret_cast<unsigned long long*>(reinterpret_cast<uint8_t*>(ws) + 8192)
                                     : nullptr;
    a.scale_log2 = 1.4426950408889634f / sqrtf((float)C);
    a.qkv = qkv;
    a.log2_theta = log2_theta;
    a.kc_w = const_cast<uint8_t*>(reinterpret_cast<const uint8_t*>(k->d_codes));
    a.vc_w = const_cast<uint8_t*>(reinterpret_cast<const uint8_t*>(v->d_codes));
    int gl = L ? L->grid_limit : 0;
    // the planner's split of T (VqbLaunch split over T): each (b, h) span is shared
    // by ~split_factor CTAs of the persistent schedule
    if (L && L->split_axis == 'T' && L->split_factor > 0) {
      const int cap = std::max(1, B * H * L->split_factor);
      gl = gl > 0 ? std::min(gl, cap) : cap;
    }
    const int gpl = (int)(gk.gpr / 32);
    if (gk.v == 2 && gpl == 2) return launch_attn_t<2, 2>(a, st, gl, L ? L->flags : 0);
    if (gk.v == 2 && gpl == 1) return launch_attn_t<2, 1>(a, st, gl, L ? L->flags : 0);
    if (gk.v == 4 && gpl == 1) return launch_attn_t<4, 1>(a, st, gl, L ? L->flags : 0);
    return set_error(VQB_ECONFIG, "no fast attention instance for this configuration");
  }
  float* kd = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ws) + VQB_WS_COUNTER_BYTES);
  float* vd = kd + BH * T_cap * C;
  float* lg =
      reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ws) + VQB_WS_COUNTER_BYTES + a256(2 * BH * T_cap * C * 4));
  s = launch_dequant(gk, k, kd, VQB_F32, st);
  if (s) return s;
  s = launch_dequant(gv, v, vd, VQB_F32, st);
  if (s) return s;
  attn_dense_kernel<<<(unsigned)BH, 256, 0, st>>>(kd, vd, q, q_dtype, T, T_cap, C, lg, out, out_dtype);
  VQB_LAUNCH_CHECK("attn_dense_kernel");
  set_kernel("attn_generic");
  return VQB_OK;
}

int attn_usage(VqbUsage* u) {
  cudaFuncAttributes at;
  auto k = attn_cq_kernel<2, 2>;
  VQB_CUDA_CHECK(cudaFuncGetAttributes(&at, k));
  constexpr size_t smem = AttnSmem<2, 2>::total;
  VQB_CUDA_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  u->shared_bytes = (int)(at.sharedSizeBytes + smem);
  u->regs_per_thread = at.numRegs;
  u->threads_per_block = kAttnThreads;
  int occ = 0;
  VQB_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, kAttnThreads, smem));
  u->max_blocks_per_sm = occ;
  return VQB_OK;
}

}  // namespace vqb

extern "C" int vqb_attn_decode(const VqbTensor* k, const VqbTensor* v, const void* d_q, int32_t q_dtype, int32_t B,
                               int32_t H, int32_t T, int32_t C, void* d_out, int32_t out_dtype,
                               const VqbLaunch* launch, void* d_ws, size_t ws_bytes, void* stream) {
  return vqb::attn_dispatch(k, v, d_q, q_dtype, B, H, T, C, nullptr, d_out, out_dtype, launch, d_ws, ws_bytes,
                            reinterpret_cast<cudaStream_t>(stream), nullptr);
}

extern "C" int vqb_attn_decode_len(const VqbTensor* k, const VqbTensor* v, const void* d_q, int32_t q_dtype,
                                   int32_t B, int32_t H, int32_t T, int32_t C, const int32_t* d_len, void* d_out,
                                   int32_t out_dtype, const VqbLaunch* launch, void* d_ws, size_t ws_bytes,
                                   void* stream) {
  return vqb::attn_dispatch(k, v, d_q, q_dtype, B, H, T, C, d_len, d_out, out_dtype, launch, d_ws, ws_bytes,
                            reinterpret_cast<cudaStream_t>(stream), nullptr);
}

extern "C" int vqb_attn_decode_append(const VqbTensor* k_cache, const VqbTensor* v_cache, const void* d_qkv, int32_t B,
                                      int32_t H, int32_t C, const int32_t* d_len, float theta, void* d_out,
                                      int32_t out_dtype, const VqbLaunch* launch, void* d_ws, size_t ws_bytes,
                                      void* stream) {
  if (!d_qkv || !d_len || theta <= 0.f) return vqb::set_error(VQB_ECONFIG, "fused append attention needs qkv, d_len and theta");
  const int T = k_cache ? (int)k_cache->dims[2] : 1;
  return vqb::attn_dispatch(k_cache, v_cache, nullptr, VQB_F16, B, H, T, C, d_len, d_out, out_dtype, launch, d_ws,
                            ws_bytes, reinterpret_cast<cudaStream_t>(stream), nullptr,
                            reinterpret_cast<const __half*>(d_qkv), log2f(theta));
}
