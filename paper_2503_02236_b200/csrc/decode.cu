// decode.cu — the kernels around the fused VQ ops in a Llama decode step (C5):
// RMSNorm with a fused residual add, RoPE on the fresh q/k, online CQ
// quantization of the new K/V rows into the KV cache, SiLU-gated FFN glue and the
// device-resident position counter that lets a whole step replay as a CUDA graph.
//
// Online KV quantization is the reference's `quantize` (pkg/src/vqforge/codec.py:
// 367-389) — nearest centroid per sub-vector and level, residual carried to the next
// level — with `_nearest`'s float64 distance |c|^2 - 2 p.c (+|p|^2) and its
// lowest-index tie rule (codec.py:239-253), evaluated on the GPU (the paper's KV
// online quantization).
#include <cfloat>
#include <type_traits>

#include "common.cuh"

namespace vqb {

// Set (bit 0) when a KV append finds its write position outside [0, capacity):
// the write is skipped instead of landing in the next head's token rows; the host
// reads and clears it with vqb_take_device_error.
__device__ unsigned int g_append_oob = 0;

__device__ __forceinline__ bool append_pos_ok(int pos, int64_t cap) {
  if (pos >= 0 && pos < cap) return true;
  atomicOr(&g_append_oob, 1u);
  return false;
}


// ---------------------------------------------------------------------------
// RMSNorm (Llama): h = x + residual (residual updated in place), out = w * norm(h);
// statistics in fp32 like the HF reference implementation.

template <int THREADS>
__global__ void __launch_bounds__(THREADS) rmsnorm_kernel(const __half* __restrict__ x, __half* __restrict__ res,
                                                          const __half* __restrict__ w, __half* __restrict__ out,
                                                          int dim, float eps) {
  pdl_launch_dependents();
  // the weight does not depend on the previous kernel: fetch it before waiting
  constexpr int PER = 8;  // halves per 16-byte vector
  const int nvec = dim / PER;
  uint4 wv[4], hv[4];
  int nv = 0;
  for (int i = threadIdx.x; i < nvec && nv < 4; i += THREADS, ++nv) wv[nv] = __ldg(reinterpret_cast<const uint4*>(w) + i);
  pdl_wait();
  const int row = blockIdx.x;
  const __half* xr = x ? x + (int64_t)row * dim : nullptr;
  __half* rr = res + (int64_t)row * dim;
  __half* orow = out + (int64_t)row * dim;
  __shared__ float red[THREADS / 32];
  float ss = 0.f;
  nv = 0;
  for (int i = threadIdx.x; i < nvec && nv < 4; i += THREADS, ++nv) {
    uint4 h = reinterpret_cast<const uint4*>(rr)[i];
    if (xr) {
      // the residual stream is fp16: round the sum like the fp16 reference add
      const uint4 a = reinterpret_cast<const uint4*>(xr)[i];
      __half2* hp = reinterpret_cast<__half2*>(&h);
      const __half2* ap = reinterpret_cast<const __half2*>(&a);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = __half22float2(hp[j]), g = __half22float2(ap[j]);
        hp[j] = __floats2half2_rn(f.x + g.x, f.y + g.y);
      }
      reinterpret_cast<uint4*>(rr)[i] = h;
    }
    hv[nv] = h;
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
    if (threadIdx.x == 0) red[0] = t;
  }
  __syncthreads();
  const float inv = rsqrtf(red[0] / (float)dim + eps);
  nv = 0;
  for (int i = threadIdx.x; i < nvec && nv < 4; i += THREADS, ++nv) {
    const __half2* hp = reinterpret_cast<const __half2*>(&hv[nv]);
    const __half2* wp = reinterpret_cast<const __half2*>(&wv[nv]);
    uint4 o;
    __half2* op = reinterpret_cast<__half2*>(&o);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 f = __half22float2(hp[j]), ww = __half22float2(wp[j]);
      // HF: weight * (h * inv).to(fp16)
      const float2 hf = __half22float2(__floats2half2_rn(f.x * inv, f.y * inv));
      op[j] = __floats2half2_rn(ww.x * hf.x, ww.y * hf.y);
    }
    reinterpret_cast<uint4*>(orow)[i] = o;
  }
}

// ---------------------------------------------------------------------------
// RoPE (rotate-half convention) on the q and k thirds of the fused qkv projection
// output (B, 3*H*C): q is written roped into a contiguous (B, H, C) buffer for the
// attention kernel, k is roped in place for the KV quantizer. pos = *d_len - 1.

__global__ void __launch_bounds__(128) qkv_rope_kernel(__half* __restrict__ qkv, __half* __restrict__ q_out, int H,
                                                       int C, const int* __restrict__ d_len, float log2_theta) {
  pdl_launch_dependents();
  pdl_wait();
  const int b = blockIdx.y, hh = blockIdx.x;  // hh in [0, 2H): q heads then k heads
  const int half = C / 2;
  const int pos = __ldg(d_len) - 1;
  __half* src = qkv + (int64_t)b * 3 * H * C + (int64_t)hh * C;
  for (int i = threadIdx.x; i < half; i += blockDim.x) {
    // inv_freq = theta^(-2i/C), angle in fp32 like the HF rotary embedding
    const float inv_freq = exp2f(-log2_theta * (2.0f * i) / (float)C);
    const float ang = (float)pos * inv_freq;
    float sn, cs;
    sincosf(ang, &sn, &cs);
    const float x0 = __half2float(src[i]), x1 = __half2float(src[i + half]);
    const __half y0 = __float2half_rn(x0 * cs - x1 * sn);
    const __half y1 = __float2half_rn(x1 * cs + x0 * sn);
    if (hh < H) {
      __half* dst = q_out + ((int64_t)b * H + hh) * C;
      dst[i] = y0;
      dst[i + half] = y1;
    } else {
      src[i] = y0;
      src[i + half] = y1;
    }
  }
}

// ---------------------------------------------------------------------------
// SiLU-gated FFN glue: out[r, i] = silu(gate[r, i]) * up[r, i] with the fused
// gate_up output laid out [gate (F) | up (F)] per row.

__global__ void __launch_bounds__(256) silu_mul_kernel(const __half* __restrict__ gu, __half* __restrict__ out,
                                                       int rows, int F) {
  pdl_launch_dependents();
  pdl_wait();
  const int64_t n = (int64_t)rows * F;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / F, c = i - r * F;
    const float g = __half2float(gu[r * 2 * F + c]);
    const float u = __half2float(gu[r * 2 * F + F + c]);
    // HF: act(gate) in fp16, then * up in fp16
    const __half s = __float2half_rn(g / (1.0f + __expf(-g)));
    out[i] = __float2half_rn(__half2float(s) * u);
  }
}

__global__ void add_len_kernel(int* d_len, int delta) {
  pdl_launch_dependents();
  pdl_wait();
  *d_len += delta;
}

// ---------------------------------------------------------------------------
// Nearest-centroid quantization of KV rows into a (B, H, T_cap, C) code stream.
// One warp per sub-vector: lane l scores entries l, l+32, ...; float64 distances,
// argmin with the lowest index on ties (codec.py:239-253); R levels quantize the
// running residual (codec.py:376-381).

// One sub-vector s of a KV tensor: R levels of nearest centroid on the running
// residual res[0..v) (float64), code written into the tensor's stream. Warp-wide.
template <int V>
__device__ __forceinline__ void quantize_subvector(const Geom& g, void* __restrict__ codes,
                                                   const __half* __restrict__ books, double* res, int64_t s,
                                                   int lane) {
  const int region = region_of(g, s);
  for (int r = 0; r < g.R; ++r) {
    const __half* book = books + (int64_t)(r * g.n_regions + region) * g.K * V;
    // d = (-2 * p.c + |c|^2) + |p|^2 in the reference's float64 operation order,
    // no FMA contraction (codec.py:241-251)
    double pn = 0.0;
#pragma unroll
    for (int j = 0; j < V; ++j) pn = __dadd_rn(pn, __dmul_rn(res[j], res[j]));
    double best = DBL_MAX;
    int best_e = 0x7fffffff;
    auto consider = [&](int e, const float* c) {
      double dot = 0.0, cn = 0.0;
#pragma unroll
      for (int j = 0; j < V; ++j) {
        const double cj = (double)c[j];
        dot = __dadd_rn(dot, __dmul_rn(res[j], cj));
        cn = __dadd_rn(cn, __dmul_rn(cj, cj));
      }
      const double d = __dadd_rn(__dadd_rn(__dmul_rn(dot, -2.0), cn), pn);
      if (d < best) {
        best = d;
        best_e = e;
      }
    };
    if (V == 2 && g.K == 256 && r == 0) {
      // the CQ case: all eight of this lane's entries are loaded up front (one L2 round
      // trip), screened with fp32 distances, and only the entries within the fp32
      // error band of the minimum are rescored in float64 — the float64 argmin is
      // always among them (|d32 - d64| <= err and tol >= 2 err), so the code is the
      // reference's, at a fraction of the float64 work
      uint32_t w[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) w[k] = __ldg(reinterpret_cast<const uint32_t*>(book) + lane + 32 * k);
      const float r0 = (float)res[0], r1 = (float)res[1];  // fp16 rows: exact in fp32
      float d32[8], dmin = FLT_MAX, scale = 0.f;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float c0 = __half2float(__ushort_as_half((unsigned short)(w[k] & 0xffff)));
        const float c1 = __half2float(__ushort_as_half((unsigned short)(w[k] >> 16)));
        const float dot = r0 * c0 + r1 * c1, cn = c0 * c0 + c1 * c1;
        d32[k] = cn - 2.f * dot;
        dmin = fminf(dmin, d32[k]);
        scale = fmaxf(scale, cn + 2.f * fabsf(dot));
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        dmin = fminf(dmin, __shfl_xor_sync(0xffffffffu, dmin, o));
        scale = fmaxf(scale, __shfl_xor_sync(0xffffffffu, scale, o));
      }
      const float tol = 1e-5f * (scale + 1e-30f);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (d32[k] <= dmin + tol) {
          const float c[2] = {__half2float(__ushort_as_half((unsigned short)(w[k] & 0xffff))),
                              __half2float(__ushort_as_half((unsigned short)(w[k] >> 16)))};
          consider(lane + 32 * k, c);
        }
      }
    } else {
      for (int e = lane; e < g.K; e += 32) {
        float c[V];
#pragma unroll
        for (int j = 0; j < V; ++j) c[j] = __half2float(book[(int64_t)e * V + j]);
        consider(e, c);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oe = __shfl_xor_sync(0xffffffffu, best_e, o);
      if (ob < best || (ob == best && oe < best_e)) {
        best = ob;
        best_e = oe;
      }
    }
    if (lane == 0) {
      const int64_t off = (g.layout == VQB_LAYOUT_PLAIN) ? (int64_t)r * g.S + s : il_offset(g, r, s);
      if (g.code_bytes == 1) reinterpret_cast<uint8_t*>(codes)[off] = (uint8_t)best_e;
      else reinterpret_cast<uint16_t*>(codes)[off] = (uint16_t)best_e;
    }
#pragma unroll
    for (int j = 0; j < V; ++j) res[j] -= (double)__half2float(book[(int64_t)best_e * V + j]);
  }
}

// runtime vector size -> compile-time register arrays
template <typename F>
__device__ __forceinline__ void with_v(int v, F&& f) {
  switch (v) {
    case 2: f(std::integral_constant<int, 2>{}); break;
    case 4: f(std::integral_constant<int, 4>{}); break;
    case 8: f(std::integral_constant<int, 8>{}); break;
    default: f(std::integral_constant<int, 16>{}); break;
  }
}

template <typename XT>
__global__ void __launch_bounds__(256) cq_quantize_kernel(Geom g, void* __restrict__ codes,
                                                          const __half* __restrict__ books, const XT* __restrict__ x,
                                                          int64_t xs_b, int64_t xs_h, int64_t xs_t, int n_tok,
                                                          int tok0, const int* __restrict__ d_len) {
  pdl_launch_dependents();
  pdl_wait();
  const int warps = blockDim.x / 32;
  const int64_t sv = (int64_t)blockIdx.x * warps + (threadIdx.x >> 5);  // sub-vector of the new rows
  const int lane = threadIdx.x & 31;
  const int B = (int)g.dims[0], H = (int)g.dims[1];
  const int G = (int)g.gpr, V = g.v;
  const int64_t total = (int64_t)B * H * n_tok * G;
  if (sv >= total) return;
  const int gi = (int)(sv % G);
  int64_t rest = sv / G;
  const int t = (int)(rest % n_tok);
  rest /= n_tok;
  const int h = (int)(rest % H);
  const int b = (int)(rest / H);
  const int p0 = d_len ? __ldg(d_len) - n_tok : tok0;  // decode: the rows end at the current length
  const int tok = p0 + t;
  if (!append_pos_ok(tok, g.d_T)) return;
  const XT* xp = x + b * xs_b + h * xs_h + t * xs_t + gi * V;
  // sub-vector index in the reference's row-major order over (B, H, T_cap, C)
  const int64_t row = ((int64_t)b * H + h) * g.d_T + tok;
  with_v(V, [&](auto vc) {
    constexpr int VV = decltype(vc)::value;
    double res[VV];
#pragma unroll
    for (int j = 0; j < VV; ++j) res[j] = (double)to_f32<XT>(xp[j]);
    quantize_subvector<VV>(g, codes, books, res, row * G + gi, lane);
  });
}

// Fused decode-step front end, one warp per work item (so the float64 nearest-
// centroid searches of every K and V sub-vector run in parallel): per (batch row,
// head), G warps rope + quantize k sub-vectors, G warps quantize v sub-vectors and
// one warp ropes q into the contiguous buffer the attention reads. One launch
// instead of three (rope, quantize K, quantize V); codes land at d_len[0]-1.
__device__ __forceinline__ float rope_channel(const __half* x, int c, int C, float log2_theta, int pos) {
  const int half = C / 2;
  const int i = c < half ? c : c - half;
  const float inv_freq = exp2f(-log2_theta * (2.0f * i) / (float)C);
  float sn, cs;
  sincosf((float)pos * inv_freq, &sn, &cs);
  const float x0 = __half2float(x[i]), x1 = __half2float(x[i + half]);
  return c < half ? x0 * cs - x1 * sn : x1 * cs + x0 * sn;
}

__global__ void __launch_bounds__(256) qkv_rope_append_kernel(const __half* __restrict__ qkv, __half* __restrict__ q_out,
                                                              Geom gk, void* __restrict__ kcodes,
                                                              const __half* __restrict__ kbooks, Geom gv,
                                                              void* __restrict__ vcodes,
                                                              const __half* __restrict__ vbooks, int B, int H, int C,
                                                              const int* __restrict__ d_len, float log2_theta) {
  pdl_launch_dependents();
  pdl_wait();
  const int G = C / gk.v;
  const int per_head = 2 * G + 1;
  const int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (w >= (int64_t)B * H * per_head) return;
  const int lane = threadIdx.x & 31;
  const int role = (int)(w % per_head);
  const int h = (int)((w / per_head) % H), b = (int)(w / per_head / H);
  const int pos = __ldg(d_len) - 1;
  const __half* row = qkv + (int64_t)b * 3 * H * C;
  if (role == 2 * G) {  // q: rope into the contiguous (B, H, C) buffer
    const __half* q = row + (int64_t)h * C;
    __half* dst = q_out + ((int64_t)b * H + h) * C;
    for (int c = lane; c < C; c += 32) dst[c] = __float2half_rn(rope_channel(q, c, C, log2_theta, pos));
    return;
  }
  const bool is_k = role < G;
  const Geom& g = is_k ? gk : gv;
  const int gi = is_k ? role : role - G;
  if (!append_pos_ok(pos, g.d_T)) return;
  const int64_t s = (((int64_t)b * H + h) * g.d_T + pos) * G + gi;
  with_v(g.v, [&](auto vc) {
    constexpr int VV = decltype(vc)::value;
    double res[VV];
    if (is_k) {
      // the roped k is an fp16 tensor in the reference step: round before quantizing
      const __half* k = row + (int64_t)(H + h) * C;
#pragma unroll
      for (int j = 0; j < VV; ++j)
        res[j] = (double)__half2float(__float2half_rn(rope_channel(k, gi * VV + j, C, log2_theta, pos)));
    } else {
      const __half* v = row + (int64_t)(2 * H + h) * C;
#pragma unroll
      for (int j = 0; j < VV; ++j) res[j] = (double)__half2float(v[gi * VV + j]);
    }
    quantize_subvector<VV>(g, is_k ? kcodes : vcodes, is_k ? kbooks : vbooks, res, s, lane);
  });
}

// CQ fast path of the front end (v = 2, 256 entries, one level on both caches): one
// warp per (head, channel group, K|V) stages that group's 256 entries in shared memory
// ({c0, c1, |c|^2} per entry) and quantizes every batch row of the step; q is roped by
// one warp per (batch row, head). The warp's lanes are (row, split) pairs: S = 32 / B'
// lanes share a row (B' = batch rounded up to a power of two, at most 32) and each
// scans every S-th entry, so a batch of 16 scans 128 entries per lane instead of the
// whole warp reducing over each row in turn. Distances are screened in fp32 (best and
// second best per lane, merged over the row's lanes); only rows whose best two lie
// within the fp32 error band rescore their candidates in float64 (the reference's
// float64 argmin, lowest index on ties, is always among them).
// Nearest-centroid codes of NR rows per lane (rows b0 + rl + r * rows) against one
// group's book bk[e] = {c0, c1, |c|^2, 0}: fp32 screen keeping the best (lowest index
// among equals) and second-best distance, S lanes per row merged, float64 rescoring of
// near ties in the reference's operation order (V/codec.py:239-253).
template <int NR>
__device__ __forceinline__ void append_rows(const __half* __restrict__ qkv, int H, int C, bool is_k, int h, int gi,
                                            const float (&cs)[2], const float (&sn)[2], const float4* bk,
                                            float cmax2, int B, int rows, int S, int split, int rl, int n_e,
                                            uint8_t* codes, int64_t bstride) {
  for (int b0 = 0; b0 < B; b0 += rows * NR) {
    float p0[NR], p1[NR], m0[NR], m1[NR], d1[NR], d2[NR];
    int e1[NR];
    bool valid[NR];
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const int b = b0 + rl + r * rows;
      valid[r] = b < B;
      p0[r] = p1[r] = 0.f;
      if (valid[r]) {
        const __half* row = qkv + (int64_t)b * 3 * H * C + (int64_t)((is_k ? H : 2 * H) + h) * C;
        float pj[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int c = gi * 2 + j;
          if (is_k) {
            const int half = C / 2, i = c < half ? c : c - half;
            const float x0 = __half2float(row[i]), x1 = __half2float(row[i + half]);
            // the roped k is an fp16 tensor in the reference step
            pj[j] = __half2float(__float2half_rn(c < half ? x0 * cs[j] - x1 * sn[j] : x1 * cs[j] + x0 * sn[j]));
          } else {
            pj[j] = __half2float(row[c]);
          }
        }
        p0[r] = pj[0];
        p1[r] = pj[1];
      }
      m0[r] = -2.f * p0[r];
      m1[r] = -2.f * p1[r];
      d1[r] = d2[r] = FLT_MAX;
      e1[r] = 0x7fffffff;
    }
#pragma unroll 8
    for (int i = 0; i < n_e; ++i) {
      const int e = i * S + split;
      const float4 c = bk[e];
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        const float d = fmaf(m0[r], c.x, fmaf(m1[r], c.y, c.z));
        // branch-free best / second best (equal distances keep the earlier, lower index)
        d2[r] = fminf(d2[r], fmaxf(d, d1[r]));
        e1[r] = d < d1[r] ? e : e1[r];
        d1[r] = fminf(d1[r], d);
      }
    }
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      for (int o = 1; o < S; o <<= 1) {  // merge the row's lanes
        const float od1 = __shfl_xor_sync(0xffffffffu, d1[r], o), od2 = __shfl_xor_sync(0xffffffffu, d2[r], o);
        const int oe1 = __shfl_xor_sync(0xffffffffu, e1[r], o);
        d2[r] = fminf(fmaxf(d1[r], od1), fminf(d2[r], od2));
        if (od1 < d1[r] || (od1 == d1[r] && oe1 < e1[r])) {
          d1[r] = od1;
          e1[r] = oe1;
        }
      }
      // screen tolerance: a bound on the fp32 rounding of |c|^2 - 2 p.c relative to the
      // float64 distance (2 sqrt(|p|^2 |c|^2) <= |p|^2 + |c|^2 keeps it sqrt-free)
      const float tol = 2e-5f * (cmax2 + p0[r] * p0[r] + p1[r] * p1[r]) + 1e-30f;
      const bool need64 = valid[r] && (d2[r] - d1[r] <= tol);
      int code = e1[r];
      if (__any_sync(0xffffffffu, need64)) {
        // several candidates: float64 distances in the reference's operation order
        double best = DBL_MAX;
        int be = 0x7fffffff;
        if (need64) {
          const double r0 = p0[r], r1 = p1[r];
          const double pn = __dadd_rn(__dmul_rn(r0, r0), __dmul_rn(r1, r1));
          for (int i = 0; i < n_e; ++i) {
            const int e = i * S + split;
            const float4 c = bk[e];
            if (fmaf(m0[r], c.x, fmaf(m1[r], c.y, c.z)) <= d1[r] + tol) {
              const double a0 = c.x, a1 = c.y;
              const double dot = __dadd_rn(__dmul_rn(r0, a0), __dmul_rn(r1, a1));
              const double cn = __dadd_rn(__dmul_rn(a0, a0), __dmul_rn(a1, a1));
              const double d = __dadd_rn(__dadd_rn(__dmul_rn(dot, -2.0), cn), pn);
              if (d < best) {  // entries ascend: the first minimum is the lowest index
                best = d;
                be = e;
              }
            }
          }
        }
        for (int o = 1; o < S; o <<= 1) {
          const double ob = __shfl_xor_sync(0xffffffffu, best, o);
          const int oe = __shfl_xor_sync(0xffffffffu, be, o);
          if (ob < best || (ob == best && oe < be)) {
            best = ob;
            be = oe;
          }
        }
        if (need64) code = be;
      }
      if (valid[r] && split == 0) codes[(int64_t)(b0 + rl + r * rows) * bstride] = (uint8_t)code;
    }
  }
}

__global__ void __launch_bounds__(256) qkv_rope_append_cq_kernel(const __half* __restrict__ qkv,
                                                               __half* __restrict__ q_out, Geom gk,
                                                               void* __restrict__ kcodes,
                                                               const __half* __restrict__ kbooks, Geom gv,
                                                               void* __restrict__ vcodes,
                                                               const __half* __restrict__ vbooks, int B, int H,
                                                               int C, const int* __restrict__ d_len,
                                                               float log2_theta) {
  __shared__ float4 books_s[8][256];  // per warp: {c0, c1, |c|^2, 0}
  pdl_launch_dependents();
  pdl_wait();
  const int G = C / 2;
  const int wl = threadIdx.x >> 5;
  const int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + wl;
  const int lane = threadIdx.x & 31;
  const int pos = __ldg(d_len) - 1;
  const int n_book_warps = 2 * H * G;
  if (w >= n_book_warps) {  // q rope
    const int64_t qi = w - n_book_warps;
    if (qi >= (int64_t)B * H) return;
    const int h = (int)(qi % H), b = (int)(qi / H);
    const __half* q = qkv + (int64_t)b * 3 * H * C + (int64_t)h * C;
    __half* dst = q_out + ((int64_t)b * H + h) * C;
    for (int c = lane; c < C; c += 32) dst[c] = __float2half_rn(rope_channel(q, c, C, log2_theta, pos));
    return;
  }
  const bool is_k = w < H * G;
  const int hg = (int)(is_k ? w : w - H * G);
  const int h = hg / G, gi = hg % G;
  const Geom& g = is_k ? gk : gv;
  if (!append_pos_ok(pos, g.d_T)) return;
  const __half* book = (is_k ? kbooks : vbooks) + (int64_t)(h * G + gi) * 256 * 2;  // region = h*G + gi
  float4* bk = books_s[wl];
  float cmax2 = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t wv = __ldg(reinterpret_cast<const uint32_t*>(book) + lane + 32 * k);
    const float c0 = __half2float(__ushort_as_half((unsigned short)(wv & 0xffff)));
    const float c1 = __half2float(__ushort_as_half((unsigned short)(wv >> 16)));
    const float cn = c0 * c0 + c1 * c1;
    bk[lane + 32 * k] = make_float4(c0, c1, cn, 0.f);
    cmax2 = fmaxf(cmax2, cn);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cmax2 = fmaxf(cmax2, __shfl_xor_sync(0xffffffffu, cmax2, o));
  __syncwarp();
  // rope factors of this group's two channels (k only): position-dependent, row-independent
  float cs[2] = {1.f, 1.f}, sn[2] = {0.f, 0.f};
  if (is_k) {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int c = gi * 2 + j, i = c < C / 2 ? c : c - C / 2;
      sincosf((float)pos * exp2f(-log2_theta * (2.0f * i) / (float)C), &sn[j], &cs[j]);
    }
  }
  // the code's address is linear in the batch row in both layouts (PLAIN and KV_IL
  // differ only inside a (b, h) block): one 64-bit index computation per warp
  const int64_t s00 = ((int64_t)h * g.d_T + pos) * G + gi;
  const int64_t off0 = (g.layout == VQB_LAYOUT_PLAIN) ? s00 : il_offset(g, 0, s00);
  const int64_t bstride = (int64_t)H * g.d_T * G;
  int rows = 1;  // B' = rows per pass (power of two <= 32)
  while (rows < B && rows < 32) rows <<= 1;
  const int S = 32 / rows;  // lanes per row
  const int split = lane & (S - 1), rl = lane / S;
  const int n_e = 256 / S;
  uint8_t* codes = reinterpret_cast<uint8_t*>(is_k ? kcodes : vcodes) + off0;
  if (B > 32)  // two rows per lane: one broadcast read of each entry serves both
    append_rows<2>(qkv, H, C, is_k, h, gi, cs, sn, bk, cmax2, B, rows, S, split, rl, n_e, codes, bstride);
  else
    append_rows<1>(qkv, H, C, is_k, h, gi, cs, sn, bk, cmax2, B, rows, S, split, rl, n_e, codes, bstride);
}

// ---- token sampling (the decode loop's last step) ----
// Gumbel-max: argmax_i (logit_i / T + g_i), g_i = -log(-log(u_i)), is an exact draw
// from softmax(logit / T); u_i comes from a counter-based hash of (seed, step, row, i),
// so a graph-replayed step draws fresh noise from the device length. top_k keeps the
// logits >= the k-th largest (ties kept, the usual top-k warper's rule), found by a
// 4-pass radix select over order-preserving 32-bit keys. T == 0 is greedy argmax.
// Ties in the score resolve to the lowest index (torch.argmax's rule).
__device__ __forceinline__ uint32_t order_key(float f) {
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__device__ __forceinline__ float sample_uniform(uint64_t seed, uint32_t step, uint32_t row, uint32_t i) {
  uint64_t z = (seed ^ ((((uint64_t)step << 32) | row) * 0x9E3779B97F4A7C15ull)) + (uint64_t)(i + 1) * 0xBF58476D1CE4E5B9ull;
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return ((float)(uint32_t)(z >> 41) + 0.5f) * 1.1920928955078125e-7f;  // (k + 0.5) / 2^23: exact, in (0, 1)
}

constexpr int kSampleUnroll = 8;  // logits loaded per thread before they are used

template <int THREADS>
__global__ void __launch_bounds__(THREADS) sample_kernel(const void* __restrict__ logits, int dtype, int V,
                                                         float inv_temp, int top_k, float top_p, uint64_t seed,
                                                         const int* __restrict__ d_step, int64_t* __restrict__ out) {
  __shared__ unsigned long long hist[256];
  __shared__ unsigned long long sel[2];  // digit, remaining weight
  __shared__ float best_s[THREADS / 32];
  __shared__ int best_i[THREADS / 32];
  __shared__ float red_f[THREADS / 32];
  __shared__ unsigned long long red_u[THREADS / 32];
  pdl_launch_dependents();
  pdl_wait();
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const float* lf = reinterpret_cast<const float*>(logits) + (int64_t)b * V;
  const __half* lh = reinterpret_cast<const __half*>(logits) + (int64_t)b * V;
  auto load = [&](int i) { return dtype == VQB_F32 ? __ldg(lf + i) : __half2float(lh[i]); };
  const bool greedy = !(inv_temp > 0.f);
  // Radix select over order-preserving keys: the largest key t with weight(keys >= t,
  // keys >= floor) >= target, weight(x) = 1 (top-k) or the fixed-point probability.
  auto select = [&](unsigned long long target, uint32_t floor, auto weight) -> uint32_t {
    uint32_t prefix = 0, mask = 0;
    if (tid == 0) sel[1] = target;
    for (int shift = 24; shift >= 0; shift -= 8) {
      for (int i = tid; i < 256; i += THREADS) hist[i] = 0ull;
      __syncthreads();
      for (int i0 = tid; i0 < V; i0 += THREADS * kSampleUnroll) {
        float xs[kSampleUnroll];  // independent loads first: one latency per kSampleUnroll elements
#pragma unroll
        for (int u = 0; u < kSampleUnroll; ++u) xs[u] = i0 + u * THREADS < V ? load(i0 + u * THREADS) : 0.f;
#pragma unroll
        for (int u = 0; u < kSampleUnroll; ++u) {
          const uint32_t k = order_key(xs[u]);
          if (i0 + u * THREADS < V && k >= floor && (k & mask) == prefix)
            atomicAdd(&hist[(k >> shift) & 255], weight(xs[u]));
        }
      }
      __syncthreads();
      if (warp == 0) {  // the digit holding the target: scan bins from the top
        unsigned long long c[8], tot = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          c[j] = hist[255 - (lane * 8 + j)];
          tot += c[j];
        }
        unsigned long long incl = tot;  // inclusive prefix over lanes (lane 0 = the highest bins)
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned long long t = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += t;
        }
        const unsigned long long rem = sel[1];
        unsigned long long run = incl - tot;
        if (run < rem && incl >= rem) {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            if (run + c[j] >= rem) {
              sel[0] = (unsigned long long)(255 - (lane * 8 + j));
              sel[1] = rem - run;
              break;
            }
            run += c[j];
          }
        }
      }
      __syncthreads();
      prefix |= (uint32_t)sel[0] << shift;
      mask |= 255u << shift;
      __syncthreads();
    }
    return prefix;
  };
  uint32_t thr = 0;  // keep keys >= thr
  if (!greedy && top_k > 0 && top_k < V) thr = select((unsigned long long)top_k, 0u, [](float) { return 1ull; });
  if (!greedy && top_p < 1.f) {
    // nucleus over the (top-k) kept logits: weights exp((x - max) / T) in 2^32 fixed point
    float mx = -INFINITY;
    for (int i = tid; i < V; i += THREADS) {
      const float x = load(i);
      if (order_key(x) >= thr) mx = fmaxf(mx, x);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) red_f[warp] = mx;
    __syncthreads();
    mx = red_f[0];
    for (int w = 1; w < THREADS / 32; ++w) mx = fmaxf(mx, red_f[w]);
    const float sc = inv_temp * 1.4426950408889634f;
    auto weight = [&](float x) {
      return (unsigned long long)(exp2f((x - mx) * sc) * 4294967296.0f);
    };
    unsigned long long tw = 0;
    for (int i = tid; i < V; i += THREADS) {
      const float x = load(i);
      if (order_key(x) >= thr) tw += weight(x);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tw += __shfl_xor_sync(0xffffffffu, tw, o);
    if (lane == 0) red_u[warp] = tw;
    __syncthreads();
    tw = 0;
    for (int w = 0; w < THREADS / 32; ++w) tw += red_u[w];
    __syncthreads();
    unsigned long long target = (unsigned long long)ceil((double)top_p * (double)tw);
    if (target < 1) target = 1;
    thr = max(thr, select(target, thr, weight));
  }
  const uint32_t step = d_step ? (uint32_t)__ldg(d_step) : 0u;
  float bs = -INFINITY;
  int bi = 0x7fffffff;
  for (int i0 = tid; i0 < V; i0 += THREADS * kSampleUnroll) {
    float xs[kSampleUnroll];
#pragma unroll
    for (int u = 0; u < kSampleUnroll; ++u) xs[u] = i0 + u * THREADS < V ? load(i0 + u * THREADS) : 0.f;
#pragma unroll
    for (int u = 0; u < kSampleUnroll; ++u) {
      const int i = i0 + u * THREADS;
      const float x = xs[u];
      if (i >= V || order_key(x) < thr) continue;
      const float s = greedy ? x : fmaf(x, inv_temp, -__logf(-__logf(sample_uniform(seed, step, (uint32_t)b, (uint32_t)i))));
      if (s > bs || bi == 0x7fffffff) {  // ascending i per thread: strict > keeps the lowest index
        bs = s;
        bi = i;
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float os = __shfl_xor_sync(0xffffffffu, bs, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (os > bs || (os == bs && oi < bi)) {
      bs = os;
      bi = oi;
    }
  }
  if (lane == 0) {
    best_s[warp] = bs;
    best_i[warp] = bi;
  }
  __syncthreads();
  if (warp == 0) {
    bs = lane < THREADS / 32 ? best_s[lane] : -INFINITY;
    bi = lane < THREADS / 32 ? best_i[lane] : 0x7fffffff;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float os = __shfl_xor_sync(0xffffffffu, bs, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (os > bs || (os == bs && oi < bi)) {
        bs = os;
        bi = oi;
      }
    }
    if (lane == 0) out[b] = bi;
  }
}

}  // namespace vqb

using namespace vqb;

extern "C" int vqb_rmsnorm(const void* d_x, void* d_residual, const void* d_weight, void* d_out, int32_t rows,
                           int32_t dim, float eps, void* stream) {
  if (rows < 1 || dim < 8 || (dim % 8) || dim > 8 * 4 * 512)
    return set_error(VQB_ESHAPE, "rmsnorm needs rows >= 1 and dim a multiple of 8 up to 16384");
  VQB_CUDA_CHECK(launch_pdl(rmsnorm_kernel<512>, dim3(rows), dim3(512), 0, reinterpret_cast<cudaStream_t>(stream),
                            reinterpret_cast<const __half*>(d_x), reinterpret_cast<__half*>(d_residual),
                            reinterpret_cast<const __half*>(d_weight), reinterpret_cast<__half*>(d_out), dim, eps));
  VQB_LAUNCH_CHECK("rmsnorm_kernel");
  set_kernel("rmsnorm");
  return VQB_OK;
}

extern "C" int vqb_qkv_rope(void* d_qkv, void* d_q_out, int32_t B, int32_t H, int32_t C, const int32_t* d_len,
                            float theta, void* stream) {
  if (B < 1 || H < 1 || C < 2 || (C & 1) || !d_len) return set_error(VQB_ESHAPE, "bad rope arguments");
  VQB_CUDA_CHECK(launch_pdl(qkv_rope_kernel, dim3(2 * H, B), dim3(128), 0, reinterpret_cast<cudaStream_t>(stream),
                            reinterpret_cast<__half*>(d_qkv), reinterpret_cast<__half*>(d_q_out), H, C, d_len,
                            log2f(theta)));
  VQB_LAUNCH_CHECK("qkv_rope_kernel");
  set_kernel("qkv_rope");
  return VQB_OK;
}

extern "C" int vqb_qkv_rope_append(const void* d_qkv, void* d_q_out, const VqbTensor* k_cache,
                                   const VqbTensor* v_cache, int32_t B, int32_t H, int32_t C, const int32_t* d_len,
                                   float theta, void* stream) {
  Geom gk, gv;
  int s = make_geom(k_cache, &gk);
  if (s) return s;
  s = make_geom(v_cache, &gv);
  if (s) return s;
  if (!d_len || C < 2 || (C & 1)) return set_error(VQB_ESHAPE, "bad rope/append arguments");
  for (const Geom* g : {&gk, &gv}) {
    if (g->ndim != 4 || g->dims[0] != B || g->dims[1] != H || g->cols != C)
      return set_error(VQB_ESHAPE, "KV cache shape does not match (B, H, *, C) = (%d, %d, *, %d)", B, H, C);
    if (g->v > 16 || (g->layout != VQB_LAYOUT_KV_IL && g->layout != VQB_LAYOUT_PLAIN))
      return set_error(VQB_ECONFIG, "KV append writes the KV_IL or PLAIN layout");
  }
  if (gk.v != gv.v) return set_error(VQB_ECONFIG, "K and V caches need one vector size");
  if (k_cache->codebook_dtype != VQB_F16 || v_cache->codebook_dtype != VQB_F16)
    return set_error(VQB_ECONFIG, "KV append needs fp16 codebooks");
  const bool cq = gk.v == 2 && gk.K == 256 && gk.R == 1 && gv.K == 256 && gv.R == 1 && gk.code_bytes == 1 &&
                  gk.sharing == VQB_SHARE_CHANNEL_GROUP && gv.sharing == VQB_SHARE_CHANNEL_GROUP &&
                  gk.group_width == 2 && gv.group_width == 2;
  if (cq) {
    const int64_t warps = (int64_t)2 * H * (C / 2) + (int64_t)B * H;
    VQB_CUDA_CHECK(launch_pdl(qkv_rope_append_cq_kernel, dim3((unsigned)((warps + 7) / 8)), dim3(256), 0,
                              reinterpret_cast<cudaStream_t>(stream), reinterpret_cast<const __half*>(d_qkv),
                              reinterpret_cast<__half*>(d_q_out), gk, const_cast<void*>(k_cache->d_codes),
                              reinterpret_cast<const __half*>(k_cache->d_codebooks), gv,
                              const_cast<void*>(v_cache->d_codes),
                              reinterpret_cast<const __half*>(v_cache->d_codebooks), B, H, C, d_len, log2f(theta)));
    set_kernel("qkv_rope_append");
    return VQB_OK;
  }
  const int64_t warps = (int64_t)B * H * (2 * (C / gk.v) + 1);
  VQB_CUDA_CHECK(launch_pdl(qkv_rope_append_kernel, dim3((unsigned)((warps + 7) / 8)), dim3(256), 0,
                            reinterpret_cast<cudaStream_t>(stream),
                            reinterpret_cast<const __half*>(d_qkv), reinterpret_cast<__half*>(d_q_out), gk,
                            const_cast<void*>(k_cache->d_codes),
                            reinterpret_cast<const __half*>(k_cache->d_codebooks), gv,
                            const_cast<void*>(v_cache->d_codes),
                            reinterpret_cast<const __half*>(v_cache->d_codebooks), B, H, C, d_len, log2f(theta)));
  set_kernel("qkv_rope_append");
  return VQB_OK;
}

extern "C" int vqb_silu_mul(const void* d_gate_up, void* d_out, int32_t rows, int32_t ffn, void* stream) {
  if (rows < 1 || ffn < 1) return set_error(VQB_ESHAPE, "bad silu_mul arguments");
  const int64_t n = (int64_t)rows * ffn;
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, (int64_t)sm_count() * 8);
  VQB_CUDA_CHECK(launch_pdl(silu_mul_kernel, dim3(blocks), dim3(256), 0, reinterpret_cast<cudaStream_t>(stream),
                            reinterpret_cast<const __half*>(d_gate_up), reinterpret_cast<__half*>(d_out), rows, ffn));
  VQB_LAUNCH_CHECK("silu_mul_kernel");
  set_kernel("silu_mul");
  return VQB_OK;
}

extern "C" int vqb_take_device_error(int32_t* out) {
  unsigned int v = 0, zero = 0;
  VQB_CUDA_CHECK(cudaMemcpyFromSymbol(&v, vqb::g_append_oob, sizeof(v)));
  VQB_CUDA_CHECK(cudaMemcpyToSymbol(vqb::g_append_oob, &zero, sizeof(zero)));
  if (out) *out = (int32_t)v;
  return VQB_OK;
}

extern "C" int vqb_sample(const void* d_logits, int32_t logits_dtype, int32_t B, int32_t vocab, float temperature,
                          int32_t top_k, float top_p, uint64_t seed, const int32_t* d_step, int64_t* d_tokens,
                          void* stream) {
  if (B < 1 || vocab < 1) return set_error(VQB_ESHAPE, "sample needs B >= 1 and vocab >= 1");
  if (logits_dtype != VQB_F16 && logits_dtype != VQB_F32) return set_error(VQB_ECONFIG, "sample reads fp16 or fp32 logits");
  if (!(temperature >= 0.f) || top_k < 0 || !(top_p > 0.f && top_p <= 1.f))
    return set_error(VQB_ECONFIG, "sample needs temperature >= 0, top_k >= 0 and 0 < top_p <= 1");
  const float inv_temp = temperature > 0.f ? 1.0f / temperature : 0.f;
  VQB_CUDA_CHECK(launch_pdl(sample_kernel<1024>, dim3(B), dim3(1024), 0, reinterpret_cast<cudaStream_t>(stream),
                            d_logits, (int)logits_dtype, (int)vocab, inv_temp, (int)top_k, top_p, seed, d_step,
                            d_tokens));
  VQB_LAUNCH_CHECK("sample_kernel");
  set_kernel("sample");
  return VQB_OK;
}

extern "C" int vqb_add_len(int32_t* d_len, int32_t delta, void* stream) {
  VQB_CUDA_CHECK(launch_pdl(add_len_kernel, dim3(1), dim3(1), 0, reinterpret_cast<cudaStream_t>(stream), d_len, delta));
  VQB_LAUNCH_CHECK("add_len_kernel");
  return VQB_OK;
}

extern "C" int vqb_cq_quantize(const VqbTensor* t, const void* d_x, int32_t x_dtype, int64_t xs_b, int64_t xs_h,
                               int64_t xs_t, int32_t n_tok, int32_t tok0, const int32_t* d_len, void* stream) {
  Geom g;
  int s = make_geom(t, &g);
  if (s) return s;
  if (g.ndim != 4) return set_error(VQB_ESHAPE, "KV quantization needs a (B, H, T, C) tensor");
  if (t->codebook_dtype != VQB_F16) return set_error(VQB_ECONFIG, "KV quantization needs fp16 codebooks");
  if (g.layout != VQB_LAYOUT_KV_IL && g.layout != VQB_LAYOUT_PLAIN)
    return set_error(VQB_ECONFIG, "KV quantization writes the KV_IL or PLAIN layout");
  if (g.v > 16 || n_tok < 1) return set_error(VQB_ESHAPE, "bad quantization extent");
  if (!d_len && (tok0 < 0 || tok0 + n_tok > g.dims[2]))
    return set_error(VQB_ESHAPE, "tokens [%d, %d) outside the cache capacity %lld", tok0, tok0 + n_tok,
                     (long long)g.dims[2]);
  const int64_t total = g.dims[0] * g.dims[1] * (int64_t)n_tok * g.gpr;
  const int64_t blocks = (total + 7) / 8;
  if (blocks > INT32_MAX) return set_error(VQB_ESHAPE, "too many sub-vectors");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  void* codes = const_cast<void*>(t->d_codes);
  const __half* books = reinterpret_cast<const __half*>(t->d_codebooks);
  if (x_dtype == VQB_F16)
    VQB_CUDA_CHECK(launch_pdl(cq_quantize_kernel<__half>, dim3((unsigned)blocks), dim3(256), 0, st, g, codes, books,
                              reinterpret_cast<const __half*>(d_x), xs_b, xs_h, xs_t, n_tok, tok0, d_len));
  else if (x_dtype == VQB_F32)
    VQB_CUDA_CHECK(launch_pdl(cq_quantize_kernel<float>, dim3((unsigned)blocks), dim3(256), 0, st, g, codes, books,
                              reinterpret_cast<const float*>(d_x), xs_b, xs_h, xs_t, n_tok, tok0, d_len));
  else
    return set_error(VQB_ECONFIG, "KV quantization takes fp16 or fp32 rows");
  VQB_LAUNCH_CHECK("cq_quantize_kernel");
  set_kernel("cq_quantize");
  return VQB_OK;
}
