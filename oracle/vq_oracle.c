/*
 * CPU ORACLE (C restatement) — TEST INFRASTRUCTURE AND CPU BASELINE ONLY.
 *
 * Multi-threaded (OpenMP) restatement of the reference's hot-path arithmetic,
 * used by tests/ to cross-check the numpy oracle and by bench.py's cpu_baseline
 * / --impl reference legs to time the reference algorithm on all host cores.
 * Never linked into or called from the product package.
 *
 *   vqo_dequant    <- vqforge.codec.dequantize       (pkg/src/vqforge/codec.py:391-408)
 *                     recon = +0.0f; recon += books[(r*n_regions + region)*K + code] per level
 *   vqo_gemv       <- reference_compute on dequantize(W) for gemv/gemm (sim.py:136-144)
 *   vqo_attention  <- reference_compute attention    (sim.py:145-155)
 *
 * Region ids are passed in (region_layout, codec.py:135-177, computed by the caller).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

int vqo_threads(void) {
#ifdef _OPENMP
  extern int omp_get_max_threads(void);
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* thread count of the following calls (the CPU baseline reports 1 thread and all cores) */
void vqo_set_threads(int n) {
#ifdef _OPENMP
  extern void omp_set_num_threads(int);
  omp_set_num_threads(n);
#else
  (void)n;
#endif
}

/* out[s*v + j] = sum over levels of books[((r*n_regions + regions[s])*K + codes[r*S + s])*v + j] */
int vqo_dequant(const int32_t* codes, int R, int64_t S, const float* books, int K, int v, int n_regions,
                const int32_t* regions, float* out) {
  int bad = 0;
#pragma omp parallel for schedule(static) reduction(| : bad)
  for (int64_t s = 0; s < S; ++s) {
    float acc[16];
    for (int j = 0; j < v; ++j) acc[j] = 0.0f;
    for (int r = 0; r < R; ++r) {
      const int32_t c = codes[(int64_t)r * S + s];
      if (c < 0 || c >= K) {
        bad = 1;
        continue;
      }
      const float* e = books + (((int64_t)r * n_regions + regions[s]) * K + c) * v;
      for (int j = 0; j < v; ++j) acc[j] = acc[j] + e[j];
    }
    memcpy(out + s * v, acc, sizeof(float) * v);
  }
  return bad ? -3 : 0;
}

/* y(rows, N) = x(rows, M) @ dequant(W)(M, N); W dequantised per row block, then a
 * cache-blocked fp32 accumulation parallelised over output columns. */
int vqo_gemv(const int32_t* codes, int R, int M, int N, int v, const float* books, int K, int n_regions,
             const int32_t* regions, const float* x, int rows, float* y) {
  const int64_t S = (int64_t)M * (N / v);
  float* w = (float*)malloc(sizeof(float) * (size_t)M * N);
  if (!w) return -4;
  int st = vqo_dequant(codes, R, S, books, K, v, n_regions, regions, w);
  if (st) {
    free(w);
    return st;
  }
  const int NB = 256;
#pragma omp parallel for schedule(static)
  for (int n0 = 0; n0 < N; n0 += NB) {
    const int n1 = n0 + NB < N ? n0 + NB : N;
    for (int b = 0; b < rows; ++b) {
      float acc[256];
      for (int n = n0; n < n1; ++n) acc[n - n0] = 0.0f;
      for (int m = 0; m < M; ++m) {
        const float xv = x[(int64_t)b * M + m];
        const float* wr = w + (int64_t)m * N;
        for (int n = n0; n < n1; ++n) acc[n - n0] += xv * wr[n];
      }
      for (int n = n0; n < n1; ++n) y[(int64_t)b * N + n] = acc[n - n0];
    }
  }
  free(w);
  return 0;
}

/* out(B,H,C) = softmax(q . K^T / sqrt(C)) V with K, V dense fp32 (B,H,T,C). */
int vqo_attention(const float* q, const float* k, const float* vv, int B, int H, int T, int C, float* out) {
  const float inv = 1.0f / sqrtf((float)C);
#pragma omp parallel for schedule(static)
  for (int bh = 0; bh < B * H; ++bh) {
    float* p = (float*)malloc(sizeof(float) * (size_t)T);
    const float* qb = q + (int64_t)bh * C;
    const float* kb = k + (int64_t)bh * T * C;
    const float* vb = vv + (int64_t)bh * T * C;
    float mx = -INFINITY;
    for (int t = 0; t < T; ++t) {
      float s = 0.0f;
      for (int c = 0; c < C; ++c) s += qb[c] * kb[(int64_t)t * C + c];
      p[t] = s * inv;
      if (p[t] > mx) mx = p[t];
    }
    float sum = 0.0f;
    for (int t = 0; t < T; ++t) {
      p[t] = expf(p[t] - mx);
      sum += p[t];
    }
    for (int c = 0; c < C; ++c) {
      float acc = 0.0f;
      for (int t = 0; t < T; ++t) acc += p[t] * vb[(int64_t)t * C + c];
      out[(int64_t)bh * C + c] = acc / sum;
    }
    free(p);
  }
  return 0;
}
