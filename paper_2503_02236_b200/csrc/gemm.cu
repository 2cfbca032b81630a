// gemm.cu — prefill GEMM entry point (placeholder until the tcgen05 kernel lands):
// routes to the generic fused kernel so the API is complete and parity-correct.
#include "common.cuh"

namespace vqb {
int gemv_dispatch(const VqbTensor* w, const void* x, int x_dtype, int rows, void* y, int y_dtype,
                  const VqbLaunch* L, void* ws, size_t ws_bytes, cudaStream_t st, bool* used_fast);

int gemm_usage(VqbUsage* u) {
  *u = VqbUsage{};
  return VQB_OK;
}
}  // namespace vqb

extern "C" int vqb_gemm(const VqbTensor* w, const void* d_x, int32_t x_dtype, int32_t rows, void* d_y,
                        int32_t y_dtype, const VqbLaunch* launch, void* d_ws, size_t ws_bytes, void* stream) {
  VqbLaunch l = launch ? *launch : VqbLaunch{};
  l.flags |= VQB_FLAG_FORCE_GENERIC;
  return vqb::gemv_dispatch(w, d_x, x_dtype, rows, d_y, y_dtype, &l, d_ws, ws_bytes,
                            reinterpret_cast<cudaStream_t>(stream), nullptr);
}
