// tp.cu — tensor-parallel collectives fused into the decode GEMV over peer memory
// (the NCCL calls they replace are in tp.py / decode.py).
//
// A row-parallel linear (Megatron o / down) ends in an all-reduce of rows x N
// partial outputs, a column-parallel one (qkv / gate_up when its output must be
// replicated) in an all-gather. At decode sizes (8-64 KB) the cost is latency, not
// bandwidth, so the B200 design is a one-shot push: the GEMV's epilogue stores
// each reduced output element straight into the current slot of every rank's
// symmetric buffer (NVLink peer stores, issued as soon as a column block is
// finished, overlapping the remaining tiles), the grid's last CTA signals every
// rank with one system-scope release add, and a small finish kernel on each rank
// waits for all `world` signals and sums the slots in rank order — the same bits on
// every rank, deterministic, no NCCL launch on the critical path. Epochs with two
// slot parities make consecutive collectives safe without any reset: the producer
// of epoch e+2 on any rank runs after every rank's finish of epoch e (it follows
// its own finish of e+1, which waited for every rank's producer of e+1, each of
// which followed that rank's finish of e).
#include <cstring>
#include <mutex>
#include <unordered_map>

#include "common.cuh"

namespace vqb {

int gemv_dispatch(const VqbTensor* w, const void* x, int x_dtype, int rows, void* y, int y_dtype,
                  const VqbLaunch* L, void* ws, size_t ws_bytes, cudaStream_t st, bool* used_fast,
                  const VqbPeerComm* tp, int tp_mode, const struct GemvXf* xf);

constexpr unsigned long long kTpTimeoutNs = 10ull * 1000 * 1000 * 1000;

__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__global__ void __launch_bounds__(256) tp_finish_kernel(char* me, int world, int mode, int rows, int n_local,
                                                        int64_t slot_elems, void* y, int y_dtype) {
  pdl_launch_dependents();
  pdl_wait();  // this rank's producer GEMV has finished (and signalled)
  const int e = tp_epoch_of(me);
  const int par = e & 1;
  const unsigned long long target = (unsigned long long)world * (unsigned long long)((e >> 1) + 1);
  if (threadIdx.x == 0) {
    const unsigned long long* arr = reinterpret_cast<const unsigned long long*>(me) + par;
    const unsigned long long t0 = gtimer();
    while (ld_acquire_sys_u64(arr) < target) {
      if (gtimer() - t0 > kTpTimeoutNs) {
        atomicOr(reinterpret_cast<unsigned*>(me + kTpOffErr), 1u);
        break;
      }
      __nanosleep(128);
    }
  }
  __syncthreads();
  const float* slots = reinterpret_cast<const float*>(me + VQB_TP_HEADER_BYTES);
  const int64_t n_out = (int64_t)rows * n_local * (mode == VQB_TP_ALLGATHER ? world : 1);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_out; i += (int64_t)gridDim.x * blockDim.x) {
    float s;
    if (mode == VQB_TP_ALLREDUCE) {
      s = 0.f;
      for (int r = 0; r < world; ++r) s += __ldcg(slots + ((int64_t)par * world + r) * slot_elems + i);
    } else {
      s = __ldcg(slots + (int64_t)par * slot_elems + i);
    }
    store_from_f32(y, y_dtype, i, s);
  }
  // the last CTA (every CTA has read the epoch) advances it for the next collective
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned prev;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;"
                 : "=r"(prev) : "l"(reinterpret_cast<unsigned*>(me + kTpOffFinish)) : "memory");
    if (prev == gridDim.x - 1) {
      *reinterpret_cast<volatile unsigned*>(me + kTpOffFinish) = 0u;
      *reinterpret_cast<volatile int*>(me + kTpOffEpoch) = e + 1;
    }
  }
}

static int check_comm(const VqbPeerComm* c) {
  if (!c || c->world < 1 || c->world > VQB_TP_MAX_WORLD || c->rank < 0 || c->rank >= c->world || c->slot_elems < 1)
    return set_error(VQB_ECONFIG, "bad peer communicator (rank/world/slot_elems)");
  for (int i = 0; i < c->world; ++i)
    if (!c->d_peer[i] || (reinterpret_cast<uintptr_t>(c->d_peer[i]) & 255))
      return set_error(VQB_ECONFIG, "peer buffer %d missing or not 256-byte aligned", i);
  return VQB_OK;
}

}  // namespace vqb

using namespace vqb;

extern "C" int64_t vqb_tp_buffer_bytes(int32_t world, int64_t slot_elems) {
  if (world < 1 || world > VQB_TP_MAX_WORLD || slot_elems < 1) return set_error(VQB_ECONFIG, "bad TP buffer size");
  return VQB_TP_HEADER_BYTES + 2 * (int64_t)world * slot_elems * 4;
}

extern "C" int vqb_ipc_get_handle(const void* d_ptr, void* handle64, int64_t* offset) {
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  // the handle names the whole allocation: report where the pointer sits inside it
  typedef int (*GetRange)(unsigned long long*, size_t*, unsigned long long);
  static GetRange get_range = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      get_range = reinterpret_cast<GetRange>(fn);
  });
  if (!get_range) return set_error(VQB_ECUDA, "cuMemGetAddressRange unavailable");
  unsigned long long base = 0;
  size_t size = 0;
  if (get_range(&base, &size, reinterpret_cast<unsigned long long>(d_ptr)) != 0)
    return set_error(VQB_ECUDA, "cuMemGetAddressRange failed for %p", d_ptr);
  cudaIpcMemHandle_t h;
  VQB_CUDA_CHECK(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  std::memcpy(handle64, &h, sizeof(h));
  *offset = (int64_t)(reinterpret_cast<unsigned long long>(d_ptr) - base);
  return VQB_OK;
}

static std::mutex g_ipc_mu;
static std::unordered_map<void*, void*> g_ipc_base;  // opened pointer -> mapped allocation base

extern "C" int vqb_ipc_open_handle(const void* handle64, int64_t offset, void** d_ptr) {
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, sizeof(h));
  void* base = nullptr;
  VQB_CUDA_CHECK(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
  *d_ptr = reinterpret_cast<char*>(base) + offset;
  std::lock_guard<std::mutex> lock(g_ipc_mu);
  g_ipc_base[*d_ptr] = base;
  return VQB_OK;
}

extern "C" int vqb_ipc_close_handle(void* d_ptr) {
  void* base = nullptr;
  {
    std::lock_guard<std::mutex> lock(g_ipc_mu);
    auto it = g_ipc_base.find(d_ptr);
    if (it == g_ipc_base.end()) return set_error(VQB_ECONFIG, "pointer was not opened with vqb_ipc_open_handle");
    base = it->second;
    g_ipc_base.erase(it);
  }
  VQB_CUDA_CHECK(cudaIpcCloseMemHandle(base));
  return VQB_OK;
}

extern "C" int vqb_gemv_tp(const VqbTensor* w, const void* d_x, int32_t x_dtype, int32_t rows, int32_t mode,
                           const VqbPeerComm* comm, const VqbLaunch* launch, void* d_ws, size_t ws_bytes,
                           void* stream) {
  int s = check_comm(comm);
  if (s) return s;
  if (mode != VQB_TP_ALLREDUCE && mode != VQB_TP_ALLGATHER) return set_error(VQB_ECONFIG, "unknown TP mode %d", mode);
  if (!w || w->ndim != 2) return set_error(VQB_ESHAPE, "quantized weight must be 2-D (M, N)");
  const int64_t need = (int64_t)rows * w->dims[1] * (mode == VQB_TP_ALLGATHER ? comm->world : 1);
  if (need > comm->slot_elems)
    return set_error(VQB_ECAPACITY, "TP slot of %lld elements < %lld needed", (long long)comm->slot_elems,
                     (long long)need);
  s = gemv_dispatch(w, d_x, x_dtype, rows, nullptr, VQB_F32, launch, d_ws, ws_bytes,
                    reinterpret_cast<cudaStream_t>(stream), nullptr, comm, mode, nullptr);
  if (s) return s;
  set_kernel("gemv_tp");
  return VQB_OK;
}

extern "C" int vqb_tp_finish(const VqbPeerComm* comm, int32_t mode, int32_t rows, int32_t n_local, void* d_y,
                             int32_t y_dtype, void* stream) {
  int s = check_comm(comm);
  if (s) return s;
  if (mode != VQB_TP_ALLREDUCE && mode != VQB_TP_ALLGATHER) return set_error(VQB_ECONFIG, "unknown TP mode %d", mode);
  if (rows < 1 || n_local < 1) return set_error(VQB_ESHAPE, "bad TP finish shape");
  if (y_dtype < VQB_F32 || y_dtype > VQB_BF16) return set_error(VQB_ECONFIG, "unknown output dtype");
  const int64_t n_out = (int64_t)rows * n_local * (mode == VQB_TP_ALLGATHER ? comm->world : 1);
  if (n_out > comm->slot_elems) return set_error(VQB_ECAPACITY, "TP slot smaller than the output");
  const int blocks = (int)std::min<int64_t>(ceil_div(n_out, 256), 2 * (int64_t)sm_count());
  VQB_CUDA_CHECK(launch_pdl(tp_finish_kernel, dim3(blocks), dim3(256), 0, reinterpret_cast<cudaStream_t>(stream),
                            reinterpret_cast<char*>(comm->d_peer[comm->rank]), (int)comm->world, (int)mode, (int)rows,
                            (int)n_local, (int64_t)comm->slot_elems, d_y, (int)y_dtype));
  VQB_LAUNCH_CHECK("tp_finish_kernel");
  set_kernel("tp_finish");
  return VQB_OK;
}

extern "C" int vqb_tp_take_error(const VqbPeerComm* comm, int32_t* out) {
  int s = check_comm(comm);
  if (s) return s;
  VQB_CUDA_CHECK(cudaDeviceSynchronize());
  unsigned v = 0;
  char* me = reinterpret_cast<char*>(comm->d_peer[comm->rank]);
  VQB_CUDA_CHECK(cudaMemcpy(&v, me + kTpOffErr, 4, cudaMemcpyDeviceToHost));
  const unsigned z = 0;
  VQB_CUDA_CHECK(cudaMemcpy(me + kTpOffErr, &z, 4, cudaMemcpyHostToDevice));
  *out = (int32_t)v;
  return VQB_OK;
}
