// reshard.cu -- device memory, CUDA IPC and byte-pattern kernels for the
// migration executor (K3).  The copy kernel itself is k_copy in spotkm.cu.
//
// The executor's context buffers are plain cudaMalloc slabs so they can be
// exported with cudaIpcGetMemHandle and mapped by the peer ranks of the same
// box (one process per GPU); the destination GPU then pulls its transfers
// straight from the source GPU's slab over NVLink.
//
// Fill / verify write and check a counter-hash pattern: the 8-byte word at
// global byte offset x of a context object (a layer's parameter array, or one
// request's KV block of one layer) holds splitmix64(key ^ x/8), so the
// expected content of ANY shard after a reshard can be regenerated and
// compared byte for byte (SURVEY.md 8(d) "reshared tensors byte-identical").

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "../../include/spotkm.h"

namespace {

thread_local char g_rerr[256] = "";

int rfail(const char* what, cudaError_t e) {
  snprintf(g_rerr, sizeof g_rerr, "%s: %s", what, cudaGetErrorString(e));
  return SK_ECUDA;
}

__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// one CTA per region chunk of up to kRegionChunk bytes; regions are 8-byte
// aligned in size and base offset
constexpr int kR_TPB = 256;

__global__ void __launch_bounds__(kR_TPB) k_fill(const sk_region* __restrict__ regions, int n) {
  for (int r = blockIdx.y; r < n; r += gridDim.y) {
    const sk_region rg = regions[r];
    unsigned long long* p = reinterpret_cast<unsigned long long*>(rg.ptr);
    const unsigned long long words = rg.bytes >> 3, w0 = rg.base >> 3;
    for (unsigned long long i = (unsigned long long)blockIdx.x * kR_TPB + threadIdx.x; i < words;
         i += (unsigned long long)gridDim.x * kR_TPB)
      p[i] = mix64(rg.key ^ (w0 + i));
  }
}

__global__ void __launch_bounds__(kR_TPB) k_verify(const sk_region* __restrict__ regions, int n,
                                                   unsigned long long* __restrict__ bad) {
  unsigned long long local = 0;
  for (int r = blockIdx.y; r < n; r += gridDim.y) {
    const sk_region rg = regions[r];
    const unsigned long long* p = reinterpret_cast<const unsigned long long*>(rg.ptr);
    const unsigned long long words = rg.bytes >> 3, w0 = rg.base >> 3;
    for (unsigned long long i = (unsigned long long)blockIdx.x * kR_TPB + threadIdx.x; i < words;
         i += (unsigned long long)gridDim.x * kR_TPB)
      local += p[i] != mix64(rg.key ^ (w0 + i));
  }
  for (int off = 16; off; off >>= 1) local += __shfl_xor_sync(0xffffffffu, local, off);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(bad, local);
}

}  // namespace

extern "C" {

int sk_dev_alloc(uint64_t bytes, void** d_ptr) {
  cudaError_t e = cudaMalloc(d_ptr, bytes ? bytes : 16);
  return e == cudaSuccess ? SK_OK : rfail("cudaMalloc", e);
}

int sk_dev_free(void* d_ptr) {
  cudaError_t e = cudaFree(d_ptr);
  return e == cudaSuccess ? SK_OK : rfail("cudaFree", e);
}

int sk_ipc_get_handle(const void* d_ptr, void* handle64) {
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, const_cast<void*>(d_ptr));
  if (e != cudaSuccess) return rfail("cudaIpcGetMemHandle", e);
  static_assert(sizeof(h) == 64, "ipc handle size");
  memcpy(handle64, &h, 64);
  return SK_OK;
}

int sk_ipc_open_handle(const void* handle64, void** d_ptr) {
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, 64);
  cudaError_t e = cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess);
  return e == cudaSuccess ? SK_OK : rfail("cudaIpcOpenMemHandle", e);
}

int sk_ipc_close_handle(void* d_ptr) {
  cudaError_t e = cudaIpcCloseMemHandle(d_ptr);
  return e == cudaSuccess ? SK_OK : rfail("cudaIpcCloseMemHandle", e);
}

int sk_fill_regions(const sk_region* d_regions, int n, void* stream) {
  if (n <= 0) return SK_OK;
  dim3 grid(148 * 2, n < 65535 ? n : 65535);
  k_fill<<<grid, kR_TPB, 0, static_cast<cudaStream_t>(stream)>>>(d_regions, n);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SK_OK : rfail("k_fill launch", e);
}

int sk_verify_regions(const sk_region* d_regions, int n, unsigned long long* d_bad, void* stream) {
  if (n <= 0) return SK_OK;
  dim3 grid(148 * 2, n < 65535 ? n : 65535);
  k_verify<<<grid, kR_TPB, 0, static_cast<cudaStream_t>(stream)>>>(d_regions, n, d_bad);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SK_OK : rfail("k_verify launch", e);
}

const char* sk_reshard_error(void) { return g_rerr; }

}  // extern "C"

// ---------------------------------------------------------------------------
// Batched T_mig estimator: plan_timeline + migration_cost (costmodel.py:189-260)
// for many candidate plans at once, one thread per plan (each plan's timeline
// is a sequential recurrence over its transfers).  Same double operations, in
// the same order, as the host sk_plan_timeline / the reference.

namespace {

__global__ void k_migration_cost(const sk_tl_plan* __restrict__ plans, int n_plans,
                                 const int32_t* __restrict__ act_ptr, const int32_t* __restrict__ act_stage,
                                 const int32_t* __restrict__ src_inst, const int32_t* __restrict__ dst_inst,
                                 const double* __restrict__ bytes, const uint8_t* __restrict__ has_release,
                                 const double* __restrict__ release, double* __restrict__ scratch,
                                 uint8_t* __restrict__ flags, double bandwidth, double latency,
                                 double* __restrict__ cost) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n_plans) return;
  const sk_tl_plan p = plans[q];
  double* out_free = scratch + 2 * (size_t)p.inst_base;
  double* in_free = out_free + p.n_inst;
  uint8_t* has_out = flags + 2 * (size_t)p.inst_base;
  uint8_t* has_in = has_out + p.n_inst;
  for (int i = 0; i < p.n_inst; ++i) {
    has_out[i] = 0;
    has_in[i] = 0;
  }
  const double start = p.start;
  double prev = start;
  // progressive start: each start_stage action's rank in the stable sort by
  // stage is counted from the (static) stage list, so no per-plan array
  // bounds the number of stages
  double stall = 0.0;
  bool any_start = false;
  for (int a = p.act_begin; a < p.act_end; ++a) {
    double end = prev;
    bool moved = false;
    for (int k = act_ptr[a]; k < act_ptr[a + 1]; ++k) {
      const int s = src_inst[k], d = dst_inst[k];
      if (s == d) continue;
      moved = true;
      const int gs = p.inst_base + s, gd = p.inst_base + d;
      const double so = has_out[s] ? out_free[s] : (has_release[gs] ? release[gs] : start);
      const double di = has_in[d] ? in_free[d] : (has_release[gd] ? release[gd] : start);
      const double begin = so > di ? so : di;
      const double fin = begin + bytes[k] / bandwidth;
      out_free[s] = fin;
      has_out[s] = 1;
      in_free[d] = fin;
      has_in[d] = 1;
      if (fin > end) end = fin;
    }
    if (moved) end += latency;
    const double e = end > prev ? end : prev;
    prev = e;
    const int st = act_stage[a];
    if (p.progressive && st >= 0) {
      int o = 0;  // entries before this one in sorted(starts, key=stage)
      for (int b = p.act_begin; b < p.act_end; ++b) {
        const int sb = act_stage[b];
        if (sb >= 0 && (sb < st || (sb == st && b < a))) ++o;
      }
      // max(stall, x) over the sorted order: the value is order-independent
      const double x = e - start - (double)o * p.step;
      if (x > stall) stall = x;
      any_start = true;
    }
  }
  const double last = p.act_end > p.act_begin ? prev : start;
  const double total = (last > start ? last : start) - start;
  if (!p.progressive || !any_start) {
    cost[q] = total;
    return;
  }
  cost[q] = stall > 0.0 ? stall : 0.0;
}

}  // namespace

extern "C" int sk_migration_cost_batched(const sk_tl_plan* d_plans, int n_plans, const int32_t* d_act_ptr,
                                         const int32_t* d_act_stage, const int32_t* d_src_inst,
                                         const int32_t* d_dst_inst, const double* d_bytes,
                                         const uint8_t* d_has_release, const double* d_release,
                                         double* d_scratch, uint8_t* d_flags, double bandwidth,
                                         double latency, double* d_cost, void* stream) {
  if (n_plans <= 0) return SK_OK;
  const int tpb = 128;
  k_migration_cost<<<(n_plans + tpb - 1) / tpb, tpb, 0, static_cast<cudaStream_t>(stream)>>>(
      d_plans, n_plans, d_act_ptr, d_act_stage, d_src_inst, d_dst_inst, d_bytes, d_has_release,
      d_release, d_scratch, d_flags, bandwidth, latency, d_cost);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SK_OK : rfail("k_migration_cost launch", e);
}
