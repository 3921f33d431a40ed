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
#include <dlfcn.h>
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

// ---------------------------------------------------------------------------
// k_exec: one persistent launch per rank executes the rank's share of a
// MigrationPlan in plan order (migration.py:311-384; the paper's engine runs
// it as batched async send/recv).
//
//   * CTA 0 is the monitor; CTAs 1.. are copy workers.
//   * Workers take 1 MiB chunks in plan (round) order from an atomic work
//     counter and copy them with 16-B vector loads/stores over the peer
//     mapping (NVLink).  After a chunk every thread fences at system scope
//     and the CTA bumps the round's done counter.
//   * A chunk whose destination range reuses arena space freed at the end of
//     round d (a plan `release`, recycled by the host-side arena allocator)
//     first waits until EVERY rank has completed rounds 0..d -- so the old
//     bytes are gone only when every reader of them is done.  This is the
//     only cross-rank wait: rounds otherwise overlap, as the reference's
//     timeline models them (costmodel.py:189-228).
//   * The monitor publishes this rank's progress (rounds 0..p-1 complete) for
//     the peers, and raises stage-ready flags (with a %globaltimer stamp) as
//     soon as global progress passes the round each start_stage marker follows
//     (migration.py:352-371) -- the device-side readiness signal a consumer
//     (context daemon client) waits on with cuStreamWaitValue32 or a poll.
//
// Control block (u32 words, device memory, IPC-exportable):
//   [0] work_next  [1] progress  [2] error  [3] reserved
//   [4 .. 4+R)     done chunks per round
//   then n_stages stage flags, then (8-B aligned) n_stages + 1 u64 stamps:
//   the launch start and each stage's ready time (ns, %globaltimer).

// a consumer-side wait on a (possibly IPC-mapped) device flag: one thread
// spins until *flag >= value, so work queued after it on the stream runs only
// once the producer has raised the flag; status = 0 ok, 1 timeout
__global__ void k_wait_flag(const unsigned* flag, unsigned value, unsigned long long timeout_ns,
                            unsigned* status) {
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (*reinterpret_cast<const volatile unsigned*>(flag) < value) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > timeout_ns) {
      if (status) *status = 1u;
      return;
    }
    __nanosleep(1000);
  }
  __threadfence_system();
  if (status) *status = 0u;
}

constexpr int kX_TPB = 512;

__device__ __forceinline__ unsigned ld_volatile_u32(const unsigned* p) {
  return *reinterpret_cast<const volatile unsigned*>(p);
}

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

struct ExecArgs {
  const sk_exec_chunk* chunks;
  int n_chunks;
  const unsigned* round_total;  // chunks per round issued by this rank
  int n_rounds;
  const int* stage_round;       // per stage: ready once rounds 0..stage_round complete (-1: at start)
  int n_stages;
  unsigned* ctl;
  const unsigned* const* peer_progress;  // every OTHER rank's progress word
  int n_peers;
  unsigned long long timeout_ns;
  unsigned* flag_mirror;  // optional host-mapped copy of the stage flags (another process polls it)
};

__device__ __forceinline__ unsigned* exec_flags(const ExecArgs& A) { return A.ctl + 4 + A.n_rounds; }
__device__ __forceinline__ unsigned long long* exec_stamps(const ExecArgs& A) {
  const size_t w = (size_t)4 + A.n_rounds + A.n_stages;
  return reinterpret_cast<unsigned long long*>(A.ctl + ((w + 1) & ~(size_t)1));
}

__device__ unsigned global_progress(const ExecArgs& A) {
  unsigned g = ld_volatile_u32(A.ctl + 1);
  for (int i = 0; i < A.n_peers; ++i) {
    const unsigned v = ld_volatile_u32(A.peer_progress[i]);
    g = v < g ? v : g;
  }
  return g;
}

__global__ void __launch_bounds__(kX_TPB) k_exec(const ExecArgs A) {
  __shared__ int s_idx;
  __shared__ int s_abort;
  __shared__ unsigned s_g;  // global progress last seen by this CTA (block-uniform)
  const unsigned long long t0 = global_ns();
  if (blockIdx.x == 0) {
    // ---- monitor ----
    if (threadIdx.x != 0) return;
    unsigned* flags = exec_flags(A);
    unsigned long long* stamps = exec_stamps(A);
    stamps[0] = t0;
    unsigned p = 0;
    int pending = A.n_stages;
    while (true) {
      unsigned q = p;
      while ((int)q < A.n_rounds && ld_volatile_u32(A.ctl + 4 + q) >= A.round_total[q]) ++q;
      if (q != p) {
        __threadfence_system();  // the rounds' data before the progress word
        *reinterpret_cast<volatile unsigned*>(A.ctl + 1) = q;
        p = q;
      }
      if (pending) {
        const unsigned g = global_progress(A);
        for (int s = 0; s < A.n_stages; ++s) {
          if (flags[s] == 0u && (long long)A.stage_round[s] < (long long)g) {
            stamps[1 + s] = global_ns();
            __threadfence_system();
            *reinterpret_cast<volatile unsigned*>(flags + s) = 1u;
            if (A.flag_mirror) *reinterpret_cast<volatile unsigned*>(A.flag_mirror + s) = 1u;
            --pending;
          }
        }
      }
      if ((int)p >= A.n_rounds && pending == 0) break;
      if (ld_volatile_u32(A.ctl + 2) != 0u) break;
      if (global_ns() - t0 > A.timeout_ns) {
        atomicExch(A.ctl + 2, 2u);  // monitor timeout
        break;
      }
      __nanosleep(200);
    }
    return;
  }
  // ---- workers ----
  if (threadIdx.x == 0) s_g = 0;
  while (true) {
    if (threadIdx.x == 0) {
      s_idx = (int)atomicAdd(A.ctl + 0, 1u);
      s_abort = 0;
    }
    __syncthreads();
    const int idx = s_idx;
    if (idx >= A.n_chunks) break;
    const sk_exec_chunk c = A.chunks[idx];
    // (s_g is read by every thread after the barrier above and written only
    // by thread 0 between two barriers: the branch is block-uniform)
    if (c.wait_round >= 0 && s_g <= (unsigned)c.wait_round) {
      if (threadIdx.x == 0) {
        // recycled space: every rank must be past round wait_round
        while (true) {
          const unsigned g = global_progress(A);
          s_g = g;
          if (g > (unsigned)c.wait_round) break;
          if (ld_volatile_u32(A.ctl + 2) != 0u || global_ns() - t0 > A.timeout_ns) {
            atomicCAS(A.ctl + 2, 0u, 1u);  // worker timeout
            s_abort = 1;
            break;
          }
          __nanosleep(500);
        }
        __threadfence_system();
      }
      __syncthreads();
      if (s_abort) break;
    }
    const unsigned char* src = reinterpret_cast<const unsigned char*>(c.src);
    unsigned char* dst = reinterpret_cast<unsigned char*>(c.dst);
    uint64_t done = 0;
    if (((c.src | c.dst) & 15ull) == 0) {
      const uint64_t nv = c.bytes >> 4;
      const int4* s4 = reinterpret_cast<const int4*>(src);
      int4* d4 = reinterpret_cast<int4*>(dst);
      uint64_t i = threadIdx.x;
      constexpr int U = 8;
      for (; i + (U - 1) * kX_TPB < nv; i += U * kX_TPB) {
        int4 t[U];
#pragma unroll
        for (int u = 0; u < U; ++u) t[u] = __ldcs(s4 + i + u * kX_TPB);
#pragma unroll
        for (int u = 0; u < U; ++u) __stcs(d4 + i + u * kX_TPB, t[u]);
      }
      for (; i < nv; i += kX_TPB) __stcs(d4 + i, __ldcs(s4 + i));
      done = nv << 4;
    }
    for (uint64_t i = done + threadIdx.x; i < c.bytes; i += kX_TPB) dst[i] = src[i];
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) atomicAdd(A.ctl + 4 + c.round, 1u);
  }
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

int sk_memcpy_batched(const sk_copy* h_copies, int n, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  for (int i = 0; i < n; ++i) {
    cudaError_t e = cudaMemcpyAsync(reinterpret_cast<void*>(h_copies[i].dst),
                                    reinterpret_cast<const void*>(h_copies[i].src), h_copies[i].bytes,
                                    cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return rfail("cudaMemcpyAsync", e);
  }
  return SK_OK;
}

int sk_d2h(void* h_dst, const void* d_src, uint64_t bytes) {
  cudaError_t e = cudaMemcpy(h_dst, d_src, bytes, cudaMemcpyDeviceToHost);
  return e == cudaSuccess ? SK_OK : rfail("cudaMemcpy D2H", e);
}

int sk_wait_flag(const uint32_t* d_flag, uint32_t value, double timeout_s, uint32_t* d_status, void* stream) {
  k_wait_flag<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(d_flag, value,
                                                                (unsigned long long)(timeout_s * 1e9), d_status);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SK_OK : rfail("k_wait_flag launch", e);
}

// cuStreamWaitValue32 from the driver, resolved at run time (no link-time
// libcuda dependency): a wait executed by the stream's front end, not by a
// kernel, so it holds no SM -- the right primitive when the producer is a
// kernel of ANOTHER process on the same GPU (contexts time-slice; a spinning
// consumer kernel can starve the producer).
typedef int (*wait_value_fn)(void* stream, unsigned long long addr, uint32_t value, unsigned flags);

int sk_stream_wait_flag(const uint32_t* d_flag, uint32_t value, void* stream) {
  static wait_value_fn fn = [] {
    void* h = dlopen("libcuda.so.1", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return (wait_value_fn) nullptr;
    void* f = dlsym(h, "cuStreamWaitValue32_v2");
    if (!f) f = dlsym(h, "cuStreamWaitValue32");
    return reinterpret_cast<wait_value_fn>(f);
  }();
  if (!fn) {
    snprintf(g_rerr, sizeof g_rerr, "cuStreamWaitValue32 not available");
    return SK_ECUDA;
  }
  const int rc = fn(stream, (unsigned long long)(uintptr_t)d_flag, value, 0x0 /* CU_STREAM_WAIT_VALUE_GEQ */);
  if (rc != 0) {
    snprintf(g_rerr, sizeof g_rerr, "cuStreamWaitValue32 failed: CUresult %d", rc);
    return SK_ECUDA;
  }
  return SK_OK;
}

int sk_host_register(void* h_ptr, uint64_t bytes, void** d_ptr) {
  cudaError_t e = cudaHostRegister(h_ptr, bytes, cudaHostRegisterMapped);
  if (e != cudaSuccess) return rfail("cudaHostRegister", e);
  e = cudaHostGetDevicePointer(d_ptr, h_ptr, 0);
  return e == cudaSuccess ? SK_OK : rfail("cudaHostGetDevicePointer", e);
}

int sk_host_unregister(void* h_ptr) {
  cudaError_t e = cudaHostUnregister(h_ptr);
  return e == cudaSuccess ? SK_OK : rfail("cudaHostUnregister", e);
}

int sk_exec_reset(uint32_t* d_ctl, int n_rounds, int n_stages, void* stream) {
  const int64_t w = 4 + (int64_t)n_rounds + n_stages;
  const size_t bytes = (size_t)(((w + 1) & ~(int64_t)1) * 4 + 8 * (int64_t)(n_stages + 1));
  cudaError_t e = cudaMemsetAsync(d_ctl, 0, bytes, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SK_OK : rfail("exec control reset", e);
}

int64_t sk_exec_ctl_bytes(int n_rounds, int n_stages) {
  const int64_t w = 4 + (int64_t)n_rounds + n_stages;
  return ((w + 1) & ~(int64_t)1) * 4 + 8 * (int64_t)(n_stages + 1);
}

int sk_exec_plan(const sk_exec_chunk* d_chunks, int n_chunks, const uint32_t* d_round_total, int n_rounds,
                 const int32_t* d_stage_round, int n_stages, uint32_t* d_ctl,
                 const uint32_t* const* d_peer_progress, int n_peers, uint32_t* d_flag_mirror, int n_ctas,
                 double timeout_s, void* stream) {
  if (n_chunks < 0 || n_rounds < 0 || n_stages < 0 || n_peers < 0) {
    snprintf(g_rerr, sizeof g_rerr, "negative sizes");
    return SK_EINVAL;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // a fresh control block per run (the caller orders this before any peer
  // reads it, e.g. with a barrier between sk_exec_plan calls of a new run)
  cudaError_t e = cudaMemsetAsync(d_ctl, 0, (size_t)sk_exec_ctl_bytes(n_rounds, n_stages), s);
  if (e != cudaSuccess) return rfail("exec control reset", e);
  if (n_ctas <= 1) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    n_ctas = 2 * sms;  // two 512-thread CTAs per SM, all co-resident: the monitor + workers
  }
  ExecArgs A{d_chunks, n_chunks, d_round_total, n_rounds, d_stage_round, n_stages, d_ctl,
             d_peer_progress, n_peers, (unsigned long long)(timeout_s * 1e9), d_flag_mirror};
  k_exec<<<n_ctas, kX_TPB, 0, s>>>(A);
  e = cudaGetLastError();
  return e == cudaSuccess ? SK_OK : rfail("k_exec launch", e);
}

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
