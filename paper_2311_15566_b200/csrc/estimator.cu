// estimator.cu -- batched latency / throughput scoring of candidate
// configurations and the controller's configuration choice, on the device.
//
// Restates, with the same double operations in the same order (no FMA:
// built with -fmad=false), the reference's
//   _prefill_at         costmodel.py:121-137 (table lookup / linear interpolation)
//   exec_latency        costmodel.py:144-152
//   throughput          costmodel.py:170-183
//   optimize_config     controller.py:79-117 (feasible branch: min latency within
//                       a 1% band, then fewest instances; fallback: max phi)
// One thread per query: a query is a (profiled shape, D, P, B, s_in, s_out)
// for the scoring kernel, and an (n_available, obtainable, rate) scenario for
// the selection kernel, which scans the candidates in sorted (D,P,M,B) order
// so every tie resolves the way the reference's stable sorts do.

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/spotkm.h"

namespace {

thread_local char g_eerr[256] = "";

int efail(const char* what, cudaError_t e) {
  snprintf(g_eerr, sizeof g_eerr, "%s: %s", what, cudaGetErrorString(e));
  return SK_ECUDA;
}

// _prefill_at over one shape's sorted (s_in, seconds) points
__device__ double prefill_at(const int64_t* xs, const double* ys, int n, int64_t s_in) {
  for (int k = 0; k < n; ++k)
    if (xs[k] == s_in) return ys[k];
  if (n == 1) return __ddiv_rn(__dmul_rn(ys[0], (double)s_in), (double)xs[0]);
  int a;
  if (s_in < xs[0]) {
    a = 0;
  } else if (s_in > xs[n - 1]) {
    a = n - 2;
  } else {
    a = n - 2;  // (unreachable fall-through keeps the last segment, as the for/else)
    for (int k = 0; k + 1 < n; ++k)
      if (xs[k] <= s_in && s_in <= xs[k + 1]) {
        a = k;
        break;
      }
  }
  const double frac = __ddiv_rn((double)(s_in - xs[a]), (double)(xs[a + 1] - xs[a]));
  return __dadd_rn(ys[a], __dmul_rn(frac, __dsub_rn(ys[a + 1], ys[a])));
}

__global__ void k_score(const sk_est_query* __restrict__ q, int n, const double* __restrict__ decode,
                        const int32_t* __restrict__ pre_ptr, const int64_t* __restrict__ pre_s,
                        const double* __restrict__ pre_v, double eta, double* __restrict__ latency,
                        double* __restrict__ phi) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const sk_est_query x = q[i];
  const int a = pre_ptr[x.shape], b = pre_ptr[x.shape + 1];
  const double init = prefill_at(pre_s + a, pre_v + a, b - a, x.s_in);
  // exec_latency: init, or init + s_out * decode
  const double lat = x.s_out == 0 ? init : __dadd_rn(init, __dmul_rn((double)x.s_out, decode[x.shape]));
  latency[i] = lat;
  if (phi) {
    // throughput: D*B / (latency / (P * eta))
    const double eff = __ddiv_rn(lat, __dmul_rn((double)x.P, eta));
    phi[i] = __ddiv_rn((double)((int64_t)x.D * x.B), eff);
  }
}

__global__ void k_select(const int32_t* __restrict__ n_inst, const double* __restrict__ phi,
                         const double* __restrict__ lat, int n_cfg, const int32_t* __restrict__ n_avail,
                         const int32_t* __restrict__ obtainable, const double* __restrict__ rate, int n_q,
                         double band, int32_t* __restrict__ choice) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_q) return;
  const int avail = n_avail[i], obt = obtainable[i];
  const double r = rate[i];
  // feasible branch: min latency (first minimum), then the band
  bool any = false;
  double best = 0.0;
  for (int c = 0; c < n_cfg; ++c)
    if (phi[c] >= r && n_inst[c] <= obt && (!any || lat[c] < best)) {
      best = lat[c];
      any = true;
    }
  if (any) {
    const double cut = __dmul_rn(best, band);
    int bc = -1;
    for (int c = 0; c < n_cfg; ++c) {
      if (!(phi[c] >= r && n_inst[c] <= obt && lat[c] <= cut)) continue;
      // min by (instances, latency, config order): strict, so ties keep the earlier config
      if (bc < 0 || n_inst[c] < n_inst[bc] || (n_inst[c] == n_inst[bc] && lat[c] < lat[bc])) bc = c;
    }
    choice[i] = bc;
    return;
  }
  // fallback: the highest phi among configs fitting n_available
  bool fit = false;
  double bphi = 0.0;
  for (int c = 0; c < n_cfg; ++c)
    if (n_inst[c] <= avail && (!fit || phi[c] > bphi)) {
      bphi = phi[c];
      fit = true;
    }
  if (!fit) {
    choice[i] = -1;
    return;
  }
  int bc = -1;
  for (int c = 0; c < n_cfg; ++c) {
    if (!(n_inst[c] <= avail && phi[c] == bphi)) continue;
    if (bc < 0 || n_inst[c] < n_inst[bc]) bc = c;
  }
  choice[i] = bc;
}

}  // namespace

extern "C" {

int sk_score_configs(const sk_est_query* d_q, int n, const double* d_decode, const int32_t* d_pre_ptr,
                     const int64_t* d_pre_s, const double* d_pre_v, double eta, double* d_latency,
                     double* d_phi, void* stream) {
  if (n <= 0) return SK_OK;
  k_score<<<(n + 127) / 128, 128, 0, static_cast<cudaStream_t>(stream)>>>(d_q, n, d_decode, d_pre_ptr, d_pre_s,
                                                                          d_pre_v, eta, d_latency, d_phi);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SK_OK : efail("k_score launch", e);
}

int sk_select_configs(const int32_t* d_n_inst, const double* d_phi, const double* d_latency, int n_cfg,
                      const int32_t* d_n_available, const int32_t* d_obtainable, const double* d_rate,
                      int n_queries, double band, int32_t* d_choice, void* stream) {
  if (n_queries <= 0) return SK_OK;
  k_select<<<(n_queries + 127) / 128, 128, 0, static_cast<cudaStream_t>(stream)>>>(
      d_n_inst, d_phi, d_latency, n_cfg, d_n_available, d_obtainable, d_rate, n_queries, band, d_choice);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SK_OK : efail("k_select launch", e);
}

const char* sk_estimator_error(void) { return g_eerr; }

}  // extern "C"
