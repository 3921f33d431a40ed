// spotkm.cu -- sm_100a kernels + C ABI for SpotServe's device-mapping and
// context-migration hot path.  See include/spotkm.h for the contract and
// DESIGN.md for the data layout and rooflines.
//
// Kernels
//   k_weights      K1  dense W[R][C] (build_graph, mapping.py:184-216)
//   k_fuse<g, lpg> K2a per fused GPU group (one fused row): g x g weight
//                      blocks built on the fly, inner KM, fused weight
//                      (mapping.py:258-269)
//   k_outer<CPL, mode, W>
//                  K2b W warps per plan: outer KM on the dictionary-coded,
//                      zero-padded fused matrix (mapping.py:271, 71-122) +
//                      expansion and total_weight in reference order
//                      (mapping.py:272-283)
//   k_sweep_expand     compact sweep descriptors -> rows/segments
//   k_copy         K3  byte-range copies (peer-mapped push/pull over NVLink)
//
// Exactness: no fast-math, -fmad=false.  Every float op of the reference's
// _hungarian_max is replayed in the same order: cost = -w;
// cur = (cost - u[i0]) - v[j]; strict '<' in the slack update and argmin with
// the lowest column winning ties.

#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdlib.h>
#include <stdint.h>
#include <type_traits>
#include <stdio.h>

#include "../../include/spotkm.h"
#include "exact.cuh"

namespace {

thread_local char g_err[512] = "";

int set_err(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int cuda_check(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_err(SK_ECUDA, "%s: %s", what, cudaGetErrorString(e));
  return SK_OK;
}

constexpr double kInf = __builtin_huge_val();
constexpr unsigned kFull = 0xffffffffu;

// ---------------------------------------------------------------------------
// context algebra on device

struct Col {
  int d;       // 1-based new pipeline
  int s0, s1;  // stage layer block [s0, s1)           (domain.py:271-283)
  int i0, i1;  // shard interval [i0, i1) in 1/K units (domain.py:286-288)
};

__device__ __forceinline__ Col col_of(const sk_plan& p, int c) {
  const int m = c % p.M;
  const int t = c / p.M;
  const int st = t % p.P;
  const int d = t / p.P;
  const int q = p.L / p.P, r = p.L % p.P;
  Col o;
  o.d = d + 1;
  o.s0 = st * q + min(st, r);
  o.s1 = o.s0 + q + (st < r ? 1 : 0);
  const int w = p.K / p.M;
  o.i0 = m * w;
  o.i1 = o.i0 + w;
  return o;
}

__device__ __forceinline__ long long seg_num(const sk_segment& s, const Col& c) {
  const int ol = min(s.l1, c.s1) - max(s.l0, c.s0);
  const int oi = min(s.b, c.i1) - max(s.a, c.i0);
  if (ol <= 0 || oi <= 0) return 0;
  if (s.pipe != 0 && s.pipe != c.d) return 0;
  return (long long)ol * (long long)oi * s.unit;
}

// N / K correctly rounded: exact N (< 2^53) and K, one IEEE division -- the
// same value float(Fraction(N, K)) gives (domain.py:320).
__device__ __forceinline__ double num_to_w(long long n, int K) {
  return __ddiv_rn(__ll2double_rn(n), (double)K);
}

// ---- general-range plans (SK_PLAN_GENERIC): 64-bit endpoints, 128-bit
// numerators, one correctly rounded conversion (exact.cuh) -- the same
// float(Fraction) value for inputs beyond the regular encoding's range

typedef __int128 i128;

struct ColW {
  int d;
  int s0, s1;
  long long i0, i1;
};

__device__ __forceinline__ ColW col_of_w(const sk_plan& p, int c) {
  const int m = c % p.M;
  const int t = c / p.M;
  const int st = t % p.P;
  const int d = t / p.P;
  const int q = p.L / p.P, r = p.L % p.P;
  ColW o;
  o.d = d + 1;
  o.s0 = st * q + min(st, r);
  o.s1 = o.s0 + q + (st < r ? 1 : 0);
  const long long w = p.Kw / p.M;
  o.i0 = (long long)m * w;
  o.i1 = o.i0 + w;
  return o;
}

__device__ __forceinline__ const sk_segment_wide& wide_at(const sk_segment* segs, int s) {
  return *reinterpret_cast<const sk_segment_wide*>(segs + s);
}

__device__ __forceinline__ i128 seg_num_wide(const sk_segment_wide& s, const ColW& c) {
  const int ol = min(s.l1, c.s1) - max(s.l0, c.s0);
  const long long oi = (s.b < c.i1 ? s.b : c.i1) - (s.a > c.i0 ? s.a : c.i0);
  if (ol <= 0 || oi <= 0) return 0;
  if (s.pipe != 0 && s.pipe != c.d) return 0;
  return (i128)ol * (i128)oi * (i128)s.unit;  // < 2^127: bounded on the host
}

__device__ __forceinline__ double weight_generic(const sk_plan& p, const int32_t* __restrict__ row_ptr,
                                                 const sk_segment* __restrict__ segs, int r, int c) {
  const ColW col = col_of_w(p, c);
  const int s0 = row_ptr[p.row_base + r], s1 = row_ptr[p.row_base + r + 1];
  i128 acc = 0;
  for (int s = s0; s < s1; s += 2) acc += seg_num_wide(wide_at(segs, s), col);
  return sk_exact::rat_to_double(acc, p.Kw);
}

// one 32-byte segment as two 16-byte loads (one L2 request per segment
// instead of one per field when the threads of a warp read different rows)
__device__ __forceinline__ sk_segment load_seg(const sk_segment* p) {
  const int4* q = reinterpret_cast<const int4*>(p);
  const int4 u = __ldg(q), v = __ldg(q + 1);
  sk_segment s;
  s.l0 = u.x;
  s.l1 = u.y;
  s.a = u.z;
  s.b = u.w;
  s.pipe = v.x;
  s.reserved = v.y;
  s.unit = (long long)(((unsigned long long)(unsigned)v.w << 32) | (unsigned)v.z);
  return s;
}

__device__ __forceinline__ double weight_at(const sk_plan& p, const int32_t* __restrict__ row_ptr,
                                            const sk_segment* __restrict__ segs, int r, int c) {
  const Col col = col_of(p, c);
  const int s0 = row_ptr[p.row_base + r], s1 = row_ptr[p.row_base + r + 1];
  long long acc = 0;
  for (int s = s0; s < s1; ++s) acc += seg_num(load_seg(segs + s), col);
  return num_to_w(acc, p.K);
}

// CPython >= 3.12 builtin sum() over floats with int start 0: the first item
// goes through int + float, the rest through Neumaier compensation, and the
// compensation is added once at the end when non-zero and finite
// (mapping.py:268-269 fused_weight="sum"; SURVEY.md finding 6).
template <int N>
__device__ __forceinline__ double py_builtin_sum(const double (&x)[N]) {
  double f = 0.0 + x[0];
  double c = 0.0;
#pragma unroll
  for (int i = 1; i < N; ++i) {
    const double xi = x[i];
    const double t = f + xi;
    if (fabs(f) >= fabs(xi))
      c += (f - t) + xi;
    else
      c += (xi - t) + f;
    f = t;
  }
  if (c != 0.0 && isfinite(c)) f += c;
  return f;
}

// register-resident dynamic indexing for tiny arrays
template <int N, typename T>
__host__ __device__ __forceinline__ T sel(const T (&a)[N], int i) {
  T r = a[0];
#pragma unroll
  for (int k = 1; k < N; ++k)
    if (i == k) r = a[k];
  return r;
}
template <int N, typename T>
__host__ __device__ __forceinline__ void put(T (&a)[N], int i, T v) {
#pragma unroll
  for (int k = 0; k < N; ++k)
    if (i == k) a[k] = v;
}

// The reference _hungarian_max (mapping.py:71-122) on an N x N block held in
// registers (N = fused group <= 8).  Returns perm[row] = column.
template <int N>
__host__ __device__ __forceinline__ void hungarian_small(const double (&w)[N][N], int (&perm)[N]) {
  double u[N + 1], v[N + 1], minv[N + 1];
  int match[N + 1], way[N + 1];
  bool used[N + 1];
#pragma unroll
  for (int j = 0; j <= N; ++j) {
    u[j] = 0.0;
    v[j] = 0.0;
    match[j] = 0;
    way[j] = 0;
  }
  for (int i = 1; i <= N; ++i) {
    match[0] = i;
    int j0 = 0;
#pragma unroll
    for (int j = 0; j <= N; ++j) {
      minv[j] = kInf;
      used[j] = false;
    }
    while (true) {
      put(used, j0, true);
      const int i0 = sel(match, j0);
      const double ui0 = sel(u, i0);
      double crow[N];
#pragma unroll
      for (int j = 0; j < N; ++j) {
        double x = w[0][j];
#pragma unroll
        for (int k = 1; k < N; ++k)
          if (i0 - 1 == k) x = w[k][j];
        crow[j] = -x;
      }
      double delta = kInf;
      int j1 = 0;
#pragma unroll
      for (int j = 1; j <= N; ++j) {
        if (!used[j]) {
          const double cur = (crow[j - 1] - ui0) - v[j];
          if (cur < minv[j]) {
            minv[j] = cur;
            way[j] = j0;
          }
          if (minv[j] < delta) {
            delta = minv[j];
            j1 = j;
          }
        }
      }
#pragma unroll
      for (int j = 0; j <= N; ++j) {
        if (used[j]) {
          const int r = match[j];
#pragma unroll
          for (int k = 0; k <= N; ++k)
            if (k == r) u[k] += delta;
          v[j] -= delta;
        } else {
          minv[j] -= delta;
        }
      }
      j0 = j1;
      if (sel(match, j0) == 0) break;
    }
    while (j0) {
      const int j1 = sel(way, j0);
      put(match, j0, sel(match, j1));
      j0 = j1;
    }
  }
#pragma unroll
  for (int j = 1; j <= N; ++j) put(perm, match[j] - 1, j - 1);
}

// ---------------------------------------------------------------------------
// K1: dense weights, two adjacent columns per thread (16-B stores)

constexpr int kW_TPB = 256;
constexpr int kW_MAXC = 2048;  // columns decoded once into a shared table
constexpr int kW_RPB = 64;     // rows per block (amortises the tables below)
constexpr int kW_SEGS = 128;   // segments of a block's rows staged in shared memory
constexpr int kW_MAXPM = 16;   // stages / shards with per-segment overlap tables

// One block per (plan, 64 rows).  The overlap of segment s with column
// c = (d, st, m) factorises (domain.py:299-320): |layers(s) & stage(st)| *
// unit(s) depends on the stage only, |[a,b) & shard(m)| on the shard only, and
// the pipeline test on d only.  So the block builds, once, a column table
// (st, m, d), and per staged segment the P stage products A[s][st] (int64)
// and M shard overlaps B[s][m]; an entry is then sum_s [pipe ok] A * B -- a
// few shared loads and one 64-bit multiply-add per segment -- converted once;
// each thread writes 4 adjacent columns (two 16-byte stores).  Plans beyond
// the tables' sizes (or general-range plans) take the per-entry path.
__global__ void __launch_bounds__(kW_TPB) k_weights(const sk_plan* __restrict__ plans,
                                                    const int32_t* __restrict__ row_ptr,
                                                    const sk_segment* __restrict__ segs,
                                                    double* __restrict__ W) {
  __shared__ int2 ctab[kW_MAXC];
  __shared__ unsigned long long sA[kW_SEGS][kW_MAXPM];
  __shared__ __align__(16) unsigned sB[kW_SEGS][kW_MAXPM];
  __shared__ int sPipe[kW_SEGS];
  __shared__ int s_rp[kW_RPB + 1];
  const sk_plan p = plans[blockIdx.y];
  const int r0 = blockIdx.x * kW_RPB;
  if (r0 >= p.rows) return;
  const int r1 = min(p.rows, r0 + kW_RPB), nr = r1 - r0;
  const int C = p.D * p.P * p.M;
  if (threadIdx.x <= nr) s_rp[threadIdx.x] = row_ptr[p.row_base + r0 + threadIdx.x];
  __syncthreads();
  const int sb = s_rp[0], nseg = s_rp[nr] - sb;
  if ((p.flags & SK_PLAN_GENERIC) || C > kW_MAXC || p.P > kW_MAXPM || p.M > kW_MAXPM || nseg > kW_SEGS) {
    // block-uniform: per-entry path
    const bool gen = (p.flags & SK_PLAN_GENERIC) != 0;
    for (long long e = threadIdx.x; e < (long long)nr * C; e += kW_TPB) {
      const int r = r0 + (int)(e / C), c = (int)(e % C);
      W[p.f_off + (long long)r * C + c] = gen ? weight_generic(p, row_ptr, segs, r, c)
                                              : weight_at(p, row_ptr, segs, r, c);
    }
    return;
  }
  for (int c = threadIdx.x; c < C; c += kW_TPB) {
    const int m = c % p.M, t = c / p.M;
    ctab[c] = make_int2((t % p.P) | (m << 16), t / p.P + 1);
  }
  const int q = p.L / p.P, rem = p.L % p.P, w = p.K / p.M;
  // (segment, stage) and (segment, shard) tables: thread = (k, x) over a
  // kW_MAXPM-wide grid, so no division per item
  for (int t = threadIdx.x; t < nseg * kW_MAXPM; t += kW_TPB) {
    const int k = t / kW_MAXPM, x = t % kW_MAXPM;
    const sk_segment sg = segs[sb + k];
    if (x < p.P) {
      const int s0 = x * q + min(x, rem), s1 = s0 + q + (x < rem ? 1 : 0);
      const int ol = min(sg.l1, s1) - max(sg.l0, s0);
      sA[k][x] = ol > 0 ? (unsigned long long)ol * (unsigned long long)sg.unit : 0ull;
    }
    if (x < p.M) {
      const int oi = min(sg.b, x * w + w) - max(sg.a, x * w);
      sB[k][x] = oi > 0 ? (unsigned)oi : 0u;
    }
    if (x == 0) sPipe[k] = sg.pipe;
  }
  __syncthreads();
  // N / K: the exact reciprocal product when K is a power of two (bit-identical
  // to the correctly rounded division), else the IEEE division
  const bool pow2 = (p.K & (p.K - 1)) == 0;
  const double inv = 1.0 / (double)p.K;
  constexpr int CPT = 4;  // columns per work item
  const int ipr = (C + CPT - 1) / CPT;  // items per row
  const float inv_ipr = 1.0f / (float)ipr;
  for (int e = threadIdx.x; e < nr * ipr; e += kW_TPB) {
    // (row, item) = divmod(e, ipr), exact for e < 2^24
    int rr = (int)((float)e * inv_ipr);
    int it = e - rr * ipr;
    rr = it < 0 ? rr - 1 : (it >= ipr ? rr + 1 : rr);
    it = it < 0 ? it + ipr : (it >= ipr ? it - ipr : it);
    const int c0 = CPT * it;
    unsigned long long nu[CPT];
#pragma unroll
    for (int u = 0; u < CPT; ++u) nu[u] = 0;
    if ((p.M & 3) == 0) {
      // the item's 4 columns share (d, stage) and take 4 consecutive shards:
      // per segment one stage product, one 16-byte load of shard overlaps
      const int2 t = ctab[c0];
      const int st = t.x & 0xffff, m0 = t.x >> 16, d = t.y;
      for (int k = s_rp[rr] - sb; k < s_rp[rr + 1] - sb; ++k) {
        const int pipe = sPipe[k];
        if (pipe != 0 && pipe != d) continue;
        const unsigned long long a = sA[k][st];
        const uint4 b = *reinterpret_cast<const uint4*>(&sB[k][m0]);
        nu[0] += a * b.x;
        nu[1] += a * b.y;
        nu[2] += a * b.z;
        nu[3] += a * b.w;
      }
    } else {
      int st[CPT], mm[CPT], dd[CPT];
#pragma unroll
      for (int u = 0; u < CPT; ++u) {
        const int2 t = ctab[min(c0 + u, C - 1)];
        st[u] = t.x & 0xffff;
        mm[u] = t.x >> 16;
        dd[u] = t.y;
      }
      for (int k = s_rp[rr] - sb; k < s_rp[rr + 1] - sb; ++k) {
        const int pipe = sPipe[k];
#pragma unroll
        for (int u = 0; u < CPT; ++u)
          if (pipe == 0 || pipe == dd[u]) nu[u] += sA[k][st[u]] * (unsigned long long)sB[k][mm[u]];
      }
    }
    double wv[CPT];
#pragma unroll
    for (int u = 0; u < CPT; ++u) wv[u] = pow2 ? __ull2double_rn(nu[u]) * inv : num_to_w((long long)nu[u], p.K);
    double* out = W + p.f_off + (long long)(r0 + rr) * C + c0;
    if (c0 + CPT <= C && ((reinterpret_cast<uintptr_t>(out) & 15) == 0)) {
      reinterpret_cast<double2*>(out)[0] = make_double2(wv[0], wv[1]);
      reinterpret_cast<double2*>(out)[1] = make_double2(wv[2], wv[3]);
    } else {
#pragma unroll
      for (int u = 0; u < CPT; ++u)
        if (c0 + u < C) out[u] = wv[u];
    }
  }
}

// ---------------------------------------------------------------------------
// K2a: per fused pair (a, b): g x g block -> inner KM -> fused weight + perm


// One fused pair's block result: fused weight and packed inner permutation.
struct FusedBlock {
  double f;
  uint32_t packed;
  bool nz;  // false: all-zero block (the row's zero fill already holds it)
};

// Block of row group a x fused slot decoded by c0, counting the model
// segments (pipe 0) and the cache segments of new pipeline `dsel` (0: model
// only).  With dsel = c0.d this is exactly the reference's block.
template <int G>
__device__ __forceinline__ FusedBlock fuse_block(const sk_plan& p, int a, const Col c0, int dsel,
                                                 const int32_t* __restrict__ row_ptr,
                                                 const sk_segment* __restrict__ segs) {
  // the G columns of fused slot b share (pipeline, stage): c0 is their decode
  const int wdt = c0.i1 - c0.i0;
  long long num[G][G];
  long long any = 0;
#pragma unroll
  for (int k = 0; k < G; ++k) {
    const int r = a * G + k;
    const int s0 = row_ptr[p.row_base + r], s1 = row_ptr[p.row_base + r + 1];
#pragma unroll
    for (int l = 0; l < G; ++l) num[k][l] = 0;
    for (int s = s0; s < s1; ++s) {
      const sk_segment sg = segs[s];
      const int ol = min(sg.l1, c0.s1) - max(sg.l0, c0.s0);
      if (ol <= 0 || (sg.pipe != 0 && sg.pipe != dsel)) continue;
      const long long per = (long long)ol * sg.unit;
#pragma unroll
      for (int l = 0; l < G; ++l) {
        const int oi = min(sg.b, c0.i0 + (l + 1) * wdt) - max(sg.a, c0.i0 + l * wdt);
        if (oi > 0) num[k][l] += per * oi;
      }
    }
#pragma unroll
    for (int l = 0; l < G; ++l) any |= num[k][l];
  }
  FusedBlock out;
  out.f = 0.0;
  out.packed = 0;
  out.nz = any != 0;
  // all-zero block: max / builtin sum of zeros are 0.0 and the inner KM's
  // answer is the (replayed) zero-matrix permutation -- exactly what the
  // row's zero fill already encodes (F = 0.0, perm stored XOR zero_perm)
  if (!out.nz) return out;
  // N / K: exact reciprocal multiply when K is a power of two (bit-identical
  // to the correctly rounded division), else the IEEE division
  const bool pow2 = (p.K & (p.K - 1)) == 0;
  const double inv = 1.0 / (double)p.K;
  double w[G][G];
#pragma unroll
  for (int k = 0; k < G; ++k)
#pragma unroll
    for (int l = 0; l < G; ++l)
      w[k][l] = pow2 ? __ll2double_rn(num[k][l]) * inv : num_to_w(num[k][l], p.K);
  if (G == 1) {
    out.f = w[0][0];  // max([w]) == sum([w]) == w for w >= 0
    return out;
  }
  int pm[G];
  // permutation-pattern block (exactly one positive weight per row and per
  // column): the replayed KM matches every row to its positive column in a
  // single Dijkstra step (the only negative reduced cost; no potential of a
  // real column ever changes), so the answer is that permutation
  bool is_perm = true;
  unsigned colmask = 0;
#pragma unroll
  for (int k = 0; k < G; ++k) {
    int cnt = 0, at = 0;
#pragma unroll
    for (int l = 0; l < G; ++l)
      if (num[k][l] != 0) {
        ++cnt;
        at = l;
      }
    is_perm = is_perm && cnt == 1 && !((colmask >> at) & 1u);
    colmask |= 1u << at;
    pm[k] = at;
  }
  if (!is_perm) hungarian_small<G>(w, pm);
  double picked[G];
#pragma unroll
  for (int k = 0; k < G; ++k) picked[k] = sel(w[k], pm[k]);
  double f;
  if (p.flags & SK_PLAN_FUSED_SUM) {
    f = py_builtin_sum<G>(picked);
  } else {
    f = picked[0];
#pragma unroll
    for (int k = 1; k < G; ++k)
      if (picked[k] > f) f = picked[k];
  }
  uint32_t packed = 0;
#pragma unroll
  for (int k = 0; k < G; ++k) packed |= (uint32_t)pm[k] << (4 * k);
  out.f = f;
  out.packed = packed;
  return out;
}

// dictionary coding of fused values: 256 one-byte codes per plan; code 0 is
// +0.0 (the zero fill); kEmpty marks a free slot
constexpr int kDictSlots = 256;
constexpr unsigned long long kEmpty = ~0ull;  // a NaN pattern: never a weight

// k_fuse's code output (CODES mode): per class-local plan q the zero-padded
// n x n code matrix at codes + q * stride + 16 (k_outer's global-code layout)
// and the 256-slot dictionary at dict + q * 256 (slot 0: overflow flag, kEmpty
// while the plan's values fit)
struct FuseCodes {
  unsigned char* codes;
  size_t stride;
  unsigned long long* dict;
};

// the code of fused value f in the plan's dictionary: open addressing over
// slots 1..255 of the global table (write-once slots, claimed by CAS), with a
// per-CTA shared-memory mirror so repeated values cost one shared load (the
// probe that misses the mirror is out of line)
__device__ __noinline__ unsigned fuse_code_slow(unsigned long long x, unsigned h, unsigned long long* s_dict,
                                                unsigned long long* g_dict) {
  volatile unsigned long long* sd = s_dict;
  for (int tries = 0; tries < kDictSlots; ++tries, h = (h + 1) & (kDictSlots - 1)) {
    if (h == 0) continue;
    unsigned long long c = sd[h];
    if (c == kEmpty) c = __ldcg(g_dict + h);  // usually claimed by another CTA already
    if (c == kEmpty) {
      c = atomicCAS(g_dict + h, kEmpty, x);
      if (c == kEmpty) c = x;
    }
    sd[h] = c;
    if (c == x) return h;
  }
  g_dict[0] = 0ull;  // overflow: the plan takes the uncoded path
  return 0;
}

__device__ __forceinline__ unsigned char fuse_code(double f, unsigned long long* s_dict,
                                                   unsigned long long* g_dict) {
  const unsigned long long x = (unsigned long long)__double_as_longlong(f);
  if (x == 0ull) return 0;
  const unsigned h = (unsigned)((x * 0x9E3779B97F4A7C15ull) >> 56);
  if (h != 0 && *reinterpret_cast<volatile unsigned long long*>(s_dict + h) == x) return (unsigned char)h;
  return (unsigned char)fuse_code_slow(x, h, s_dict, g_dict);
}

// One lane group (LPG lanes) per fused GPU group a.  The group first writes
// its whole fused row as zeros (F = 0.0, perm = 0 meaning "zero-matrix
// permutation"; coalesced full sectors, no separate clear and no partial-
// sector fills), then visits only pairs (a, b) that CAN be non-zero: the
// lanes reduce the group's layer span [L0, L1) over its segments, and per new
// pipeline d only the fused slots of stages overlapping that span are
// candidates (a contiguous run of b).  Every other block is all-zero by
// construction.
//
// A block depends on the new pipeline d only through the cache segments
// tagged with d, so the lanes also reduce the set of pipelines the group's
// cache segments name (a 128-bit mask).  The group's work items are then the
// model-only block of each slot offset -- stored for every pipeline the mask
// does not name -- and the full block of each (named pipeline, offset): the
// same numbers give the same inner KM, so the reuse is exact, and a group
// builds span * (1 + named pipelines) blocks instead of D * span.
// 3 warps per CTA: at 112 registers a warp takes 3.5 K registers, so the SM
// holds 18 warps as six 3-warp CTAs but only 16 as four 4-warp CTAs
// (measured: k_fuse 8.70 -> 8.50 ms per step; 32/64/128/160/192/256 slower)
#ifndef SK_F_TPB
#define SK_F_TPB 96
#endif
constexpr int kF_TPB = SK_F_TPB;
constexpr int kF_WARPS = kF_TPB / 32;
constexpr int kF_MAXD = 128;  // pipelines tracked by the cache-pipeline mask

__device__ __forceinline__ int stage_of(int x, int L, int P) {
  const int q = L / P, r = L % P;
  return x < r * (q + 1) ? x / (q + 1) : r + (x - r * (q + 1)) / q;
}

template <int G, int LPG, bool CODES>
__device__ __forceinline__ void fuse_rows(const sk_plan& p, int q, int bx,
                                          const int32_t* __restrict__ row_ptr,
                                          const sk_segment* __restrict__ segs,
                                          double* __restrict__ F, uint32_t* __restrict__ perm,
                                          uint32_t zero_perm, const FuseCodes& fc,
                                          unsigned long long* s_dict) {
  // LPG lanes per GPU group: small targets have few candidate slots per group
  const int nA = p.rows / G;
  const int nB = (p.D * p.P * p.M) / G;
  const int n = nA > nB ? nA : nB;
  const int lane = threadIdx.x & 31, sub = lane % LPG;
  const int a = (bx * kF_WARPS + (threadIdx.x >> 5)) * (32 / LPG) + lane / LPG;
  const bool live = a < nA;
  int lo = 0x7fffffff, hi = -1;
  unsigned long long pm0 = 0, pm1 = 0;  // cache pipelines 1..128 named by the group
  bool pm_over = false;
  if (live) {
    const int s_begin = row_ptr[p.row_base + a * G], s_end = row_ptr[p.row_base + a * G + G];
    for (int s = s_begin + sub; s < s_end; s += LPG) {
      const sk_segment sg = segs[s];
      if (sg.l1 > sg.l0 && sg.b > sg.a && sg.unit != 0) {
        lo = min(lo, sg.l0);
        hi = max(hi, sg.l1);
        // cache segments of pipelines outside 1..D match no column
        // (seg_num compares pipe with the column's d <= D): not named
        if (sg.pipe != 0 && sg.pipe <= p.D) {
          const int q = sg.pipe - 1;
          if (q < 64)
            pm0 |= 1ull << q;
          else if (q < kF_MAXD)
            pm1 |= 1ull << (q - 64);
          else
            pm_over = true;
        }
      }
    }
  }
#pragma unroll
  for (int off = LPG / 2; off; off >>= 1) {
    lo = min(lo, __shfl_xor_sync(kFull, lo, off));
    hi = max(hi, __shfl_xor_sync(kFull, hi, off));
    pm0 |= __shfl_xor_sync(kFull, pm0, off);
    pm1 |= __shfl_xor_sync(kFull, pm1, off);
  }
  pm_over = __any_sync(kFull, pm_over);
  lo = max(lo, 0);
  hi = min(hi, p.L);
  // the groups write their whole fused rows: zeros first (the encoding of an
  // all-zero block), then the candidate blocks.  A warp's groups own
  // consecutive rows, i.e. one contiguous span of F and of perm: the 32 lanes
  // zero it together with 16-byte stores (scalar head/tail to alignment)
  const long long row0 = p.f_off + (long long)a * nB;
  // CODES: the plan's zero-padded n x n one-byte code matrix (k_outer's layout)
  unsigned char* const crow = CODES ? fc.codes + (size_t)q * fc.stride + 16 + (size_t)a * n : nullptr;
  {
    const int a_first = a - lane / LPG;
    const int rows_live = max(0, min(32 / LPG, nA - a_first));
    const long long s0 = p.f_off + (long long)a_first * nB, cnt = (long long)rows_live * nB;
    if (CODES) {
      // code 0 (+0.0) over the warp's rows of the n x n matrix, padding rows
      // nA..n-1 and columns nB..n-1 included
      const int crows = max(0, min(32 / LPG, n - a_first));
      unsigned char* c0p = fc.codes + (size_t)q * fc.stride + 16 + (size_t)a_first * n;
      const long long ccnt = (long long)crows * n;
      const long long ch = min(ccnt, (long long)((16 - (reinterpret_cast<uintptr_t>(c0p) & 15)) & 15));
      if (lane < ch) c0p[lane] = 0;
      const long long cv = (ccnt - ch) >> 4;
      uint4* C4 = reinterpret_cast<uint4*>(c0p + ch);
      for (long long v = lane; v < cv; v += 32) C4[v] = make_uint4(0u, 0u, 0u, 0u);
      const long long ct0 = ch + (cv << 4);
      if (lane < ccnt - ct0) c0p[ct0 + lane] = 0;
    } else {
      // F: doubles, 2 per 16 bytes
      const long long fh = min(cnt, (long long)(s0 & 1));
      if (lane < fh) F[s0 + lane] = 0.0;
      const long long fv = (cnt - fh) >> 1;
      double2* F2 = reinterpret_cast<double2*>(F + s0 + fh);
      for (long long v = lane; v < fv; v += 32) F2[v] = make_double2(0.0, 0.0);
      if (lane == 0 && ((cnt - fh) & 1)) F[s0 + cnt - 1] = 0.0;
    }
    // perm: uint32, 4 per 16 bytes
    const long long ph = min(cnt, (long long)((4 - (s0 & 3)) & 3));
    if (lane < ph) perm[s0 + lane] = 0u;
    const long long pv = (cnt - ph) >> 2;
    uint4* P4 = reinterpret_cast<uint4*>(perm + s0 + ph);
    for (long long v = lane; v < pv; v += 32) P4[v] = make_uint4(0u, 0u, 0u, 0u);
    const long long pt0 = ph + (pv << 2);
    if (lane < cnt - pt0) perm[s0 + pt0 + lane] = 0u;
  }
  __syncwarp();
  if (!live || lo >= hi) return;  // the whole row group is zero
  const int p_lo = stage_of(lo, p.L, p.P), p_hi = stage_of(hi - 1, p.L, p.P);
  const int span = ((p_hi + 1 - p_lo) * p.M) / G;  // fused slots per pipeline
  const int per_d = (p.P * p.M) / G;
  const int b0 = (p_lo * p.M) / G;
  if (pm_over) {
    // more pipelines than the mask tracks: every candidate block in full
    const int total = p.D * span;
    for (int t = sub; t < total; t += LPG) {
      const int d = t / span;
      const int b = d * per_d + b0 + (t - d * span);
      const Col c0 = col_of(p, b * G);
      const FusedBlock r = fuse_block<G>(p, a, c0, c0.d, row_ptr, segs);
      if (r.nz) {
        const long long idx = p.f_off + (long long)a * nB + b;
        if (CODES)
          crow[b] = fuse_code(r.f, s_dict, fc.dict + (size_t)q * kDictSlots);
        else
          F[idx] = r.f;
        perm[idx] = r.packed ^ zero_perm;
      }
    }
    return;
  }
  // work items: the model-only block of every slot offset (stored for every
  // pipeline the group's cache does not name), then the full block of every
  // (named pipeline, offset)
  const int nbits = __popcll(pm0) + __popcll(pm1);
  const int n_items = span * (1 + nbits);
  for (int it = sub; it < n_items; it += LPG) {
    int o = it, dq = -1;  // dq: 0-based named pipeline, -1 = model only
    if (it >= span) {
      const int k = (it - span) / span;
      o = it - span - k * span;
      // k-th set bit of the mask
      unsigned long long m = pm0;
      int base = 0, kk = k;
      if (kk >= __popcll(pm0)) {
        kk -= __popcll(pm0);
        m = pm1;
        base = 64;
      }
      for (int z = 0; z < kk; ++z) m &= m - 1;
      dq = base + __ffsll(m) - 1;
    }
    const int bq = (dq < 0 ? 0 : dq) * per_d + b0 + o;
    const FusedBlock r = fuse_block<G>(p, a, col_of(p, bq * G), dq + 1, row_ptr, segs);
    if (!r.nz) continue;
    const uint32_t pk = r.packed ^ zero_perm;
    unsigned char code = 0;
    if (CODES) code = fuse_code(r.f, s_dict, fc.dict + (size_t)q * kDictSlots);
    if (dq >= 0) {
      if (CODES)
        crow[bq] = code;
      else
        F[row0 + bq] = r.f;
      perm[row0 + bq] = pk;
    } else {
      for (int d = 0; d < p.D; ++d) {
        const bool named = d < 64 ? ((pm0 >> d) & 1ull) : d < kF_MAXD ? ((pm1 >> (d - 64)) & 1ull) : false;
        if (named) continue;
        const int b = d * per_d + b0 + o;
        if (CODES)
          crow[b] = code;
        else
          F[row0 + b] = r.f;
        perm[row0 + b] = pk;
      }
    }
  }
}

#ifndef SK_FF_MINB
#define SK_FF_MINB 0  // 0: unspecified (an explicit 1 costs k_fuse 20%: measured 7.61 -> 9.34 ms)
#endif
#ifndef SK_FC_MINB
#define SK_FC_MINB 6
#endif
template <int G, int LPG, bool CODES>
__global__ void __launch_bounds__(kF_TPB, CODES && G <= 4 ? SK_FC_MINB : SK_FF_MINB) k_fuse(const sk_plan* __restrict__ plans, int plan0,
                                                 const int32_t* __restrict__ row_ptr,
                                                 const sk_segment* __restrict__ segs,
                                                 double* __restrict__ F, uint32_t* __restrict__ perm,
                                                 uint32_t zero_perm, const FuseCodes fc) {
  const int q = plan0 + blockIdx.y;
  const sk_plan p = plans[q];
  if (p.group != G || (p.flags & SK_PLAN_GENERIC)) return;
  __shared__ unsigned long long s_dict[CODES ? kDictSlots : 1];
  if (CODES) {
    for (int t = threadIdx.x; t < kDictSlots; t += kF_TPB) s_dict[t] = kEmpty;
    __syncthreads();
  }
  fuse_rows<G, LPG, CODES>(p, q, blockIdx.x, row_ptr, segs, F, perm, zero_perm, fc, s_dict);
}

// After a CODES pass: the plans whose fused values overflowed the 255-entry
// dictionary (its slot 0 set) are listed, then get their fused rows as
// doubles for the outer KM's uncoded path -- work units (listed plan, row
// block) spread over a fixed grid, so a few big overflowed plans do not
// serialise on a few CTAs.
__global__ void k_overflow_list(const unsigned long long* __restrict__ dict, int n_plans, int* list,
                                int* count) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q < n_plans && __ldcg(dict + (size_t)q * kDictSlots) != kEmpty) list[atomicAdd(count, 1)] = q;
}

constexpr int kF_MAXBX = (4095 + kF_WARPS * 8 - 1) / (kF_WARPS * 8);  // row blocks of a plan (LPG 4)

template <int G>
__global__ void __launch_bounds__(kF_TPB) k_fuse_overflow(const sk_plan* __restrict__ plans,
                                                          const int* __restrict__ list,
                                                          const int* __restrict__ count,
                                                          const int32_t* __restrict__ row_ptr,
                                                          const sk_segment* __restrict__ segs,
                                                          double* __restrict__ F, uint32_t* __restrict__ perm,
                                                          uint32_t zero_perm, const FuseCodes fc) {
  constexpr int kGroupsPerBlock = kF_WARPS * (32 / 4);
  const long long units = (long long)__ldcg(count) * kF_MAXBX;
  for (long long u = blockIdx.x; u < units; u += gridDim.x) {
    const int q = list[u / kF_MAXBX], bx = (int)(u % kF_MAXBX);
    const sk_plan p = plans[q];
    if (p.group != G || (p.flags & SK_PLAN_GENERIC)) continue;
    if (bx * kGroupsPerBlock >= p.rows / G) continue;
    fuse_rows<G, 4, false>(p, q, bx, row_ptr, segs, F, perm, zero_perm, fc, nullptr);
  }
}

// The inner KM's answer on an all-zero g x g block, replayed once on the host
// with the same code the device runs (a constant of the algorithm).
template <int G>
uint32_t zero_block_perm() {
  double z[G][G];
  for (int k = 0; k < G; ++k)
    for (int l = 0; l < G; ++l) z[k][l] = 0.0;
  int pm[G];
  hungarian_small<G>(z, pm);
  uint32_t packed = 0;
  for (int k = 0; k < G; ++k) packed |= (uint32_t)pm[k] << (4 * k);
  return packed;
}

uint32_t zero_perm_of(int g) {
  switch (g) {
    case 2: { static const uint32_t z = zero_block_perm<2>(); return z; }
    case 3: { static const uint32_t z = zero_block_perm<3>(); return z; }
    case 4: { static const uint32_t z = zero_block_perm<4>(); return z; }
    case 5: { static const uint32_t z = zero_block_perm<5>(); return z; }
    case 6: { static const uint32_t z = zero_block_perm<6>(); return z; }
    case 7: { static const uint32_t z = zero_block_perm<7>(); return z; }
    case 8: { static const uint32_t z = zero_block_perm<8>(); return z; }
    default: return 0u;
  }
}

template <int G>
int launch_fuse(const sk_plan* d_plans, int p0, int np, int max_na, int max_nb, const int32_t* row_ptr,
                const sk_segment* segs, double* F, uint32_t* perm, cudaStream_t s) {
  // lanes per GPU group ~ the candidate slots a group typically has
  // a group has ~span * (1 + cache pipelines) blocks to build, whatever nB
  static const int env_lpg = [] {
    const char* e = getenv("SK_FUSE_LPG");
    return e ? atoi(e) : 0;
  }();
  const int lpg = env_lpg ? env_lpg : 4;
  const int groups_per_block = kF_WARPS * (32 / lpg);
  dim3 grid((max_na + groups_per_block - 1) / groups_per_block, np);
  const uint32_t zp = zero_perm_of(G);
  if (lpg == 2)
    k_fuse<G, 2, false><<<grid, kF_TPB, 0, s>>>(d_plans, p0, row_ptr, segs, F, perm, zp, FuseCodes{});
  else if (lpg == 4)
    k_fuse<G, 4, false><<<grid, kF_TPB, 0, s>>>(d_plans, p0, row_ptr, segs, F, perm, zp, FuseCodes{});
  else if (lpg == 8)
    k_fuse<G, 8, false><<<grid, kF_TPB, 0, s>>>(d_plans, p0, row_ptr, segs, F, perm, zp, FuseCodes{});
  else if (lpg == 16)
    k_fuse<G, 16, false><<<grid, kF_TPB, 0, s>>>(d_plans, p0, row_ptr, segs, F, perm, zp, FuseCodes{});
  else
    k_fuse<G, 32, false><<<grid, kF_TPB, 0, s>>>(d_plans, p0, row_ptr, segs, F, perm, zp, FuseCodes{});
  return cuda_check("k_fuse launch");
}

template <int G>
int launch_fuse_coded(const sk_plan* d_plans, int p0, int np, int max_n, const int32_t* row_ptr,
                      const sk_segment* segs, uint32_t* perm, const FuseCodes& fc, cudaStream_t s) {
  constexpr int kGroupsPerBlock = kF_WARPS * (32 / 4);
  dim3 grid((max_n + kGroupsPerBlock - 1) / kGroupsPerBlock, np);
  k_fuse<G, 4, true><<<grid, kF_TPB, 0, s>>>(d_plans, p0, row_ptr, segs, nullptr, perm, zero_perm_of(G), fc);
  return cuda_check("k_fuse (coded) launch");
}

template <int G>
int launch_fuse_overflow(const sk_plan* d_plans, const int* list, const int* count, const int32_t* row_ptr,
                         const sk_segment* segs, double* F, uint32_t* perm, const FuseCodes& fc,
                         cudaStream_t s) {
  k_fuse_overflow<G><<<148 * 4, kF_TPB, 0, s>>>(d_plans, list, count, row_ptr, segs, F, perm, zero_perm_of(G), fc);
  return cuda_check("k_fuse_overflow launch");
}

// ---------------------------------------------------------------------------
// K2a for general-range plans (SK_PLAN_GENERIC: fused groups up to 32,
// 128-bit numerators, 64-bit K).  One warp per fused pair (a, b): the g x g
// block is built in shared memory (lane l = block column l) and the
// reference's _hungarian_max (mapping.py:71-122) runs with lane j - 1 owning
// column j: per Dijkstra step every unused column updates its own slack and
// predecessor, the warp argmin picks the lowest column among equal minima
// (mapping.py:103-105), and the potential update touches distinct rows.
// The fused weight goes to F; the matched weights and the permutation go to
// the plan's side area (sk_fused_elems) for the outer KM's expansion.

constexpr int kG_WARPS = 4;
constexpr int kG_MAX = 32;

__device__ __forceinline__ unsigned long long order_key_g(double x) {
  unsigned long long b = (unsigned long long)__double_as_longlong(x);
  if ((b << 1) == 0ull) b = 0ull;  // -0.0 ties with +0.0, as under '<'
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__global__ void __launch_bounds__(32 * kG_WARPS) k_fuse_generic(const sk_plan* __restrict__ plans, int plan0,
                                                                const int32_t* __restrict__ row_ptr,
                                                                const sk_segment* __restrict__ segs,
                                                                double* __restrict__ F) {
  __shared__ double s_w[kG_WARPS][kG_MAX][kG_MAX + 1];
  __shared__ double s_u[kG_WARPS][kG_MAX + 1];
  __shared__ int s_match[kG_WARPS][kG_MAX + 1];
  __shared__ int s_way[kG_WARPS][kG_MAX + 1];
  __shared__ int s_perm[kG_WARPS][kG_MAX];
  const sk_plan p = plans[plan0 + blockIdx.y];
  if (!(p.flags & SK_PLAN_GENERIC)) return;
  const int g = p.group;
  const int nA = p.rows / g, nB = (p.D * p.P * p.M) / g;
  const int wi = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long pair = (long long)blockIdx.x * kG_WARPS + wi;
  if (pair >= (long long)nA * nB) return;  // warp-uniform
  const int a = (int)(pair / nB), b = (int)(pair % nB);
  double(*w)[kG_MAX + 1] = s_w[wi];
  double* u = s_u[wi];
  int* match = s_match[wi];
  int* way = s_way[wi];
  const bool col_on = lane < g;  // column j = lane + 1
  if (col_on) {
    const ColW c = col_of_w(p, b * g + lane);
    for (int k = 0; k < g; ++k) {
      const int r = a * g + k;
      i128 acc = 0;
      for (int s = row_ptr[p.row_base + r]; s < row_ptr[p.row_base + r + 1]; s += 2)
        acc += seg_num_wide(wide_at(segs, s), c);
      w[k][lane] = sk_exact::rat_to_double(acc, p.Kw);
    }
  }
  if (lane <= g) {
    u[lane] = 0.0;
    match[lane] = 0;
  }
  __syncwarp();
  double v = 0.0, minv = kInf;
  int wr = 0;
  for (int i = 1; i <= g; ++i) {
    if (lane == 0) match[0] = i;
    __syncwarp();
    bool used = false;
    minv = kInf;
    int j0 = 0;
    while (true) {
      const int i0 = match[j0];
      const double ui0 = u[i0];
      const bool on = col_on && !used;
      if (on) {
        const double cur = (-w[i0 - 1][lane] - ui0) - v;
        if (cur < minv) {
          minv = cur;
          wr = j0;
        }
      }
      const unsigned long long key = on ? order_key_g(minv) : ~0ull;
      const unsigned hi = __reduce_min_sync(kFull, (unsigned)(key >> 32));
      const bool c1 = (unsigned)(key >> 32) == hi;
      const unsigned lo = __reduce_min_sync(kFull, c1 ? (unsigned)key : 0xffffffffu);
      const bool c2 = c1 && (unsigned)key == lo;
      const unsigned jw = __reduce_min_sync(kFull, c2 && on ? (unsigned)(lane + 1) : 0xffffffffu);
      const double delta = __shfl_sync(kFull, minv, (int)(jw - 1) & 31);
      // u[match[j]] += delta, v[j] -= delta for used j (incl. column 0);
      // minv[j] -= delta otherwise
      if (lane == 0) u[match[0]] += delta;
      if (col_on && used) {
        u[match[lane + 1]] += delta;
        v -= delta;
      } else if (col_on) {
        minv -= delta;
      }
      __syncwarp();
      j0 = (int)jw;
      if (lane + 1 == j0) used = true;
      if (match[j0] == 0) break;
    }
    if (col_on) way[lane + 1] = wr;
    __syncwarp();
    if (lane == 0) {
      while (j0) {
        const int j1 = way[j0];
        match[j0] = match[j1];
        j0 = j1;
      }
    }
    __syncwarp();
  }
  if (col_on) s_perm[wi][match[lane + 1] - 1] = lane;
  __syncwarp();
  const long long nAB = (long long)nA * nB;
  double* side_w = F + p.f_off + nAB;
  unsigned char* side_p = reinterpret_cast<unsigned char*>(F + p.f_off + nAB * (1 + g));
  if (col_on) {
    side_w[pair * g + lane] = w[lane][s_perm[wi][lane]];
    side_p[pair * g + lane] = (unsigned char)s_perm[wi][lane];
  }
  if (lane == 0) {
    double f;
    if (p.flags & SK_PLAN_FUSED_SUM) {
      // CPython >= 3.12 builtin sum (see py_builtin_sum)
      f = 0.0 + w[0][s_perm[wi][0]];
      double c = 0.0;
      for (int k = 1; k < g; ++k) {
        const double xi = w[k][s_perm[wi][k]];
        const double t = f + xi;
        if (fabs(f) >= fabs(xi))
          c += (f - t) + xi;
        else
          c += (xi - t) + f;
        f = t;
      }
      if (c != 0.0 && isfinite(c)) f += c;
    } else {
      f = w[0][s_perm[wi][0]];
      for (int k = 1; k < g; ++k) {
        const double x = w[k][s_perm[wi][k]];
        if (x > f) f = x;
      }
    }
    F[p.f_off + pair] = f;
  }
}

// ---------------------------------------------------------------------------
// K2b: outer KM, one warp per plan.
//
// Column j (1..n) is owned by thread (j - 1) % T, slot k = (j - 1) / T (T =
// threads per plan); the reference's virtual column 0 has no slot (it is
// always used; only its row potential, ucol[0], is ever read).  The owner
// keeps the column's slack minv[j], potential v[j], predecessor way[j] and
// used bit in registers.  Row potentials are kept per COLUMN (ucol[j] = u[match[j]],
// shared memory): the reference only ever reads u[i0] with i0 = match[j0]
// and adds delta to u[match[j]] for used j, so indexing by column removes the
// match[] indirection from the step's critical path; the augmenting walk
// moves ucol together with match.  The current row's u starts at 0.0 (it is
// untouched before its own iteration) and lives in ucol[0].
//
// Per Dijkstra step: one predicated cost-row gather, the slack update, a
// per-lane first-minimum, and a warp argmin that reproduces the reference's
// "lowest j among equal minima" (mapping.py:103-105) with three redux.sync
// (order-preserving 64-bit key, -0.0 folded to +0.0 so signed zeros tie as
// they do under '<'), then delta = the winner's own minv (bit-exact).

constexpr int kO_WARPS = 4;

// doubles at the head of a plan's shared region: ucol (n + 1), and in the
// epilogue the per-row weights (rows) unless those go to the dictionary area
__host__ __device__ __forceinline__ int outer_dbl_elems(int max_n, int max_rows, bool wv_in_dict) {
  return wv_in_dict || max_n + 1 > max_rows ? max_n + 1 : max_rows;
}
// Dictionary coding of the fused matrix: real fused weights take few distinct
// values (2-5 distinct per row), so the warp packs its plan's
// nA x nB matrix into one-byte codes + a 256-entry table in shared memory and
// every Dijkstra step gathers its cost row from shared memory instead of L2.
// A plan with more than 256 distinct values falls back to the L2 gather.

// match / way are int16 (n <= 4095)
__host__ __device__ __forceinline__ size_t outer_base_bytes(int max_n, int dbl_elems) {
  size_t bytes = (size_t)dbl_elems * 8 + (size_t)(max_n + 1) * 2 * 2;
  return (bytes + 15) & ~(size_t)15;
}
// codes: the zero-padded n x n matrix (row stride n) + slack for the
// unpredicated per-step row reads (slot k of thread t reads column t + T k)
__host__ __device__ __forceinline__ size_t outer_dict_bytes(int max_n, int slack) {
  return (size_t)kDictSlots * 8 + (((size_t)max_n * max_n + slack + 15) & ~(size_t)15);
}
// outer-KM modes: 0 = cost rows gathered from the fused matrix in L2,
// 1 = one-byte codes in shared memory, 2 = codes in a global (L2-resident)
// scratch, only the 256-entry table in shared memory -- for big plans whose
// shared-memory codes would leave few warps per SM
enum { kOuterL2 = 0, kOuterSmemCodes = 1, kOuterGlobalCodes = 2 };

__host__ __device__ __forceinline__ bool outer_wv_in_dict(int max_n, int max_rows, int mode) {
  const size_t room = mode == kOuterSmemCodes ? outer_dict_bytes(max_n, 0)
                      : mode == kOuterGlobalCodes ? (size_t)kDictSlots * 8 : 0;
  return (size_t)max_rows * 8 <= room;
}
__host__ __device__ __forceinline__ size_t outer_smem_per_warp(int max_n, int max_rows, int mode,
                                                              int warps, int cpl) {
  size_t bytes = outer_base_bytes(max_n, outer_dbl_elems(max_n, max_rows, outer_wv_in_dict(max_n, max_rows, mode)));
  if (mode == kOuterSmemCodes) bytes += outer_dict_bytes(max_n, 32 * warps * cpl);
  if (mode == kOuterGlobalCodes) bytes += (size_t)kDictSlots * 8;
  if (warps > 1) bytes += (size_t)2 * warps * 24 + (size_t)4 * warps * 4;  // step partials
  return bytes;
}

struct OuterArgs {
  const sk_plan* plans;
  int n_plans;
  const int32_t* row_ptr;
  const sk_segment* segs;
  const double* F;
  const uint32_t* perm;
  int32_t* assign;
  double* total;
  int64_t* steps;  // optional: {Dijkstra steps, cost loads} per plan (profiling)
  uint32_t zero_perm[9];  // perm buffer stores (perm XOR zero_perm[g])
  size_t smem_per_warp;
  int max_n;
  int dbl_elems;
  int wv_in_dict;  // coded modes: epilogue row weights live in the dictionary area
  unsigned char* codes;  // kOuterGlobalCodes: per plan q at codes + q * codes_stride + 16
  size_t codes_stride;
  // optional: k_fuse's dictionaries (FuseCodes); a plan whose slot 0 is still
  // kEmpty arrives coded (codes as above, in every mode) -- no build from F
  const unsigned long long* dict;
};

// per-plan stride of the global code scratch: a 16-byte head (the step's
// column-0 read lands there), the padded n x n codes and the read slack
__host__ __device__ __forceinline__ size_t outer_codes_stride(int max_n, int warps, int cpl) {
  return ((size_t)16 + (size_t)max_n * max_n + (size_t)32 * warps * cpl + 15) & ~(size_t)15;
}

__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ unsigned lds_u8(unsigned a) {
  unsigned v;
  asm("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ double lds_f64(unsigned a) {
  double v;
  asm("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}

__device__ __forceinline__ unsigned long long order_key(double x) {
  unsigned long long b = (unsigned long long)__double_as_longlong(x);
  if ((b << 1) == 0ull) b = 0ull;  // -0.0 ties with +0.0, as under '<'
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// expansion of a general-range plan's matched pair: member k's column offset
// and matched weight from the side area (kept out of line: the regular
// plans' register allocation must not pay for it)
__device__ __noinline__ double generic_pick(const double* Fp, long long nAB, int g, long long pair, int k,
                                            int* col) {
  const long long e = pair * g + k;
  *col += reinterpret_cast<const unsigned char*>(Fp + nAB * (1 + g))[e];
  return Fp[nAB + e];
}

// W = warps per plan.  W == 1: one warp per plan, several plans per block,
// warp-synchronous (the common case: many plans, small n).  W > 1: one block
// per plan, columns spread over W warps, one __syncthreads per Dijkstra step
// (the warp winners are combined through double-buffered shared partials) --
// for big plans (n >~ 250) where per-plan latency, not throughput, binds.
template <int W>
__device__ __forceinline__ void plan_sync() {
  if (W == 1)
    __syncwarp();
  else
    __syncthreads();
}

template <int CPL, int MODE, int W>
__global__ void __launch_bounds__(32 * (W > kO_WARPS ? W : kO_WARPS)) k_outer(const OuterArgs A) {
  constexpr bool CODED = MODE != kOuterL2;
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int T = 32 * W;  // threads per plan
  const int pt = threadIdx.x % T, slot = threadIdx.x / T;
  const int lane = threadIdx.x & 31, pw = pt >> 5;
  const int q = blockIdx.x * (blockDim.x / T) + slot;
  if (q >= A.n_plans) return;  // uniform per plan (W > 1: per block)
  const sk_plan p = A.plans[q];
  const int g = p.group;
  const bool dense = (p.flags & SK_PLAN_DENSE) != 0;
  const int C = p.D * p.P * p.M;
  const int nA = p.rows / g, nB = C / g;
  const int n = nA > nB ? nA : nB;
  const int n1 = A.max_n + 1;

  // per-plan layout: [double ucol (/ wv): dbl_elems] [i16 match: n1] [i16 way: n1]
  //                  [CODED: u64 table[256] | mode 1: u8 codes[max_n^2] (/ wv)] ; W > 1 partials after
  unsigned char* base = smem + (size_t)slot * A.smem_per_warp;
  double* ucol = reinterpret_cast<double*>(base);
  unsigned short* match = reinterpret_cast<unsigned short*>(base + (size_t)A.dbl_elems * 8);
  unsigned short* way = match + n1;

  const double* Fp = A.F + p.f_off;
  // dictionary-code the fused matrix into shared memory (CODED variant).
  // (pointers derived unconditionally from the __shared__ array so the
  // compiler addresses them as shared memory: plain LDS, no generic windows)
  bool coded = false;
  unsigned long long* table =
      reinterpret_cast<unsigned long long*>(base + outer_base_bytes(A.max_n, A.dbl_elems));
  unsigned char* codes = MODE == kOuterGlobalCodes ? A.codes + (size_t)q * A.codes_stride + 16
                                                   : reinterpret_cast<unsigned char*>(table + kDictSlots);
  const unsigned table_s = smem_addr(table), codes_s = smem_addr(codes);
  // W > 1: warp-winner partials, double-buffered by step parity
  struct Partial {
    unsigned long long key;
    double val;
    unsigned j, pad;
  };
  Partial* partial = reinterpret_cast<Partial*>(
      base + (A.smem_per_warp - (size_t)2 * W * sizeof(Partial)));
  unsigned* fastx = reinterpret_cast<unsigned*>(partial) - 4 * W;  // [2][W] x {neg, zero j}
  const bool precoded = CODED && A.dict != nullptr && !(p.flags & SK_PLAN_GENERIC) &&
                        __ldcg(A.dict + (size_t)q * kDictSlots) == kEmpty;
  if (precoded) {
    // k_fuse coded the plan: its dictionary into shared memory (+ the codes
    // themselves in the shared-memory mode; the global mode reads them in place)
    const unsigned long long* gd = A.dict + (size_t)q * kDictSlots;
    for (int t = pt; t < kDictSlots; t += T) table[t] = t == 0 ? 0ull : __ldcg(gd + t);
    if (MODE == kOuterSmemCodes) {
      // whole 16-byte words: the tail read stays inside the plan's stride and
      // the tail write inside the shared slack
      const uint4* src = reinterpret_cast<const uint4*>(A.codes + (size_t)q * A.codes_stride + 16);
      uint4* dst = reinterpret_cast<uint4*>(codes);
      const int c16 = (n * n + 15) >> 4;
      for (int e = pt; e < c16; e += T) dst[e] = __ldcs(src + e);
    }
    plan_sync<W>();
    coded = true;
  } else if (CODED) {
    // slot 0 holds +0.0 (its own hash slot), the code of the zero padding
    for (int t = pt; t < kDictSlots; t += T) table[t] = t == 0 ? 0ull : kEmpty;
    plan_sync<W>();
    bool fail = false;
    constexpr int U = 8;  // independent loads in flight per thread
    const int cnt = n * n;  // < 2^24: exact in float
    const float inv_n = 1.0f / (float)n;
    for (int e0 = 0; e0 < cnt; e0 += T * U) {
      unsigned long long bits[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        // branch-free (r, c) = divmod(e, n) and an always-valid address, so
        // the U loads stay in flight together
        const int e = e0 + u * T + pt;
        int r = (int)((float)e * inv_n);
        int c = e - r * n;
        r = c < 0 ? r - 1 : (c >= n ? r + 1 : r);
        c = c < 0 ? c + n : (c >= n ? c - n : c);
        const bool in = e < cnt && r < nA && c < nB;
        const unsigned long long x = (unsigned long long)__double_as_longlong(__ldcs(Fp + (in ? r * nB + c : 0)));
        bits[u] = in ? x : (e < cnt ? 0ull : kEmpty);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int e = e0 + u * T + pt;
        if (bits[u] == kEmpty) continue;
        // open addressing, every thread for itself: a plain shared load finds
        // values already in the table (almost all of them); only an empty
        // slot takes a CAS, and racing inserts of one value agree through it
        unsigned h = (unsigned)((bits[u] * 0x9E3779B97F4A7C15ull) >> 56);
        for (int tries = 0;; ++tries) {
          unsigned long long cur = *reinterpret_cast<volatile unsigned long long*>(table + h);
          if (cur == kEmpty) cur = atomicCAS(table + h, kEmpty, bits[u]);
          if (cur == kEmpty || cur == bits[u]) break;
          h = (h + 1) & (kDictSlots - 1);
          if (tries + 1 == kDictSlots) {
            fail = true;
            break;
          }
        }
        codes[e] = (unsigned char)h;
      }
    }
    if (W == 1) {
      coded = !__any_sync(kFull, fail);
      __syncwarp();
    } else {
      coded = !__syncthreads_or(fail);
    }
  }

  // static column masks: valid = 1..n, real = 1..nB (beyond: zero padding)
  static_assert(CPL <= 32, "32-bit column masks");
  unsigned valid = 0u, real = 0u;
#pragma unroll
  for (int k = 0; k < CPL; ++k) {
    const int j = 1 + pt + T * k;  // the virtual column 0 has no slot
    if (j >= 1 && j <= n) valid |= 1u << k;
    if (j >= 1 && j <= nB) real |= 1u << k;
  }
  double v[CPL], minv[CPL];
  int wr[CPL];
#pragma unroll
  for (int k = 0; k < CPL; ++k) {
    v[k] = 0.0;
    wr[k] = 0;
  }
  for (int j = pt; j <= n; j += T) {
    ucol[j] = 0.0;
    match[j] = 0;
  }
  plan_sync<W>();
  if (pt == 0) match[0] = 1;  // row 1 (ucol[0] = 0.0 already)
  plan_sync<W>();

  int nsteps = 0, nloads = 0;  // nloads: uncoded path only
  int parity = 0;
  // the row loop, instantiated once per cost-row source so the Dijkstra step
  // carries no per-step branch on whether the dictionary build succeeded
  auto km_rows = [&](auto use_codes) {
  constexpr bool UC = decltype(use_codes)::value;
  for (int i = 1; i <= n; ++i) {
    unsigned used = 0u;  // slot columns; column 0 (always used) is implicit
#pragma unroll
    for (int k = 0; k < CPL; ++k) minv[k] = kInf;
    int j0 = 0;
    // (W == 1) the row whose costs the step scans is carried from the previous
    // step's match[j0] read (match[0] = i); multi-warp shapes reload it,
    // which keeps their register count (and occupancy) down
    int i0c = i;
    while (true) {
      const int i0 = W == 1 ? i0c : (int)match[j0];
      const double ui0 = ucol[j0];
      const unsigned act = valid & ~used;
      // the row's weights w (cost = -w; padded entries are 0.0 -> cost -0.0)
      double wx[CPL];
      if constexpr (UC) {
        // the padded n x n code matrix: unpredicated reads, one LDS.U8 + one
        // LDS.64 per column (32-bit shared-window addresses); reads for
        // columns outside 1..n land in the slack and are never used
        const int rowo = (i0 - 1) * n + pt;
        if (MODE == kOuterGlobalCodes) {
          const unsigned char* rowg = codes + rowo;
#pragma unroll
          for (int k = 0; k < CPL; ++k) wx[k] = lds_f64(table_s + 8u * (unsigned)rowg[T * k]);
        } else {
          const unsigned rowc = codes_s + (unsigned)rowo;
#pragma unroll
          for (int k = 0; k < CPL; ++k) wx[k] = lds_f64(table_s + 8u * lds_u8(rowc + (unsigned)(T * k)));
        }
      } else {
        const unsigned ld = (i0 - 1) < nA ? (act & real) : 0u;
        const double* rowp = Fp + (i0 - 1) * nB + pt;
#pragma unroll
        for (int k = 0; k < CPL; ++k) {
          double x = 0.0;
          if ((ld >> k) & 1u) x = __ldg(rowp + T * k);
          wx[k] = x;
        }
        nloads += __popc(ld);
      }
      double best = kInf;
      unsigned bj = 0xffffffffu;  // column of the first minimum (none while best is +inf)
      int bk = 0;
#pragma unroll
      for (int k = 0; k < CPL; ++k) {
        const bool on = (act >> k) & 1u;
        // (cost - u[i0]) - v[j] with cost = -w: the negation folds into the
        // first DADD's operand modifiers (exact, same bits)
        const double cur = (-wx[k] - ui0) - v[k];
        const bool imp = on && cur < minv[k];
        minv[k] = imp ? cur : minv[k];
        wr[k] = imp ? j0 : wr[k];
        const bool better = on && minv[k] < best;
        best = better ? minv[k] : best;
        if (W == 1)
          bj = better ? (unsigned)(1 + pt + T * k) : bj;
        else
          bk = better ? k : bk;
      }
      if (W > 1) bj = (best < kInf) ? (unsigned)(1 + pt + T * bk) : 0xffffffffu;
      unsigned jw;
      double delta;
      // fast path (~90% of steps on real plans): no negative slack and some
      // zero slack -> the minimum is 0 and the reference's j1 is the lowest
      // column whose slack is (+-)0; delta = 0 changes no potential
      // one redux on a combined key: 0 = this lane has a negative slack,
      // its lowest zero-slack column (1..n) if any, else all ones; the
      // minimum is 0 (some negative: slow path), all ones (no zero: slow
      // path), or the reference's j1 of a zero step
      const unsigned fkey = best < 0.0 ? 0u : (best == 0.0 ? bj : 0xffffffffu);
      unsigned fm = __reduce_min_sync(kFull, fkey);
      if (W > 1) {
        // block-wide: the minimum over the warps' minima
        unsigned* fp = fastx + parity * 2 * W;
        if (lane == 0) fp[pw] = fm;
        __syncthreads();
        fm = fp[0];
#pragma unroll
        for (int w = 1; w < W; ++w) fm = min(fm, fp[w]);
      }
      const bool fast = fm != 0u && fm != 0xffffffffu;
      if (fast) jw = fm;
      if (fast) {
        delta = 0.0;
      } else {
      // argmin over (value, lowest j): order-preserving key, three redux.sync
      const unsigned long long key = order_key(best);
      const unsigned hi = __reduce_min_sync(kFull, (unsigned)(key >> 32));
      const bool c1 = (unsigned)(key >> 32) == hi;
      const unsigned lo = __reduce_min_sync(kFull, c1 ? (unsigned)key : 0xffffffffu);
      const bool c2 = c1 && (unsigned)key == lo;
      jw = __reduce_min_sync(kFull, c2 ? bj : 0xffffffffu);
      delta = __shfl_sync(kFull, best, ((jw - 1) % T) & 31);
      if (W > 1) {
        Partial* pp = partial + parity * W;
        if (lane == 0) pp[pw] = {((unsigned long long)hi << 32) | lo, delta, jw, 0u};
        __syncthreads();
        unsigned long long bkey = pp[0].key;
        jw = pp[0].j;
        delta = pp[0].val;
#pragma unroll
        for (int w = 1; w < W; ++w) {
          const Partial o = pp[w];
          if (o.key < bkey || (o.key == bkey && o.j < jw)) {
            bkey = o.key;
            jw = o.j;
            delta = o.val;
          }
        }
      }
      }
      if (W > 1) parity ^= 1;
      const int j1 = (int)jw;
      // a zero delta leaves every potential and slack numerically unchanged
      // (at most flips the sign of a zero, which no comparison or later
      // non-zero result can observe), so the update is skipped
      if (delta != 0.0) {
        if (pt == 0) ucol[0] += delta;  // column 0: the current row's u
#pragma unroll
        for (int k = 0; k < CPL; ++k) {
          const bool u = (used >> k) & 1u;
          if (u) ucol[1 + pt + T * k] += delta;
          v[k] = u ? v[k] - delta : v[k];
          minv[k] = (!u && ((valid >> k) & 1u)) ? minv[k] - delta : minv[k];
        }
      }
      j0 = j1;
      if ((unsigned)(j0 - 1) % (unsigned)T == (unsigned)pt) used |= 1u << ((unsigned)(j0 - 1) / (unsigned)T);
      if (W == 1) {
        i0c = match[j0];
        if (i0c == 0) break;
      } else if (match[j0] == 0) {
        break;
      }
    }
    // every step marked one column used: the row's step count
    if (A.steps) nsteps += __popc(used);
    // publish predecessors, then walk the augmenting path (one thread), then
    // seed the next row
#pragma unroll
    for (int k = 0; k < CPL; ++k)
      if (((used | valid) >> k) & 1u) way[1 + pt + T * k] = (unsigned short)wr[k];
    plan_sync<W>();
    if (pt == 0) {
      while (j0) {
        const int j1 = way[j0];
        match[j0] = match[j1];
        ucol[j0] = ucol[j1];
        j0 = j1;
      }
      match[0] = (unsigned short)(i + 1);
      ucol[0] = 0.0;
    }
    plan_sync<W>();
  }
  };
  if (CODED && coded)
    km_rows(std::true_type{});
  else
    km_rows(std::false_type{});

  // row_to_col for real fused rows -> way[] (free now)
  for (int j = pt + 1; j <= n; j += T) {
    const int r = match[j];
    if (r >= 1 && r <= nA) way[r - 1] = (unsigned short)(j - 1);
  }
  plan_sync<W>();
  double* wv = (CODED && A.wv_in_dict) ? reinterpret_cast<double*>(table) : ucol;
  int32_t* out = A.assign + p.out_off;
  const int32_t* __restrict__ row_ptr = A.row_ptr;
  const sk_segment* __restrict__ segs = A.segs;
  for (int r = pt; r < p.rows; r += T) {
    const int a = r / g, k = r % g;
    const int b = way[a];
    if (b < nB) {
      int col = b * g;
      double w;
      if (p.flags & SK_PLAN_GENERIC) {
        // matched weights and permutation from the plan's side area
        const long long nAB = (long long)nA * nB;
        const long long e = ((long long)a * nB + b) * g + k;
        col += reinterpret_cast<const unsigned char*>(Fp + nAB * (1 + g))[e];
        w = Fp[nAB + e];
      } else {
        if (g > 1)
          col += (int)(((A.perm[p.f_off + (long long)a * nB + b] ^ A.zero_perm[g]) >> (4 * k)) & 15u);
        w = dense ? Fp[(long long)r * nB + col] : weight_at(p, row_ptr, segs, r, col);
      }
      out[r] = col;
      wv[r] = w;
    } else {
      out[r] = -1;
      wv[r] = -1.0;
    }
  }
  plan_sync<W>();
  if (A.steps) {
#pragma unroll
    for (int off = 16; off; off >>= 1) {  // < 2^31 per plan
      nloads += __shfl_xor_sync(kFull, nloads, off);
      nsteps += __shfl_xor_sync(kFull, nsteps, off);
    }
    if (W == 1) {
      if (lane == 0) {
        A.steps[2 * q] = nsteps;
        A.steps[2 * q + 1] = nloads;
      }
    } else {
      if (pt == 0) A.steps[2 * q] = A.steps[2 * q + 1] = 0;
      __syncthreads();
      if (lane == 0) {
        atomicAdd(reinterpret_cast<unsigned long long*>(A.steps + 2 * q), (unsigned long long)nsteps);
        atomicAdd(reinterpret_cast<unsigned long long*>(A.steps + 2 * q + 1), (unsigned long long)nloads);
      }
    }
  }
  if (pt == 0) {
    // total_weight in the reference's order (mapping.py:143-148 / 274-282)
    double t = 0.0;
    for (int r = 0; r < p.rows; ++r) {
      const double w = wv[r];
      if (w >= 0.0) t += w;
    }
    A.total[q] = t;
  }
}

// ---------------------------------------------------------------------------
// K2b for outer problems beyond the register-resident shapes (n > 4095):
// one 1024-thread CTA per plan runs the reference's _hungarian_max
// (mapping.py:71-122) literally, with the per-column state (u, v, minv,
// match, way, used) in a per-plan device scratch.  Thread t scans columns
// t + 1, t + 1 + 1024, ... (ascending, first minimum), the block argmin keeps
// the lowest column among equal minima, and the potential update touches
// distinct rows -- the same results as the sequential scan at any n.

constexpr int kH_TPB = 1024;

__host__ __device__ __forceinline__ size_t huge_stride(int max_n, int max_rows) {
  const size_t n1 = (size_t)max_n + 1;
  return ((n1 * (3 * 8 + 2 * 4 + 1) + 8 + (size_t)max_rows * 8) + 255) & ~(size_t)255;
}

__global__ void __launch_bounds__(kH_TPB) k_outer_huge(const OuterArgs A, unsigned char* __restrict__ scratch,
                                                       size_t stride) {
  __shared__ unsigned long long s_key[kH_TPB / 32];
  __shared__ unsigned s_j[kH_TPB / 32];
  __shared__ double s_val[kH_TPB / 32];
  __shared__ int s_j1;
  __shared__ double s_delta;
  const int q = blockIdx.x;
  if (q >= A.n_plans) return;
  const sk_plan p = A.plans[q];
  const int g = p.group;
  const bool dense = (p.flags & SK_PLAN_DENSE) != 0;
  const int C = p.D * p.P * p.M;
  const int nA = p.rows / g, nB = C / g;
  const int n = nA > nB ? nA : nB;
  const int t = threadIdx.x, lane = t & 31, wi = t >> 5;
  const size_t n1 = (size_t)n + 1;
  unsigned char* base = scratch + (size_t)q * stride;
  double* u = reinterpret_cast<double*>(base);
  double* v = u + n1;
  double* minv = v + n1;
  int* match = reinterpret_cast<int*>(minv + n1);
  int* way = match + n1;
  unsigned char* used = reinterpret_cast<unsigned char*>(way + n1);
  double* wv = reinterpret_cast<double*>(base + ((n1 * (3 * 8 + 2 * 4 + 1) + 7) & ~(size_t)7));
  const double* Fp = A.F + p.f_off;
  for (int j = t; j <= n; j += kH_TPB) {
    u[j] = 0.0;
    v[j] = 0.0;
    match[j] = 0;
    way[j] = 0;
  }
  __syncthreads();
  for (int i = 1; i <= n; ++i) {
    for (int j = t; j <= n; j += kH_TPB) {
      minv[j] = kInf;
      used[j] = 0;
    }
    if (t == 0) match[0] = i;
    __syncthreads();
    int j0 = 0;
    while (true) {
      if (t == 0) used[j0] = 1;
      __syncthreads();
      const int i0 = match[j0];
      const double ui0 = u[i0];
      const double* row = Fp + (long long)(i0 - 1) * nB;
      double best = kInf;
      unsigned bj = 0xffffffffu;
      for (int j = t + 1; j <= n; j += kH_TPB) {
        if (used[j]) continue;
        const double wgt = (i0 - 1 < nA && j - 1 < nB) ? row[j - 1] : 0.0;
        const double cur = (-wgt - ui0) - v[j];
        double mv = minv[j];
        if (cur < mv) {
          mv = cur;
          minv[j] = cur;
          way[j] = j0;
        }
        if (mv < best) {
          best = mv;
          bj = (unsigned)j;
        }
      }
      // block argmin on (value, lowest j)
      const unsigned long long key = bj == 0xffffffffu ? ~0ull : order_key_g(best);
      const unsigned hi = __reduce_min_sync(kFull, (unsigned)(key >> 32));
      const bool c1 = (unsigned)(key >> 32) == hi;
      const unsigned lo = __reduce_min_sync(kFull, c1 ? (unsigned)key : 0xffffffffu);
      const bool c2 = c1 && (unsigned)key == lo;
      const unsigned jw = __reduce_min_sync(kFull, c2 ? bj : 0xffffffffu);
      const unsigned src = __ffs(__ballot_sync(kFull, c2 && bj == jw)) - 1;
      const double dv = __shfl_sync(kFull, best, src);
      if (lane == 0) {
        s_key[wi] = ((unsigned long long)hi << 32) | lo;
        s_j[wi] = jw;
        s_val[wi] = dv;
      }
      __syncthreads();
      if (t == 0) {
        unsigned long long bk = s_key[0];
        unsigned bjj = s_j[0];
        double bv = s_val[0];
        for (int w = 1; w < kH_TPB / 32; ++w)
          if (s_key[w] < bk || (s_key[w] == bk && s_j[w] < bjj)) {
            bk = s_key[w];
            bjj = s_j[w];
            bv = s_val[w];
          }
        s_j1 = (int)bjj;
        s_delta = bv;
      }
      __syncthreads();
      const double delta = s_delta;
      const int j1 = s_j1;
      for (int j = t; j <= n; j += kH_TPB) {
        if (used[j]) {
          u[match[j]] += delta;
          v[j] -= delta;
        } else {
          minv[j] -= delta;
        }
      }
      __syncthreads();
      j0 = j1;
      if (match[j0] == 0) break;
    }
    if (t == 0) {
      while (j0) {
        const int j1 = way[j0];
        match[j0] = match[j1];
        j0 = j1;
      }
    }
    __syncthreads();
  }
  // row_to_col for real fused rows -> way[] (free now), then the expansion
  for (int j = t + 1; j <= n; j += kH_TPB) {
    const int r = match[j];
    if (r >= 1 && r <= nA) way[r - 1] = j - 1;
  }
  __syncthreads();
  const bool generic = (p.flags & SK_PLAN_GENERIC) != 0;
  const long long nAB = (long long)nA * nB;
  int32_t* out = A.assign + p.out_off;
  for (int r = t; r < p.rows; r += kH_TPB) {
    const int a = r / g, k = r % g;
    const int b = way[a];
    if (b < nB) {
      int col = b * g;
      double w;
      if (generic) {
        w = generic_pick(Fp, nAB, g, (long long)a * nB + b, k, &col);
      } else {
        if (g > 1)
          col += (int)(((A.perm[p.f_off + (long long)a * nB + b] ^ A.zero_perm[g]) >> (4 * k)) & 15u);
        w = dense ? Fp[(long long)r * nB + col] : weight_at(p, A.row_ptr, A.segs, r, col);
      }
      out[r] = col;
      wv[r] = w;
    } else {
      out[r] = -1;
      wv[r] = -1.0;
    }
  }
  __syncthreads();
  if (t == 0) {
    double tot = 0.0;
    for (int r = 0; r < p.rows; ++r)
      if (wv[r] >= 0.0) tot += wv[r];
    A.total[q] = tot;
    if (A.steps) A.steps[2 * q] = A.steps[2 * q + 1] = 0;
  }
}

int launch_outer_huge(const OuterArgs& A, int max_rows, cudaStream_t s) {
  const size_t stride = huge_stride(A.max_n, max_rows);
  void* scratch = nullptr;
  if (cudaMallocAsync(&scratch, stride * (size_t)A.n_plans, s) != cudaSuccess)
    return cuda_check("outer KM scratch (cudaMallocAsync)");
  k_outer_huge<<<A.n_plans, kH_TPB, 0, s>>>(A, static_cast<unsigned char*>(scratch), stride);
  int rc = cuda_check("k_outer_huge launch");
  cudaFreeAsync(scratch, s);
  return rc;
}

// ---------------------------------------------------------------------------
// sweep expansion: compact descriptors -> rows x 2 segments (model + cache)

__global__ void k_sweep_expand(const sk_sweep_desc* __restrict__ desc, const uint32_t* __restrict__ alive,
                               const int64_t* __restrict__ tok, const sk_plan* __restrict__ plans,
                               int32_t* __restrict__ row_ptr, sk_segment* __restrict__ segs) {
  const sk_sweep_desc ds = desc[blockIdx.y];
  const sk_plan p = plans[ds.plan];
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= p.rows) return;
  const int G = ds.G;
  const int rank = r / G, g = r % G;
  // index of the rank-th alive instance (instances i-0..i-(n-1) in natural order)
  const int words = (ds.n_inst + 31) >> 5;
  int k = -1, seen = 0;
  for (int w = 0; w < words; ++w) {
    const uint32_t bits = alive[ds.alive_off + w];
    const int c = __popc(bits);
    if (seen + c > rank) {
      uint32_t b = bits;
      for (int t = rank - seen; t > 0; --t) b &= b - 1;
      k = w * 32 + __ffs(b) - 1;
      break;
    }
    seen += c;
  }
  const long long x = (long long)p.row_base + r;
  if (r == 0) row_ptr[p.row_base] = (int32_t)(2 * (long long)p.row_base);
  row_ptr[x + 1] = (int32_t)(2 * (x + 1));
  sk_segment ms = {0, 0, 0, 0, 0, 0, 0};
  sk_segment cs = {0, 0, 0, 0, 0, 0, 0};
  const int q = k * G + g;
  if (k >= 0 && q < ds.oD * ds.oP * ds.oM) {
    const int m = q % ds.oM, st = (q / ds.oM) % ds.oP, d = q / (ds.oM * ds.oP);
    const int qq = p.L / ds.oP, rr = p.L % ds.oP;
    const int s0 = st * qq + min(st, rr);
    const int s1 = s0 + qq + (st < rr ? 1 : 0);
    const int w = p.K / ds.oM;
    ms.l0 = s0;
    ms.l1 = s1;
    ms.a = m * w;
    ms.b = m * w + w;
    ms.pipe = 0;
    ms.unit = ds.bpl;
    const long long tsum = tok[ds.tok_off + d];
    if (tsum > 0 && d + 1 <= p.D) {  // identity inheritance on min(D_old, D_new)
      cs = ms;
      cs.pipe = d + 1;
      cs.unit = ds.kv * tsum;
    }
  }
  segs[2 * x] = ms;
  segs[2 * x + 1] = cs;
}

// ---------------------------------------------------------------------------
// K3: batched byte-range copies (the executor's data path).  Each CTA walks
// whole chunks; 16-B vector loads from the (peer-mapped) source with 4
// independent requests in flight per thread.

constexpr int kC_TPB = 512;

__global__ void __launch_bounds__(kC_TPB) k_copy(const sk_copy* __restrict__ copies, int n) {
  for (int c = blockIdx.x; c < n; c += gridDim.x) {
    const sk_copy cp = copies[c];
    const unsigned char* src = reinterpret_cast<const unsigned char*>(cp.src);
    unsigned char* dst = reinterpret_cast<unsigned char*>(cp.dst);
    const uint64_t bytes = cp.bytes;
    const bool aligned = ((cp.src | cp.dst) & 15ull) == 0;
    uint64_t done = 0;
    if (aligned) {
      const uint64_t nv = bytes >> 4;
      const int4* s4 = reinterpret_cast<const int4*>(src);
      int4* d4 = reinterpret_cast<int4*>(dst);
      uint64_t i = threadIdx.x;
      constexpr int U = 8;  // 64 KB in flight per CTA hides NVLink read latency
      for (; i + (U - 1) * kC_TPB < nv; i += U * kC_TPB) {
        int4 t[U];
#pragma unroll
        for (int u = 0; u < U; ++u) t[u] = __ldcs(s4 + i + u * kC_TPB);
#pragma unroll
        for (int u = 0; u < U; ++u) __stcs(d4 + i + u * kC_TPB, t[u]);
      }
      for (; i < nv; i += kC_TPB) __stcs(d4 + i, __ldcs(s4 + i));
      done = nv << 4;
    }
    for (uint64_t i = done + threadIdx.x; i < bytes; i += kC_TPB) dst[i] = src[i];
  }
}

// plans per block (W == 1) maximising the plans resident per SM under the
// shared-memory (incl. the 1 KB per-block reserve), thread and block limits;
// *resident receives that count (0: does not fit)
int best_per_block(size_t plan_smem, int W, size_t cap, int* resident = nullptr) {
  constexpr size_t kSmemSM = 228 * 1024, kReserve = 1024;
  int best = 0, best_res = 0;
  for (int pb = 1; pb <= (W == 1 ? kO_WARPS : 1); ++pb) {
    const size_t blk = plan_smem * pb;
    if (blk > cap) break;
    int nb = (int)(kSmemSM / (blk + kReserve));
    nb = nb < 2048 / (32 * W * pb) ? nb : 2048 / (32 * W * pb);
    nb = nb < 32 ? nb : 32;
    if (nb * pb >= best_res && nb > 0) {
      best_res = nb * pb;
      best = pb;
    }
  }
  if (resident) *resident = best_res;
  return best;
}

constexpr size_t kSmemCodedCap = 200 * 1024;

// plans resident per SM below which big plans move their codes to the global
// scratch (when the caller provides one); SK_OUTER_GMIN overrides (tuning)
int global_codes_threshold() {
  static const int v = [] {
    const char* e = getenv("SK_OUTER_GMIN");
    return e ? atoi(e) : 12;
  }();
  return v;
}

// mode the launcher picks for n_plans plans of (max_n, max_rows) at (CPL, W):
// global codes when shared-memory codes would leave few plans per SM and the
// launch is big enough (>= 2 waves) for the extra concurrency to pay
int outer_mode(int n_plans, int max_n, int max_rows, int W, int CPL, bool have_codes) {
  constexpr int kSMs = 148;
  static const bool force_global = [] {  // testing: every class with a scratch
    const char* e = getenv("SK_OUTER_FORCE_GLOBAL");
    return e && atoi(e) != 0;
  }();
  if (have_codes && force_global) return kOuterGlobalCodes;
  int res = 0;
  best_per_block(outer_smem_per_warp(max_n, max_rows, kOuterSmemCodes, W, CPL), W, kSmemCodedCap, &res);
  const bool few = res < global_codes_threshold() && (long long)n_plans > 2LL * kSMs * res;
  if (have_codes && (res == 0 || few)) return kOuterGlobalCodes;
  return res > 0 ? kOuterSmemCodes : kOuterL2;
}

// (columns per thread, warps per plan) for a size class -- must match
// outer_dispatch's instantiations
void outer_shape(int max_n, int* cpl, int* w) {
  const int need = (max_n + 31) / 32;  // columns 1..n over the slots
  *w = 1;
  if (need <= 6) {
    *cpl = need < 1 ? 1 : need;
    return;
  }
  if (need <= 8) {
    *cpl = 8;
    return;
  }
  // two warps per plan up to n = 512: fewer instructions per step than four
  // warps and still a short per-step chain (measured: +16% at 512 positions,
  // +5% at 1,024; two warps with 12 columns per thread lose to four warps)
  const int need2 = (max_n + 63) / 64;
  if (need2 <= 8) {
    *w = 2;
    *cpl = need2 <= 5 ? 5 : (need2 <= 6 ? 6 : 8);
    return;
  }
  const int need4 = (max_n + 127) / 128;
  *w = 4;
  if (need4 <= 3) *cpl = 3;
  else if (need4 <= 6) *cpl = need4;
  else if (need4 <= 8) *cpl = 8;
  else if (need4 <= 12) *cpl = 12;
  else if (need4 <= 16) *cpl = 16;
  else {
    const int need8 = (max_n + 255) / 256;
    *w = 8;
    *cpl = need8 <= 12 ? 12 : 16;
  }
}

template <int CPL, int MODE, int W>
void configure_outer() {
  // per launch (a few microseconds): the attribute belongs to the current
  // device's context, and callers may switch devices between launches
  cudaFuncSetAttribute(k_outer<CPL, MODE, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
}

template <int CPL, int W>
int launch_outer(OuterArgs A, int max_rows, size_t codes_bytes, cudaStream_t s) {
  const size_t stride = outer_codes_stride(A.max_n, W, CPL);
  const bool have_codes = A.codes != nullptr && codes_bytes >= stride * (size_t)A.n_plans;
  const int mode = outer_mode(A.n_plans, A.max_n, max_rows, W, CPL, have_codes);
  const size_t plan_smem = outer_smem_per_warp(A.max_n, max_rows, mode, W, CPL);
  const int per_block = best_per_block(plan_smem, W, mode == kOuterSmemCodes ? kSmemCodedCap : 227 * 1024);
  if (per_block == 0)
    return set_err(SK_EINVAL, "outer KM shared memory %zu B too large", plan_smem);
  A.wv_in_dict = outer_wv_in_dict(A.max_n, max_rows, mode);
  A.dbl_elems = outer_dbl_elems(A.max_n, max_rows, A.wv_in_dict != 0);
  A.smem_per_warp = plan_smem;
  A.codes_stride = stride;
  const size_t smem = plan_smem * per_block;
  const int blocks = (A.n_plans + per_block - 1) / per_block;
  if (mode == kOuterSmemCodes) {
    configure_outer<CPL, kOuterSmemCodes, W>();
    k_outer<CPL, kOuterSmemCodes, W><<<blocks, per_block * 32 * W, smem, s>>>(A);
  } else if (mode == kOuterGlobalCodes) {
    configure_outer<CPL, kOuterGlobalCodes, W>();
    k_outer<CPL, kOuterGlobalCodes, W><<<blocks, per_block * 32 * W, smem, s>>>(A);
  } else {
    configure_outer<CPL, kOuterL2, W>();
    k_outer<CPL, kOuterL2, W><<<blocks, per_block * 32 * W, smem, s>>>(A);
  }
  return cuda_check("k_outer launch");
}

// Small plans: one warp per plan (columns per lane = need).  Bigger plans:
// one 2-, 4- or 8-warp block per plan.
int outer_dispatch(const OuterArgs& A, int max_rows, size_t codes_bytes, cudaStream_t s) {
  int cpl = 0, w = 0;
  if (A.max_n > 4095) return launch_outer_huge(A, max_rows, s);
  outer_shape(A.max_n, &cpl, &w);
#define SK_OUTER_CASE(C, WW) \
  if (cpl == C && w == WW) return launch_outer<C, WW>(A, max_rows, codes_bytes, s);
  SK_OUTER_CASE(1, 1) SK_OUTER_CASE(2, 1) SK_OUTER_CASE(3, 1) SK_OUTER_CASE(4, 1)
  SK_OUTER_CASE(5, 1) SK_OUTER_CASE(6, 1) SK_OUTER_CASE(8, 1)
  SK_OUTER_CASE(5, 2) SK_OUTER_CASE(6, 2) SK_OUTER_CASE(8, 2)
  SK_OUTER_CASE(3, 4) SK_OUTER_CASE(4, 4) SK_OUTER_CASE(5, 4) SK_OUTER_CASE(6, 4)
  SK_OUTER_CASE(8, 4) SK_OUTER_CASE(12, 4) SK_OUTER_CASE(16, 4)
  SK_OUTER_CASE(12, 8) SK_OUTER_CASE(16, 8)
#undef SK_OUTER_CASE
  return set_err(SK_EINVAL, "outer KM shape (%d, %d) not instantiated", cpl, w);
}

constexpr int kMaxGridY = 65535;

}  // namespace

// ---------------------------------------------------------------------------
// C ABI

extern "C" {

int sk_abi_version(void) { return SPOTKM_ABI_VERSION; }

int64_t sk_fused_elems(int32_t nA, int32_t nB, int32_t group, int32_t flags) {
  const int64_t pairs = (int64_t)nA * nB;
  if (!(flags & SK_PLAN_GENERIC)) return pairs;
  return pairs * (1 + group) + (pairs * group + 7) / 8;
}

const char* sk_last_error(void) { return g_err; }

int sk_build_weights(const sk_plan* d_plans, int n_plans, const int32_t* d_row_ptr,
                     const sk_segment* d_segs, double* d_W, int max_rows, int max_cols, void* stream) {
  if (n_plans < 0 || max_rows < 0 || max_cols < 0) return set_err(SK_EINVAL, "negative sizes");
  if (n_plans == 0 || max_rows == 0 || max_cols == 0) return SK_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  for (int p0 = 0; p0 < n_plans; p0 += kMaxGridY) {
    const int np = n_plans - p0 < kMaxGridY ? n_plans - p0 : kMaxGridY;
    dim3 grid((max_rows + kW_RPB - 1) / kW_RPB, np);
    k_weights<<<grid, kW_TPB, 0, s>>>(d_plans + p0, d_row_ptr, d_segs, d_W);
    int rc = cuda_check("k_weights launch");
    if (rc) return rc;
  }
  return SK_OK;
}

int sk_map_fuse(const sk_plan* d_plans, int n_plans, const int32_t* d_row_ptr,
                const sk_segment* d_segs, double* d_fused, uint32_t* d_perm, int max_na, int max_nb,
                int group_mask, int64_t clear_begin, int64_t clear_count, void* stream) {
  if (n_plans < 0 || max_na < 0 || max_nb < 0) return set_err(SK_EINVAL, "negative sizes");
  if (n_plans == 0 || max_na == 0 || max_nb == 0) return SK_OK;
  if (clear_count > 0) {
    cudaStream_t cs = static_cast<cudaStream_t>(stream);
    if (cudaMemsetAsync(d_fused + clear_begin, 0, (size_t)clear_count * sizeof(double), cs) != cudaSuccess ||
        cudaMemsetAsync(d_perm + clear_begin, 0, (size_t)clear_count * sizeof(uint32_t), cs) != cudaSuccess)
      return cuda_check("clear fused buffers");
  }
  if (((long long)max_na * max_nb + kF_TPB - 1) / kF_TPB > 0x7fffffffLL)
    return set_err(SK_EINVAL, "too many fused pairs");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int mask = group_mask ? group_mask : 0x1ff;
  for (int p0 = 0; p0 < n_plans; p0 += kMaxGridY) {
    const int np = n_plans - p0 < kMaxGridY ? n_plans - p0 : kMaxGridY;
    int rc = SK_OK;
    if (mask & 1) {  // general-range plans: one warp per fused pair
      const long long pairs = (long long)max_na * max_nb;
      if ((pairs + kG_WARPS - 1) / kG_WARPS > 0x7fffffffLL) return set_err(SK_EINVAL, "too many fused pairs");
      dim3 grid((unsigned)((pairs + kG_WARPS - 1) / kG_WARPS), np);
      k_fuse_generic<<<grid, 32 * kG_WARPS, 0, s>>>(d_plans, p0, d_row_ptr, d_segs, d_fused);
      rc = cuda_check("k_fuse_generic launch");
    }
    if (!rc && (mask & (1 << 1))) rc = launch_fuse<1>(d_plans, p0, np, max_na, max_nb, d_row_ptr, d_segs, d_fused, d_perm, s);
    if (!rc && (mask & (1 << 2))) rc = launch_fuse<2>(d_plans, p0, np, max_na, max_nb, d_row_ptr, d_segs, d_fused, d_perm, s);
    if (!rc && (mask & (1 << 3))) rc = launch_fuse<3>(d_plans, p0, np, max_na, max_nb, d_row_ptr, d_segs, d_fused, d_perm, s);
    if (!rc && (mask & (1 << 4))) rc = launch_fuse<4>(d_plans, p0, np, max_na, max_nb, d_row_ptr, d_segs, d_fused, d_perm, s);
    if (!rc && (mask & (1 << 5))) rc = launch_fuse<5>(d_plans, p0, np, max_na, max_nb, d_row_ptr, d_segs, d_fused, d_perm, s);
    if (!rc && (mask & (1 << 6))) rc = launch_fuse<6>(d_plans, p0, np, max_na, max_nb, d_row_ptr, d_segs, d_fused, d_perm, s);
    if (!rc && (mask & (1 << 7))) rc = launch_fuse<7>(d_plans, p0, np, max_na, max_nb, d_row_ptr, d_segs, d_fused, d_perm, s);
    if (!rc && (mask & (1 << 8))) rc = launch_fuse<8>(d_plans, p0, np, max_na, max_nb, d_row_ptr, d_segs, d_fused, d_perm, s);
    if (rc) return rc;
  }
  return SK_OK;
}

int64_t sk_precoded_bytes(int n_plans, int max_n, int64_t* dict_bytes) {
  if (dict_bytes) *dict_bytes = 0;
  if (n_plans <= 0 || max_n <= 0 || max_n > 4095) return 0;
  int cpl = 0, w = 0;
  outer_shape(max_n, &cpl, &w);
  // the dictionaries, then the overflow list (n_plans ints) and its count
  if (dict_bytes) *dict_bytes = (int64_t)n_plans * kDictSlots * 8 + 4 * ((int64_t)n_plans + 1);
  return (int64_t)(outer_codes_stride(max_n, w, cpl) * (size_t)n_plans);
}

int sk_map_fuse_coded(const sk_plan* d_plans, int n_plans, const int32_t* d_row_ptr,
                      const sk_segment* d_segs, double* d_fused, uint32_t* d_perm, int max_na,
                      int max_nb, int group_mask, uint8_t* d_codes, int64_t codes_bytes,
                      uint64_t* d_dict, int64_t dict_bytes, void* stream) {
  if (n_plans < 0 || max_na < 0 || max_nb < 0) return set_err(SK_EINVAL, "negative sizes");
  if (n_plans == 0 || max_na == 0 || max_nb == 0) return SK_OK;
  const int max_n = max_na > max_nb ? max_na : max_nb;
  int64_t need_dict = 0;
  const int64_t need = sk_precoded_bytes(n_plans, max_n, &need_dict);
  if (need == 0 || d_codes == nullptr || d_dict == nullptr || codes_bytes < need || dict_bytes < need_dict)
    return set_err(SK_EINVAL, "coded fuse: code scratch %lld B / dictionaries %lld B needed (max_n %d)",
                   (long long)need, (long long)need_dict, max_n);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t tables = (size_t)n_plans * kDictSlots * 8;
  int* list = reinterpret_cast<int*>(reinterpret_cast<unsigned char*>(d_dict) + tables);
  int* count = list + n_plans;
  if (cudaMemsetAsync(d_dict, 0xff, tables, s) != cudaSuccess || cudaMemsetAsync(count, 0, 4, s) != cudaSuccess)
    return cuda_check("clear dictionaries");
  int cpl = 0, w = 0;
  outer_shape(max_n, &cpl, &w);
  const FuseCodes fc{d_codes, outer_codes_stride(max_n, w, cpl), reinterpret_cast<unsigned long long*>(d_dict)};
  const int mask = group_mask ? group_mask : 0x1ff;
  for (int p0 = 0; p0 < n_plans; p0 += kMaxGridY) {
    const int np = n_plans - p0 < kMaxGridY ? n_plans - p0 : kMaxGridY;
    int rc = SK_OK;
    if (mask & 1) {  // general-range plans keep the double matrix (the outer KM codes them itself)
      const long long pairs = (long long)max_na * max_nb;
      if ((pairs + kG_WARPS - 1) / kG_WARPS > 0x7fffffffLL) return set_err(SK_EINVAL, "too many fused pairs");
      dim3 grid((unsigned)((pairs + kG_WARPS - 1) / kG_WARPS), np);
      k_fuse_generic<<<grid, 32 * kG_WARPS, 0, s>>>(d_plans, p0, d_row_ptr, d_segs, d_fused);
      rc = cuda_check("k_fuse_generic launch");
    }
#define SK_FUSE_CODED(GG) \
    if (!rc && (mask & (1 << GG))) rc = launch_fuse_coded<GG>(d_plans, p0, np, max_n, d_row_ptr, d_segs, d_perm, fc, s);
    SK_FUSE_CODED(1) SK_FUSE_CODED(2) SK_FUSE_CODED(3) SK_FUSE_CODED(4)
    SK_FUSE_CODED(5) SK_FUSE_CODED(6) SK_FUSE_CODED(7) SK_FUSE_CODED(8)
#undef SK_FUSE_CODED
    if (rc) return rc;
  }
  k_overflow_list<<<(n_plans + 255) / 256, 256, 0, s>>>(fc.dict, n_plans, list, count);
  int rc = cuda_check("k_overflow_list launch");
#define SK_FUSE_OVF(GG) \
  if (!rc && (mask & (1 << GG))) rc = launch_fuse_overflow<GG>(d_plans, list, count, d_row_ptr, d_segs, d_fused, d_perm, fc, s);
  SK_FUSE_OVF(1) SK_FUSE_OVF(2) SK_FUSE_OVF(3) SK_FUSE_OVF(4)
  SK_FUSE_OVF(5) SK_FUSE_OVF(6) SK_FUSE_OVF(7) SK_FUSE_OVF(8)
#undef SK_FUSE_OVF
  return rc;
}

int sk_map_outer_coded(const sk_plan* d_plans, int n_plans, const int32_t* d_row_ptr,
                       const sk_segment* d_segs, const double* d_fused, const uint32_t* d_perm,
                       int32_t* d_assign, double* d_total, int64_t* d_steps, int max_n, int max_rows,
                       uint8_t* d_codes, int64_t codes_bytes, const uint64_t* d_dict, void* stream) {
  if (n_plans < 0 || max_n < 0 || max_rows < 0 || codes_bytes < 0) return set_err(SK_EINVAL, "negative sizes");
  if (n_plans == 0) return SK_OK;
  if (sk_precoded_bytes(n_plans, max_n, nullptr) > codes_bytes || d_codes == nullptr || d_dict == nullptr)
    return set_err(SK_EINVAL, "coded outer KM: code scratch too small");
  OuterArgs A{d_plans, n_plans, d_row_ptr, d_segs, d_fused, d_perm, d_assign, d_total, d_steps, {}, 0, max_n, 0,
              0, d_codes, 0, reinterpret_cast<const unsigned long long*>(d_dict)};
  for (int g = 0; g <= 8; ++g) A.zero_perm[g] = zero_perm_of(g);
  return outer_dispatch(A, max_rows, (size_t)codes_bytes, static_cast<cudaStream_t>(stream));
}

int sk_map_outer_codes(const sk_plan* d_plans, int n_plans, const int32_t* d_row_ptr,
                       const sk_segment* d_segs, const double* d_fused, const uint32_t* d_perm,
                       int32_t* d_assign, double* d_total, int64_t* d_steps, int max_n, int max_rows,
                       uint8_t* d_codes, int64_t codes_bytes, void* stream) {
  if (n_plans < 0 || max_n < 0 || max_rows < 0 || codes_bytes < 0) return set_err(SK_EINVAL, "negative sizes");
  if (n_plans == 0) return SK_OK;
  OuterArgs A{d_plans, n_plans, d_row_ptr, d_segs, d_fused, d_perm, d_assign, d_total, d_steps, {}, 0, max_n, 0,
              0, d_codes, 0};
  for (int g = 0; g <= 8; ++g) A.zero_perm[g] = zero_perm_of(g);
  return outer_dispatch(A, max_rows, (size_t)codes_bytes, static_cast<cudaStream_t>(stream));
}

int64_t sk_outer_codes_bytes(int n_plans, int max_n, int max_rows) {
  if (n_plans <= 0 || max_n <= 0 || max_n > 4095 || max_rows < 0) return 0;
  int cpl = 0, w = 0;
  outer_shape(max_n, &cpl, &w);
  if (outer_mode(n_plans, max_n, max_rows, w, cpl, true) != kOuterGlobalCodes) return 0;
  return (int64_t)(outer_codes_stride(max_n, w, cpl) * (size_t)n_plans);
}

int sk_map_outer(const sk_plan* d_plans, int n_plans, const int32_t* d_row_ptr,
                 const sk_segment* d_segs, const double* d_fused, const uint32_t* d_perm,
                 int32_t* d_assign, double* d_total, int64_t* d_steps, int max_n, int max_rows,
                 void* stream) {
  return sk_map_outer_codes(d_plans, n_plans, d_row_ptr, d_segs, d_fused, d_perm, d_assign, d_total,
                            d_steps, max_n, max_rows, nullptr, 0, stream);
}

int sk_map_batched(const sk_plan* d_plans, int n_plans, const int32_t* d_row_ptr,
                   const sk_segment* d_segs, double* d_fused, uint32_t* d_perm, int32_t* d_assign,
                   double* d_total, int max_na, int max_nb, int max_rows, int group_mask,
                   int64_t fused_elems, void* stream) {
  (void)fused_elems;  // k_fuse writes every fused element itself
  int rc = sk_map_fuse(d_plans, n_plans, d_row_ptr, d_segs, d_fused, d_perm, max_na, max_nb,
                       group_mask, 0, 0, stream);
  if (rc) return rc;
  const int max_n = max_na > max_nb ? max_na : max_nb;
  return sk_map_outer(d_plans, n_plans, d_row_ptr, d_segs, d_fused, d_perm, d_assign, d_total, nullptr,
                      max_n, max_rows, stream);
}

int sk_km_dense(const sk_plan* d_plans, int n_plans, const double* d_W, int32_t* d_assign,
                double* d_total, int max_n, int max_rows, void* stream) {
  return sk_map_outer(d_plans, n_plans, nullptr, nullptr, d_W, nullptr, d_assign, d_total, nullptr,
                      max_n, max_rows, stream);
}

int sk_sweep_expand(const sk_sweep_desc* d_desc, int n_desc, const uint32_t* d_alive,
                    const int64_t* d_tok, const sk_plan* d_plans, int32_t* d_row_ptr,
                    sk_segment* d_segs, int max_rows, void* stream) {
  if (n_desc < 0 || max_rows < 0) return set_err(SK_EINVAL, "negative sizes");
  if (n_desc == 0 || max_rows == 0) return SK_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  for (int p0 = 0; p0 < n_desc; p0 += kMaxGridY) {
    const int np = n_desc - p0 < kMaxGridY ? n_desc - p0 : kMaxGridY;
    // 64-row blocks: plans have ~R = 64 k + small rows, so 128-row blocks
    // would leave up to half of a plan's last block idle
    dim3 grid((max_rows + 63) / 64, np);
    k_sweep_expand<<<grid, 64, 0, s>>>(d_desc + p0, d_alive, d_tok, d_plans, d_row_ptr, d_segs);
    int rc = cuda_check("k_sweep_expand launch");
    if (rc) return rc;
  }
  return SK_OK;
}

int sk_copy_batched(const sk_copy* d_copies, int n_copies, int n_ctas, void* stream) {
  if (n_copies < 0) return set_err(SK_EINVAL, "negative copy count");
  if (n_copies == 0) return SK_OK;
  if (n_ctas <= 0) n_ctas = 148 * 4;
  k_copy<<<n_ctas, kC_TPB, 0, static_cast<cudaStream_t>(stream)>>>(d_copies, n_copies);
  return cuda_check("k_copy launch");
}

int sk_enable_peer_access(int device, const int* peers, int n_peers) {
  int prev = 0;
  cudaGetDevice(&prev);
  if (cudaSetDevice(device) != cudaSuccess) return set_err(SK_ECUDA, "cudaSetDevice(%d)", device);
  for (int i = 0; i < n_peers; ++i) {
    if (peers[i] == device) continue;
    int ok = 0;
    cudaDeviceCanAccessPeer(&ok, device, peers[i]);
    if (!ok) {
      cudaSetDevice(prev);
      return set_err(SK_ENOPEER, "device %d cannot access peer %d", device, peers[i]);
    }
    cudaError_t e = cudaDeviceEnablePeerAccess(peers[i], 0);
    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
      cudaSetDevice(prev);
      return set_err(SK_ECUDA, "enable peer %d->%d: %s", device, peers[i], cudaGetErrorString(e));
    }
    cudaGetLastError();
  }
  cudaSetDevice(prev);
  return SK_OK;
}

}  // extern "C"
