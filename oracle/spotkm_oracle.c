/*
 * TEST INFRASTRUCTURE ONLY -- plain-C restatement of the reference's device
 * mapping for the structured preemption sweep, used as the
 * full-size parity checker and as the multi-core CPU baseline of bench.py.
 * The product (libspotkm.so) never links or calls this.
 *
 * Restated reference functions (under /root/reference/pkg/src/spotsim/):
 *   stage_layers        domain.py:271-283
 *   shard_interval      domain.py:286-288
 *   overlap_bytes       domain.py:299-320  (closed form for the structured
 *                        layout: SURVEY.md finding 2, exact integer numerator
 *                        over K = lcm(M_old, M_new), one rounded division)
 *   build_graph rows    mapping.py:193-198 (alive instances in index order)
 *   _hungarian_max      mapping.py:71-122  (same double operation order)
 *   map_devices         mapping.py:222-283 (two-step; flat when G == 1)
 *
 * The sweep semantics: instances i-0..i-(n-1), old config laid out
 * positionally (GPU k*G+g holds old position k*G+g), some instances
 * preempted (alive bitmask), each old pipeline d carries cached requests
 * whose token counts sum to tok[d], identity inheritance on min(D_old, D_new).
 * The input structs are the same byte layout as include/spotkm.h's
 * sk_sweep_desc / sk_plan so bench and tests share one generator.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int32_t oD, oP, oM, G, n_inst, alive_off, tok_off, plan;
  int64_t bpl, kv;
} oc_desc;

typedef struct {
  int32_t rows, D, P, M, L, K, group, flags, row_base, reserved;
  int64_t f_off, out_off, reserved2;
} oc_plan;

static void stage_block(int L, int P, int st, int* s0, int* s1) {
  int q = L / P, r = L % P;
  *s0 = st * q + (st < r ? st : r);
  *s1 = *s0 + q + (st < r ? 1 : 0);
}

static int imin(int a, int b) { return a < b ? a : b; }
static int imax(int a, int b) { return a > b ? a : b; }

/* reference _hungarian_max on an n x n row-major matrix; out[row] = col */
static void hungarian_max(const double* w, int n, int* out, double* u, double* v, double* minv,
                          int* match, int* way, char* used) {
  if (n == 0) return;
  for (int j = 0; j <= n; ++j) {
    u[j] = 0.0;
    v[j] = 0.0;
    match[j] = 0;
    way[j] = 0;
  }
  for (int i = 1; i <= n; ++i) {
    match[0] = i;
    int j0 = 0;
    for (int j = 0; j <= n; ++j) {
      minv[j] = INFINITY;
      used[j] = 0;
    }
    for (;;) {
      used[j0] = 1;
      int i0 = match[j0];
      double delta = INFINITY;
      int j1 = 0;
      const double* row = w + (size_t)(i0 - 1) * n;
      for (int j = 1; j <= n; ++j) {
        if (used[j]) continue;
        double cost = -row[j - 1];
        double cur = cost - u[i0] - v[j];
        if (cur < minv[j]) {
          minv[j] = cur;
          way[j] = j0;
        }
        if (minv[j] < delta) {
          delta = minv[j];
          j1 = j;
        }
      }
      for (int j = 0; j <= n; ++j) {
        if (used[j]) {
          u[match[j]] += delta;
          v[j] -= delta;
        } else {
          minv[j] -= delta;
        }
      }
      j0 = j1;
      if (match[j0] == 0) break;
    }
    while (j0) {
      int j1 = way[j0];
      match[j0] = match[j1];
      j0 = j1;
    }
  }
  for (int j = 1; j <= n; ++j) out[match[j] - 1] = j - 1;
}

/* CPython >= 3.12 builtin sum over floats (int start 0, Neumaier) */
static double py_sum(const double* x, int n) {
  double f = 0.0 + x[0], c = 0.0;
  for (int i = 1; i < n; ++i) {
    double t = f + x[i];
    if (fabs(f) >= fabs(x[i]))
      c += (f - t) + x[i];
    else
      c += (x[i] - t) + f;
    f = t;
  }
  if (c != 0.0 && isfinite(c)) f += c;
  return f;
}

typedef struct {
  int has;         /* holds an old position */
  int d, s0, s1;   /* old pipeline (1-based) and layer block */
  int a, b;        /* old shard interval in 1/K units */
} oc_row;

static double weight(const oc_row* r, int c, const oc_plan* p, const oc_desc* ds, const int64_t* tok) {
  if (!r->has) return 0.0;
  int m = c % p->M, t = c / p->M, st = t % p->P, d = t / p->P + 1;
  int s0, s1;
  stage_block(p->L, p->P, st, &s0, &s1);
  int wdt = p->K / p->M;
  int ol = imin(r->s1, s1) - imax(r->s0, s0);
  int oi = imin(r->b, (m + 1) * wdt) - imax(r->a, m * wdt);
  if (ol <= 0 || oi <= 0) return 0.0;
  int64_t per = ds->bpl;
  int64_t ts = tok[ds->tok_off + r->d - 1];
  if (ts > 0 && r->d <= ds->oD && r->d <= p->D && r->d == d) per += ds->kv * ts;
  int64_t num = (int64_t)ol * oi * per;
  return (double)num / (double)p->K;
}

static int solve(const oc_desc* ds, const oc_plan* p, const uint32_t* alive, const int64_t* tok,
                 int32_t* assign, double* total) {
  const int R = p->rows, C = p->D * p->P * p->M, G = ds->G;
  oc_row* rows = (oc_row*)calloc((size_t)(R > 0 ? R : 1), sizeof(oc_row));
  int r = 0;
  for (int k = 0; k < ds->n_inst && r < R; ++k) {
    if (!((alive[ds->alive_off + (k >> 5)] >> (k & 31)) & 1u)) continue;
    for (int g = 0; g < G; ++g, ++r) {
      int q = k * G + g;
      oc_row* o = &rows[r];
      if (q >= ds->oD * ds->oP * ds->oM) continue;
      int m = q % ds->oM, st = (q / ds->oM) % ds->oP, d = q / (ds->oM * ds->oP);
      o->has = 1;
      o->d = d + 1;
      stage_block(p->L, ds->oP, st, &o->s0, &o->s1);
      int w = p->K / ds->oM;
      o->a = m * w;
      o->b = m * w + w;
    }
  }
  const int g = p->group;
  const int nA = R / g, nB = C / g, n = nA > nB ? nA : nB;
  double* fused = (double*)calloc((size_t)n * n + 1, sizeof(double));
  int* perm = (int*)calloc((size_t)nA * nB * g + 1, sizeof(int));
  double* u = (double*)malloc(sizeof(double) * (n + 1));
  double* v = (double*)malloc(sizeof(double) * (n + 1));
  double* mv = (double*)malloc(sizeof(double) * (n + 1));
  int* match = (int*)malloc(sizeof(int) * (n + 1));
  int* way = (int*)malloc(sizeof(int) * (n + 1));
  char* used = (char*)malloc(n + 1);
  int* outer = (int*)malloc(sizeof(int) * (n + 1));
  double sub[64], picked[8], iu[9], iv[9], imv[9];
  int im[9], iw[9], ip[8];
  char iused[9];
  for (int a = 0; a < nA; ++a) {
    for (int b = 0; b < nB; ++b) {
      for (int k = 0; k < g; ++k)
        for (int l = 0; l < g; ++l) sub[k * g + l] = weight(&rows[a * g + k], b * g + l, p, ds, tok);
      int* pm = perm + ((size_t)a * nB + b) * g;
      if (g == 1) {
        pm[0] = 0;
        picked[0] = sub[0];
      } else {
        hungarian_max(sub, g, pm, iu, iv, imv, im, iw, iused);
        for (int k = 0; k < g; ++k) picked[k] = sub[k * g + pm[k]];
      }
      double f;
      if (p->flags & 1) {
        f = py_sum(picked, g);
      } else {
        f = picked[0];
        for (int k = 1; k < g; ++k)
          if (picked[k] > f) f = picked[k];
      }
      fused[(size_t)a * n + b] = f;
    }
  }
  (void)ip;
  hungarian_max(fused, n, outer, u, v, mv, match, way, used);
  double t = 0.0;
  for (int i = 0; i < R; ++i) assign[i] = -1;
  for (int a = 0; a < nA; ++a) {
    int b = outer[a];
    if (b >= nB) continue;
    int* pm = perm + ((size_t)a * nB + b) * g;
    for (int k = 0; k < g; ++k) {
      int row = a * g + k, col = b * g + pm[k];
      assign[row] = col;
      t += weight(&rows[row], col, p, ds, tok);
    }
  }
  *total = t;
  free(rows);
  free(fused);
  free(perm);
  free(u);
  free(v);
  free(mv);
  free(match);
  free(way);
  free(used);
  free(outer);
  return 0;
}

/* Solve plans [0, n_desc) of a sweep batch; assign at plan.out_off. */
int oc_map_sweep(const void* descs, int n_desc, const void* plans, const uint32_t* alive,
                 const int64_t* tok, int32_t* assign, double* totals, int n_threads) {
  const oc_desc* ds = (const oc_desc*)descs;
  const oc_plan* ps = (const oc_plan*)plans;
#pragma omp parallel for schedule(dynamic, 1) num_threads(n_threads > 0 ? n_threads : 1)
  for (int i = 0; i < n_desc; ++i) {
    const oc_plan* p = &ps[ds[i].plan];
    solve(&ds[i], p, alive, tok, assign + p->out_off, &totals[ds[i].plan]);
  }
  return 0;
}

/* Flat _hungarian_max on one dense n x n matrix (for tests). */
int oc_hungarian(const double* w, int n, int32_t* out) {
  double* u = (double*)malloc(sizeof(double) * (n + 1) * 3);
  int* ib = (int*)malloc(sizeof(int) * (n + 1) * 3);
  char* used = (char*)malloc(n + 1);
  hungarian_max(w, n, ib + 2 * (n + 1), u, u + (n + 1), u + 2 * (n + 1), ib, ib + (n + 1), used);
  for (int i = 0; i < n; ++i) out[i] = ib[2 * (n + 1) + i];
  free(u);
  free(ib);
  free(used);
  return 0;
}
