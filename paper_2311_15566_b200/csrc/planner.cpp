// planner.cpp -- native, bit-exact migration planner and T_mig estimator
// (host C++ inside libspotkm.so).
//
// Restates, with exact integer rationals over one denominator K and the same
// double-precision operation order, the reference's
//   _cover_from_holders  migration.py:149-194
//   derive_transfers     migration.py:201-305
//   memopt_layer_order   migration.py:89-143
//   plan_migration       migration.py:311-384
//   simulate_buffer_usage migration.py:387-401
//   plan_timeline / migration_cost  costmodel.py:189-260
// The plan is the migration executor's (K3) input: it is produced here, on
// the host, and shipped to the GPUs as byte-range copies.
//
// Every interval endpoint is an integer numerator over K (the lcm of all
// interval denominators, computed by the caller).  Every float() the
// reference applies to an exact Fraction is reproduced by rat_to_double(), a
// correctly rounded integer-ratio -> double conversion.

#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <thread>
#include <cmath>
#include <map>
#include <string>
#include <vector>

#include "../../include/spotkm.h"
#include "exact.cuh"

namespace {

thread_local char g_perr[512] = "";

typedef __int128 i128;

// correctly rounded num / den: the value float(Fraction) gives (exact.cuh)
using sk_exact::rat_to_double;

struct Seg {
  int64_t lo, hi;
};

// base minus the union of cuts, cuts in sorted order (domain.py:158-172)
std::vector<Seg> subtract(Seg base, std::vector<Seg> cuts) {
  std::sort(cuts.begin(), cuts.end(), [](const Seg& a, const Seg& b) {
    return a.lo != b.lo ? a.lo < b.lo : a.hi < b.hi;
  });
  std::vector<Seg> pieces{base};
  for (const Seg& c : cuts) {
    std::vector<Seg> nxt;
    for (const Seg& p : pieces) {
      if (c.hi <= p.lo || c.lo >= p.hi) {
        nxt.push_back(p);
        continue;
      }
      if (p.lo < c.lo) nxt.push_back({p.lo, c.lo});
      if (c.hi < p.hi) nxt.push_back({c.hi, p.hi});
    }
    pieces.swap(nxt);
  }
  return pieces;
}

int64_t overlap(int64_t a0, int64_t a1, int64_t b0, int64_t b1) {
  const int64_t lo = a0 > b0 ? a0 : b0, hi = a1 < b1 ? a1 : b1;
  return hi > lo ? hi - lo : 0;
}

struct ModelShard {
  int32_t layer;
  int64_t lo, hi;
};
struct CacheShard {
  int64_t rid;
  int32_t layer;
  int64_t lo, hi, tokens;
};
struct Inventory {
  std::vector<ModelShard> model;
  std::vector<CacheShard> cache;
};

struct Transfer {
  int32_t kind;  // 0 model, 1 cache
  int32_t layer;
  int64_t lo, hi;
  int32_t src, dst;  // gpu indices
  double bytes;
  int64_t rid;  // -1 for model
  int64_t tokens;
};

struct Need {
  int32_t dst, kind, layer;
  Seg piece;
  i128 unit;  // bytes per full interval
  int64_t rid, tokens;
};

struct Planner {
  const sk_mig_input& in;
  int64_t K;
  std::vector<Inventory> have, need;
  // releases in first-seen order
  std::vector<int32_t> layer_rel_layers;                 // first-seen layer order
  std::map<int32_t, std::vector<std::pair<int32_t, double>>> layer_rel;  // layer -> [(inst, bytes)] first-seen
  std::vector<std::pair<int32_t, double>> cache_rel;      // [(inst, bytes)] first-seen
  std::vector<Transfer> model_tr, cache_tr;               // model in generation order (layer-tagged)
  int err = SK_OK;
  int64_t err_lo = 0, err_hi = 0;

  explicit Planner(const sk_mig_input& i) : in(i), K(i.K) {}

  static void add_rel(std::vector<std::pair<int32_t, double>>& v, int32_t inst, double b) {
    for (auto& e : v)
      if (e.first == inst) {
        e.second = e.second + b;
        return;
      }
    v.push_back({inst, 0.0 + b});
  }

  void load_inventories() {
    const int G = in.n_gpus;
    have.resize(G);
    need.resize(G);
    for (int g = 0; g < G; ++g) {
      for (int s = in.model_ptr[g]; s < in.model_ptr[g + 1]; ++s)
        have[g].model.push_back({(int32_t)in.model_shards[3 * (size_t)s], in.model_shards[3 * (size_t)s + 1],
                                 in.model_shards[3 * (size_t)s + 2]});
      for (int s = in.cache_ptr[g]; s < in.cache_ptr[g + 1]; ++s) {
        const int64_t* c = in.cache_shards + 5 * (size_t)s;
        have[g].cache.push_back({c[0], (int32_t)c[1], c[2], c[3], c[4]});
      }
      const int pos = in.gpu_pos[g];
      if (pos < 0) continue;
      // required_context_with_cache (mapping.py:155-169)
      const int m = pos % in.M, st = (pos / in.M) % in.P, d = pos / (in.M * in.P) + 1;
      const int q = in.L / in.P, r = in.L % in.P;
      const int l0 = st * q + (st < r ? st : r), l1 = l0 + q + (st < r ? 1 : 0);
      const int64_t w = K / in.M, lo = m * w, hi = lo + w;
      for (int l = l0; l < l1; ++l) need[g].model.push_back({l, lo, hi});
      if (in.inh_ptr && d <= in.D) {
        for (int k = in.inh_ptr[d]; k < in.inh_ptr[d + 1]; ++k) {
          const int64_t rid = in.inh_items[2 * k], tok = in.inh_items[2 * k + 1];
          if (tok <= 0) continue;
          for (int l = l0; l < l1; ++l) need[g].cache.push_back({rid, l, lo, hi, tok});
        }
      }
    }
  }

  // _cover_from_holders (migration.py:149-194)
  struct Holder {
    int32_t gpu;
    std::vector<Seg> ivs;
  };

  bool cover(Seg piece, const std::vector<Holder>& holders, int32_t dst, std::vector<double>& load,
             i128 unit, double budget, std::vector<std::pair<int32_t, Seg>>& out) {
    const int32_t dinst = in.gpu_inst[dst];
    Seg seg = piece;
    while (true) {
      const int64_t start = seg.lo;
      bool found = false;
      int k_remote = 0, k_np = 0, k_nat = 0, k_loc = 0;
      double k_cur = 0.0, k_negend = 0.0;
      int32_t b_gpu = -1;
      int64_t b_end = 0;
      for (const Holder& h : holders) {
        if (h.gpu == dst) continue;
        const int32_t ginst = in.gpu_inst[h.gpu];
        for (const Seg& iv : h.ivs) {
          if (!(iv.lo <= start && start < iv.hi)) continue;
          const int64_t end = iv.hi < seg.hi ? iv.hi : seg.hi;
          const int remote = ginst != dinst;
          const double cur = load[ginst];
          bool pref = false;
          if (in.inst_departing[ginst]) {
            const double x = rat_to_double((i128)(end - start) * unit, K);
            pref = cur + x <= budget + 1e-6;
          }
          const int np = pref ? 0 : 1;
          const double ck = remote ? cur : 0.0;
          const int nat = in.inst_natrank[ginst], loc = in.gpu_local[h.gpu];
          const double negend = -rat_to_double((i128)end, K);
          bool better;
          if (!found) {
            better = true;
          } else if (remote != k_remote) {
            better = remote < k_remote;
          } else if (np != k_np) {
            better = np < k_np;
          } else if (ck != k_cur) {
            better = ck < k_cur;
          } else if (nat != k_nat) {
            better = nat < k_nat;
          } else if (loc != k_loc) {
            better = loc < k_loc;
          } else {
            better = negend < k_negend;
          }
          if (better) {
            found = true;
            k_remote = remote;
            k_np = np;
            k_cur = ck;
            k_nat = nat;
            k_loc = loc;
            k_negend = negend;
            b_gpu = h.gpu;
            b_end = end;
          }
        }
      }
      if (!found) {
        err = SK_ENOSOURCE;
        err_lo = start;
        err_hi = seg.hi;
        return false;
      }
      out.push_back({b_gpu, {start, b_end}});
      const int32_t binst = in.gpu_inst[b_gpu];
      if (binst != dinst) load[binst] = load[binst] + rat_to_double((i128)(b_end - start) * unit, K);
      if (b_end < seg.hi)
        seg = {b_end, seg.hi};
      else
        break;
    }
    return true;
  }

  // derive_transfers (migration.py:201-305)
  bool derive() {
    const int G = in.n_gpus;
    // holders (gpu order, shard order)
    std::map<int32_t, std::vector<Holder>> mh;
    std::map<std::pair<int64_t, int32_t>, std::vector<std::pair<int32_t, std::pair<Seg, int64_t>>>> ch;
    for (int g = 0; g < G; ++g) {
      for (const ModelShard& s : have[g].model) mh[s.layer].push_back({g, {{s.lo, s.hi}}});
      for (const CacheShard& c : have[g].cache) ch[{c.rid, c.layer}].push_back({g, {{c.lo, c.hi}, c.tokens}});
    }
    std::vector<Need> needs;
    std::vector<double> incoming(in.n_inst, 0.0);
    std::vector<char> seen_in(in.n_inst, 0);
    for (int g = 0; g < G; ++g) {
      const int32_t inst = in.gpu_inst[g];
      for (const ModelShard& s : need[g].model) {
        std::vector<Seg> cuts;
        for (const ModelShard& h : have[g].model)
          if (h.layer == s.layer) cuts.push_back({h.lo, h.hi});
        for (const Seg& p : subtract({s.lo, s.hi}, cuts)) {
          needs.push_back({g, 0, s.layer, p, (i128)in.bpl, -1, 0});
          incoming[inst] = incoming[inst] + rat_to_double((i128)(p.hi - p.lo) * in.bpl, K);
          seen_in[inst] = 1;
        }
      }
      for (const CacheShard& c : need[g].cache) {
        std::vector<Seg> own;
        for (const CacheShard& h : have[g].cache)
          if (h.rid == c.rid && h.layer == c.layer && h.tokens >= c.tokens) own.push_back({h.lo, h.hi});
        const i128 unit = (i128)in.kv * c.tokens;
        for (const Seg& p : subtract({c.lo, c.hi}, own)) {
          needs.push_back({g, 1, c.layer, p, unit, c.rid, c.tokens});
          incoming[inst] = incoming[inst] + rat_to_double((i128)(p.hi - p.lo) * unit, K);
          seen_in[inst] = 1;
        }
      }
    }
    double budget = 0.0;
    bool any = false;
    for (int i = 0; i < in.n_inst; ++i)
      if (seen_in[i]) {
        if (!any || incoming[i] > budget) budget = incoming[i];
        any = true;
      }
    std::vector<double> load(in.n_inst, 0.0);
    std::vector<std::pair<int32_t, Seg>> covers;
    for (const Need& nd : needs) {
      std::vector<Holder> holders;
      if (nd.kind == 0) {
        auto it = mh.find(nd.layer);
        if (it != mh.end()) holders = it->second;
      } else {
        auto it = ch.find({nd.rid, nd.layer});
        if (it != ch.end())
          for (auto& e : it->second) {
            Holder h{e.first, {}};
            if (e.second.second >= nd.tokens) h.ivs.push_back(e.second.first);
            holders.push_back(h);
          }
      }
      covers.clear();
      if (!cover(nd.piece, holders, nd.dst, load, nd.unit, budget, covers)) return false;
      for (auto& cv : covers) {
        Transfer t{nd.kind, nd.layer, cv.second.lo, cv.second.hi, cv.first, nd.dst,
                   rat_to_double((i128)(cv.second.hi - cv.second.lo) * nd.unit, K),
                   nd.kind ? nd.rid : -1, nd.kind ? nd.tokens : 0};
        (nd.kind == 0 ? model_tr : cache_tr).push_back(t);
      }
    }
    // releases
    for (int g = 0; g < G; ++g) {
      const int32_t inst = in.gpu_inst[g];
      for (const ModelShard& h : have[g].model) {
        int64_t kept = 0;
        for (const ModelShard& n : need[g].model)
          if (n.layer == h.layer) kept += overlap(h.lo, h.hi, n.lo, n.hi);
        const i128 ex = (i128)((h.hi - h.lo) - kept) * in.bpl;
        const double extra = ex > 0 ? rat_to_double(ex, K) : (ex < 0 ? -rat_to_double(-ex, K) : 0.0);
        if (extra > 0) {
          auto it = layer_rel.find(h.layer);
          if (it == layer_rel.end()) {
            layer_rel_layers.push_back(h.layer);
            it = layer_rel.emplace(h.layer, std::vector<std::pair<int32_t, double>>{}).first;
          }
          add_rel(it->second, inst, extra);
        }
      }
      for (const CacheShard& h : have[g].cache) {
        const i128 held = (i128)(h.hi - h.lo) * h.tokens;
        i128 kept = 0;
        for (const CacheShard& n : need[g].cache)
          if (n.rid == h.rid && n.layer == h.layer)
            kept += (i128)overlap(h.lo, h.hi, n.lo, n.hi) * (h.tokens < n.tokens ? h.tokens : n.tokens);
        const i128 ex = (held - kept) * in.kv;
        const double extra = ex > 0 ? rat_to_double(ex, K) : (ex < 0 ? -rat_to_double(-ex, K) : 0.0);
        if (extra > 0) add_rel(cache_rel, inst, extra);
      }
    }
    return true;
  }
};

// memopt_layer_order (migration.py:89-143); traffic per layer 0..L-1
struct Traffic {
  std::vector<std::pair<int32_t, double>> incoming, freed;  // insertion order
};

double peak_if_applied(const std::vector<double>& usage, const std::vector<char>& present,
                       const Traffic& t) {
  double peak = 0.0;
  bool any = false;
  for (size_t i = 0; i < usage.size(); ++i)
    if (present[i]) {
      if (!any || usage[i] > peak) peak = usage[i];
      any = true;
    }
  if (!any) peak = 0.0;
  for (auto& e : t.incoming) {
    const double x = (present[e.first] ? usage[e.first] : 0.0) + e.second;
    if (x > peak) peak = x;
  }
  return peak;
}

void apply(std::vector<double>& usage, std::vector<char>& present, const Traffic& t) {
  for (auto& e : t.incoming) {
    usage[e.first] = (present[e.first] ? usage[e.first] : 0.0) + e.second;
    present[e.first] = 1;
  }
  for (auto& e : t.freed) {
    usage[e.first] = (present[e.first] ? usage[e.first] : 0.0) - e.second;
    present[e.first] = 1;
  }
}

double order_peak(const std::vector<int>& order, const std::vector<Traffic>& tr, int n_inst) {
  std::vector<double> usage(n_inst, 0.0);
  std::vector<char> present(n_inst, 0);
  double peak = 0.0;
  for (int l : order) {
    const double p = peak_if_applied(usage, present, tr[l]);
    if (p > peak) peak = p;
    apply(usage, present, tr[l]);
  }
  return peak;
}

std::vector<int> memopt(const std::vector<Traffic>& tr, bool has_umax, double umax, int n_inst) {
  const int L = (int)tr.size();
  std::vector<double> usage(n_inst, 0.0);
  std::vector<char> present(n_inst, 0);
  std::vector<int> order, deferred;
  for (int l = 0; l < L; ++l) {
    if (!has_umax || peak_if_applied(usage, present, tr[l]) <= umax) {
      apply(usage, present, tr[l]);
      order.push_back(l);
    } else {
      deferred.push_back(l);
    }
  }
  while (!deferred.empty()) {
    size_t bi = 0;
    double bp = 0.0;
    for (size_t i = 0; i < deferred.size(); ++i) {
      const double p = peak_if_applied(usage, present, tr[deferred[i]]);
      if (i == 0 || p < bp || (p == bp && deferred[i] < deferred[bi])) {
        bp = p;
        bi = i;
      }
    }
    apply(usage, present, tr[deferred[bi]]);
    order.push_back(deferred[bi]);
    deferred.erase(deferred.begin() + bi);
  }
  std::vector<int> idx(L);
  for (int l = 0; l < L; ++l) idx[l] = l;
  if (order != idx && order_peak(order, tr, n_inst) > order_peak(idx, tr, n_inst)) return idx;
  return order;
}

struct Action {
  int32_t kind;  // 0 migrate_cache, 1 migrate_layer, 2 start_stage
  int32_t layer, stage;
  std::vector<int32_t> trs;                      // indices into the transfer table
  std::vector<std::pair<int32_t, double>> rels;  // sorted by instance id string
};

struct Assembled {
  std::vector<Action> actions;
  std::vector<double> peak;  // per instance
};

}  // namespace

struct sk_mig_result {
  std::vector<Transfer> transfers;
  std::vector<sk_mig_action> actions;
  std::vector<int32_t> action_transfers;
  std::vector<sk_mig_release> releases;
  std::vector<double> peak;
  std::vector<sk_mig_release> layer_releases_flat;  // derive mode: (layer in .pad)
  int32_t n_model_transfers = 0;
};

namespace {

Assembled assemble(const sk_mig_input& in, const std::vector<int>& order, const Planner& pl,
                   const std::vector<int32_t>& model_idx_by_layer_start,
                   const std::vector<std::vector<int32_t>>& model_by_layer, int32_t n_model) {
  Assembled A;
  std::vector<std::pair<int32_t, double>> crel = pl.cache_rel;
  auto by_str = [&](const std::pair<int32_t, double>& a, const std::pair<int32_t, double>& b) {
    return in.inst_strrank[a.first] < in.inst_strrank[b.first];
  };
  std::vector<Action> rounds;
  if (!pl.cache_tr.empty() || !crel.empty()) {
    Action a{0, -1, -1, {}, {}};
    for (size_t i = 0; i < pl.cache_tr.size(); ++i) a.trs.push_back(n_model + (int32_t)i);
    std::sort(crel.begin(), crel.end(), by_str);
    a.rels = crel;
    rounds.push_back(a);
  }
  for (int l : order) {
    Action a{1, l, -1, {}, {}};
    if (l < (int)model_by_layer.size()) a.trs = model_by_layer[l];
    auto it = pl.layer_rel.find(l);
    if (it != pl.layer_rel.end()) {
      a.rels = it->second;
      std::sort(a.rels.begin(), a.rels.end(), by_str);
    }
    if (!a.trs.empty() || !a.rels.empty()) rounds.push_back(a);
  }
  (void)model_idx_by_layer_start;
  // stage readiness (migration.py:352-371)
  std::vector<int> ready(in.P + 1, -1);
  for (size_t idx = 0; idx < rounds.size(); ++idx)
    for (int32_t t : rounds[idx].trs) {
      const Transfer& tr = t < n_model ? pl.model_tr[t] : pl.cache_tr[t - n_model];
      const int pos = in.gpu_pos[tr.dst];
      if (pos < 0) continue;
      const int st = (pos / in.M) % in.P + 1;
      if ((int)idx > ready[st]) ready[st] = (int)idx;
    }
  for (int p = 1; p <= in.P; ++p)
    if (ready[p] < 0) A.actions.push_back({2, -1, p, {}, {}});
  for (size_t idx = 0; idx < rounds.size(); ++idx) {
    A.actions.push_back(rounds[idx]);
    for (int p = 1; p <= in.P; ++p)
      if (ready[p] == (int)idx) A.actions.push_back({2, -1, p, {}, {}});
  }
  // simulate_buffer_usage (migration.py:387-401)
  std::vector<double> usage(in.n_inst, 0.0);
  std::vector<double> peaks(in.n_inst, 0.0);
  for (const Action& a : A.actions) {
    std::vector<char> touched(in.n_inst, 0);
    for (int32_t t : a.trs) {
      const Transfer& tr = t < n_model ? pl.model_tr[t] : pl.cache_tr[t - n_model];
      const int32_t inst = in.gpu_inst[tr.dst];
      usage[inst] = usage[inst] + tr.bytes;
      touched[inst] = 1;
    }
    for (int i = 0; i < in.n_inst; ++i)
      if (touched[i] && usage[i] > peaks[i]) peaks[i] = usage[i];
    for (auto& r : a.rels) usage[r.first] = usage[r.first] - r.second;
  }
  A.peak = peaks;
  return A;
}

double max_peak(const std::vector<double>& p, const std::vector<char>& present) {
  double m = 0.0;
  bool any = false;
  for (size_t i = 0; i < p.size(); ++i)
    if (present[i]) {
      if (!any || p[i] > m) m = p[i];
      any = true;
    }
  return m;
}

}  // namespace

extern "C" {

int sk_plan_migration(const sk_mig_input* in, int derive_only, sk_mig_result** out) {
  *out = nullptr;
  if (!in || in->K <= 0 || in->M <= 0 || in->P <= 0 || in->D <= 0 || in->K % in->M) {
    snprintf(g_perr, sizeof g_perr, "invalid planner input");
    return SK_EINVAL;
  }
  Planner pl(*in);
  pl.load_inventories();
  if (!pl.derive()) {
    snprintf(g_perr, sizeof g_perr, "%lld %lld", (long long)pl.err_lo, (long long)pl.err_hi);
    return pl.err;
  }
  sk_mig_result* R = new sk_mig_result();
  R->n_model_transfers = (int32_t)pl.model_tr.size();
  R->transfers = pl.model_tr;
  R->transfers.insert(R->transfers.end(), pl.cache_tr.begin(), pl.cache_tr.end());
  if (derive_only) {
    for (int32_t l : pl.layer_rel_layers)
      for (auto& e : pl.layer_rel.at(l)) R->layer_releases_flat.push_back({e.first, l, e.second});
    for (auto& e : pl.cache_rel) R->releases.push_back({e.first, -1, e.second});
    *out = R;
    return SK_OK;
  }
  const int32_t n_model = (int32_t)pl.model_tr.size();
  std::vector<std::vector<int32_t>> by_layer(in->L);
  std::vector<Traffic> traffic(in->L);
  for (int32_t i = 0; i < n_model; ++i) {
    const Transfer& t = pl.model_tr[i];
    if (t.layer >= 0 && t.layer < in->L) {
      by_layer[t.layer].push_back(i);
      Traffic& tr = traffic[t.layer];
      const int32_t inst = in->gpu_inst[t.dst];
      bool hit = false;
      for (auto& e : tr.incoming)
        if (e.first == inst) {
          e.second = e.second + t.bytes;
          hit = true;
        }
      if (!hit) tr.incoming.push_back({inst, 0.0 + t.bytes});
    }
  }
  for (int l = 0; l < in->L; ++l) {
    auto it = pl.layer_rel.find(l);
    if (it != pl.layer_rel.end())
      for (auto& e : it->second) traffic[l].freed.push_back({e.first, 0.0 + e.second});
  }
  const std::vector<int> order = memopt(traffic, in->has_umax != 0, in->u_max, in->n_inst);
  std::vector<char> present(in->n_inst, 0);
  for (int g = 0; g < in->n_gpus; ++g) present[in->gpu_inst[g]] = 1;
  std::vector<int32_t> unused;
  Assembled plan = assemble(*in, order, pl, unused, by_layer, n_model);
  std::vector<int> idx(in->L);
  for (int l = 0; l < in->L; ++l) idx[l] = l;
  if (order != idx) {
    Assembled naive = assemble(*in, idx, pl, unused, by_layer, n_model);
    if (max_peak(naive.peak, present) < max_peak(plan.peak, present)) plan = naive;
  }
  for (const Action& a : plan.actions) {
    sk_mig_action x;
    x.kind = a.kind;
    x.layer = a.layer;
    x.stage = a.stage;
    x.tr_begin = (int32_t)R->action_transfers.size();
    for (int32_t t : a.trs) R->action_transfers.push_back(t);
    x.tr_end = (int32_t)R->action_transfers.size();
    x.rel_begin = (int32_t)R->releases.size();
    for (auto& r : a.rels) R->releases.push_back({r.first, -1, r.second});
    x.rel_end = (int32_t)R->releases.size();
    R->actions.push_back(x);
  }
  R->peak = plan.peak;
  *out = R;
  return SK_OK;
}

// Many independent plans at once ("host, one thread per
// plan"): a pool of n_threads std::threads takes plans in index order.  Per
// plan: status[i] (sk_status), outs[i] (NULL unless SK_OK), and for
// SK_ENOSOURCE the uncovered piece's numerators in err_range[2i..2i+1].
int sk_plan_migration_many(const sk_mig_input* ins, int n, int derive_only, int n_threads,
                           sk_mig_result** outs, int32_t* status, int64_t* err_range) {
  if (n <= 0) return SK_OK;
  if (n_threads <= 0) n_threads = (int)std::thread::hardware_concurrency();
  if (n_threads <= 0) n_threads = 1;
  if (n_threads > n) n_threads = n;
  std::atomic<int> next(0);
  auto work = [&]() {
    for (int i = next++; i < n; i = next++) {
      outs[i] = nullptr;
      status[i] = sk_plan_migration(&ins[i], derive_only, &outs[i]);
      if (status[i] == SK_ENOSOURCE && err_range) {
        long long lo = 0, hi = 0;
        sscanf(g_perr, "%lld %lld", &lo, &hi);
        err_range[2 * i] = lo;
        err_range[2 * i + 1] = hi;
      }
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < n_threads; ++t) pool.emplace_back(work);
  work();
  for (auto& th : pool) th.join();
  return SK_OK;
}

int sk_mig_counts(const sk_mig_result* r, int64_t* counts) {
  counts[0] = (int64_t)r->transfers.size();
  counts[1] = (int64_t)r->actions.size();
  counts[2] = (int64_t)r->action_transfers.size();
  counts[3] = (int64_t)r->releases.size();
  counts[4] = (int64_t)r->peak.size();
  counts[5] = (int64_t)r->layer_releases_flat.size();
  counts[6] = (int64_t)r->n_model_transfers;
  return SK_OK;
}

int sk_mig_export(const sk_mig_result* r, sk_mig_transfer* transfers, sk_mig_action* actions,
                  int32_t* action_transfers, sk_mig_release* releases, double* peak,
                  sk_mig_release* layer_releases) {
  for (size_t i = 0; i < r->transfers.size(); ++i) {
    const Transfer& t = r->transfers[i];
    transfers[i] = {t.kind, t.layer, t.lo, t.hi, t.src, t.dst, t.bytes, t.rid, t.tokens};
  }
  if (actions && !r->actions.empty()) memcpy(actions, r->actions.data(), r->actions.size() * sizeof(sk_mig_action));
  if (action_transfers && !r->action_transfers.empty())
    memcpy(action_transfers, r->action_transfers.data(), r->action_transfers.size() * 4);
  if (releases && !r->releases.empty())
    memcpy(releases, r->releases.data(), r->releases.size() * sizeof(sk_mig_release));
  if (peak && !r->peak.empty()) memcpy(peak, r->peak.data(), r->peak.size() * 8);
  if (layer_releases && !r->layer_releases_flat.empty())
    memcpy(layer_releases, r->layer_releases_flat.data(),
           r->layer_releases_flat.size() * sizeof(sk_mig_release));
  return SK_OK;
}

void sk_mig_free(sk_mig_result* r) { delete r; }

const char* sk_planner_error(void) { return g_perr; }

// plan_timeline / migration_cost (costmodel.py:189-260) over a flattened plan:
// transfers carry instance indices; `ends` receives one completion time per
// action.  release: per-instance earliest start (has_release[i] = 0 -> start).
int sk_plan_timeline(const sk_timeline_input* t, double* ends) {
  std::vector<double> out_free(t->n_inst, 0.0), in_free(t->n_inst, 0.0);
  std::vector<char> has_out(t->n_inst, 0), has_in(t->n_inst, 0);
  double prev = t->start;
  for (int a = 0; a < t->n_actions; ++a) {
    double end = prev;
    bool moved = false;
    for (int k = t->action_ptr[a]; k < t->action_ptr[a + 1]; ++k) {
      const int s = t->src_inst[k], d = t->dst_inst[k];
      if (s == d) continue;
      moved = true;
      const double so = has_out[s] ? out_free[s]
                                   : (t->has_release && t->has_release[s] ? t->release[s] : t->start);
      const double di = has_in[d] ? in_free[d]
                                  : (t->has_release && t->has_release[d] ? t->release[d] : t->start);
      const double begin = so > di ? so : di;  // max(out, in)
      const double fin = begin + t->bytes[k] / t->bandwidth;
      out_free[s] = fin;
      has_out[s] = 1;
      in_free[d] = fin;
      has_in[d] = 1;
      if (fin > end) end = fin;
    }
    if (moved) end += t->latency;
    ends[a] = end > prev ? end : prev;
    prev = ends[a];
  }
  return SK_OK;
}

// migration_cost (costmodel.py:231-260): the timeline above, then the full
// duration or, with progressive start, the worst stage-ready constraint over
// the start_stage actions taken in stable stage order
int sk_migration_cost(const sk_timeline_input* t, const int32_t* act_stage, double step, int32_t progressive,
                      double* cost) {
  std::vector<double> ends(t->n_actions > 0 ? t->n_actions : 1, 0.0);
  sk_plan_timeline(t, ends.data());
  const double last = t->n_actions > 0 ? ends[t->n_actions - 1] : t->start;
  const double total = (last > t->start ? last : t->start) - t->start;
  std::vector<std::pair<int32_t, double>> starts;
  if (progressive)
    for (int a = 0; a < t->n_actions; ++a)
      if (act_stage[a] >= 0) starts.push_back({act_stage[a], ends[a]});
  if (starts.empty()) {
    *cost = total;
    return SK_OK;
  }
  std::stable_sort(starts.begin(), starts.end(),
                   [](const std::pair<int32_t, double>& x, const std::pair<int32_t, double>& y) {
                     return x.first < y.first;
                   });
  double stall = 0.0;
  for (size_t o = 0; o < starts.size(); ++o) {
    const double v = starts[o].second - t->start - (double)o * step;
    if (v > stall) stall = v;  // max(stall, v): the first maximum is kept
  }
  *cost = stall > 0.0 ? stall : 0.0;
  return SK_OK;
}

// simulate_buffer_usage (migration.py:387-401): per-instance usage replay.
// Instances 0..n_seed-1 are the old layout's (in its order); `order` receives
// the instances in the result dict's insertion order, *n_order their count.
int sk_simulate_buffer_usage(int32_t n_inst, int32_t n_seed, int32_t n_actions, const int32_t* tr_ptr,
                             const int32_t* tr_dst, const double* tr_bytes, const int32_t* rel_ptr,
                             const int32_t* rel_inst, const double* rel_bytes, const int32_t* name_rank,
                             double* peaks, int32_t* order, int32_t* n_order) {
  std::vector<double> usage(n_inst, 0.0);
  std::vector<char> in_peaks(n_inst, 0);
  int32_t no = 0;
  for (int i = 0; i < n_seed; ++i) {
    peaks[i] = 0.0;
    in_peaks[i] = 1;
    order[no++] = i;
  }
  for (int a = 0; a < n_actions; ++a) {
    std::vector<int32_t> touched;
    for (int k = tr_ptr[a]; k < tr_ptr[a + 1]; ++k) {
      usage[tr_dst[k]] = usage[tr_dst[k]] + tr_bytes[k];
      touched.push_back(tr_dst[k]);
    }
    // sorted({t.dst[0] ...}): by instance name (name_rank = rank of the string)
    std::sort(touched.begin(), touched.end(),
              [&](int32_t x, int32_t y) { return name_rank[x] < name_rank[y]; });
    touched.erase(std::unique(touched.begin(), touched.end()), touched.end());
    for (int32_t i : touched) {
      if (!in_peaks[i]) {
        in_peaks[i] = 1;
        peaks[i] = usage[i];  // max(peaks.get(inst, 0.0), usage) with 0.0 first
        if (!(usage[i] > 0.0)) peaks[i] = 0.0;
        order[no++] = i;
      } else if (usage[i] > peaks[i]) {
        peaks[i] = usage[i];
      }
    }
    for (int k = rel_ptr[a]; k < rel_ptr[a + 1]; ++k) usage[rel_inst[k]] = usage[rel_inst[k]] - rel_bytes[k];
  }
  *n_order = no;
  return SK_OK;
}

int sk_memopt_order(int32_t n_layers, int32_t n_inst, const int32_t* in_ptr, const int32_t* in_inst,
                    const double* in_bytes, const int32_t* fr_ptr, const int32_t* fr_inst,
                    const double* fr_bytes, int32_t has_umax, double u_max, int32_t* order) {
  std::vector<Traffic> tr(n_layers);
  for (int l = 0; l < n_layers; ++l) {
    for (int k = in_ptr[l]; k < in_ptr[l + 1]; ++k) tr[l].incoming.push_back({in_inst[k], in_bytes[k]});
    for (int k = fr_ptr[l]; k < fr_ptr[l + 1]; ++k) tr[l].freed.push_back({fr_inst[k], fr_bytes[k]});
  }
  const std::vector<int> o = memopt(tr, has_umax != 0, u_max, n_inst);
  for (int l = 0; l < n_layers; ++l) order[l] = o[l];
  return SK_OK;
}

double sk_rat_to_double(int64_t num_hi, uint64_t num_lo, int64_t den) {
  const i128 num = ((i128)num_hi << 64) | (i128)num_lo;
  return rat_to_double(num, den);
}

}  // extern "C"
