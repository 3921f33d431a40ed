// hostpack.cpp -- CPython extension: flatten the caller's Python inventories
// (tuples of Fractions, the reference's ContextInventory layout,
// domain.py:175-220) into the integer arrays the C ABI consumes, without a
// Python-level loop per shard.
//
//   common_denominator(invs, M)                 -> K
//   pack_rows(invs, K, bpl, kv, need[, wide])   -> (row_ptr bytes, segments bytes, wide)
//       the segment encoding of pack.py (closed form of overlap_bytes,
//       domain.py:299-320, on required_context_with_cache, mapping.py:155-169)
//   flatten(invs, K, rid_index, rid_names)      -> (model_ptr, model_shards, cache_ptr, cache_shards)
//       the planner input of include/spotkm.h sk_mig_input (rid strings interned
//       into rid_index / rid_names)
//
// Exactness: all interval endpoints become integer numerators over K; the
// numerator bound is checked exactly with 128-bit integers: < 2^53 (and
// K <= 2^31 - 1) keeps the regular sk_segment encoding, anything below 2^127
// (K < 2^62) is emitted as sk_segment_wide for the general-range kernels.

#define PY_SSIZE_T_CLEAN
#include <Python.h>

#include <stdint.h>
#include <string.h>

#include <map>
#include <numeric>
#include <string>
#include <tuple>
#include <unordered_map>
#include <vector>

namespace {

typedef __int128 i128;

// y# with a NULL pointer builds None; empty buffers must stay bytes
template <typename T>
const char* bptr(const std::vector<T>& v) {
  static const char empty = 0;
  return v.empty() ? &empty : reinterpret_cast<const char*>(v.data());
}

struct Seg {
  int32_t l0, l1, a, b, pipe, reserved;
  int64_t unit;
};
static_assert(sizeof(Seg) == 32, "sk_segment layout");

// sk_segment_wide (include/spotkm.h): two sk_segment slots
struct WideSeg {
  int32_t l0, l1, pipe, reserved;
  int64_t a, b, unit;
  int64_t reserved2[3];
};
static_assert(sizeof(WideSeg) == 64, "sk_segment_wide layout");

// a segment while packing: 64-bit endpoints and units
struct RunSeg {
  int32_t l0, l1, pipe;
  int64_t a, b, unit;
};

const int64_t kKMax = (int64_t)1 << 62;   // general-range plans: K < 2^62
const int64_t kKRegular = 0x7fffffffLL;   // regular plans: K <= 2^31 - 1

PyObject* g_num = nullptr;  // interned "numerator"
PyObject* g_num_slot = nullptr;  // interned "_numerator"
PyObject* g_den_slot = nullptr;  // interned "_denominator"
PyObject* g_den = nullptr;  // interned "denominator"

bool as_i64(PyObject* o, int64_t* out) {
  int overflow = 0;
  long long v = PyLong_AsLongLongAndOverflow(o, &overflow);
  if (overflow || (v == -1 && PyErr_Occurred())) {
    if (!PyErr_Occurred()) PyErr_SetString(PyExc_OverflowError, "integer out of int64 range");
    return false;
  }
  *out = v;
  return true;
}

// numerator / denominator of a Fraction (or int), memoised by object identity:
// inventories share their endpoint objects
struct FracCache {
  std::unordered_map<PyObject*, std::pair<int64_t, int64_t>> m;
  bool get(PyObject* x, int64_t* n, int64_t* d) {
    auto it = m.find(x);
    if (it != m.end()) {
      *n = it->second.first;
      *d = it->second.second;
      return true;
    }
    // fractions.Fraction keeps its value in the _numerator / _denominator
    // slots; reading them skips the Python-level properties (ints and other
    // rationals fall back to numerator / denominator)
    PyObject* pn = PyObject_GetAttr(x, g_num_slot);
    PyObject* pd = pn ? PyObject_GetAttr(x, g_den_slot) : nullptr;
    if (!pn || !pd) {
      PyErr_Clear();
      Py_XDECREF(pn);
      pn = PyObject_GetAttr(x, g_num);
      if (!pn) return false;
      pd = PyObject_GetAttr(x, g_den);
    }
    if (!pd) {
      Py_DECREF(pn);
      return false;
    }
    const bool ok = as_i64(pn, n) && as_i64(pd, d);
    Py_DECREF(pn);
    Py_DECREF(pd);
    if (!ok) return false;
    m.emplace(x, std::make_pair(*n, *d));
    return true;
  }
  bool scaled(PyObject* x, int64_t K, int64_t* v) {
    int64_t n, d;
    if (!get(x, &n, &d)) return false;
    *v = n * (K / d);
    return true;
  }
};

// fetch attribute `name` of obj as a fast sequence (tuple/list)
PyObject* seq_attr(PyObject* obj, const char* name) {
  PyObject* a = PyObject_GetAttrString(obj, name);
  if (!a) return nullptr;
  PyObject* s = PySequence_Fast(a, "inventory shards must be a sequence");
  Py_DECREF(a);
  return s;
}

PyObject* py_common_denominator(PyObject*, PyObject* args) {
  PyObject* invs;
  long long M;
  if (!PyArg_ParseTuple(args, "OL", &invs, &M)) return nullptr;
  PyObject* seq = PySequence_Fast(invs, "inventories must be a sequence");
  if (!seq) return nullptr;
  FracCache fc;
  int64_t K = M;
  const Py_ssize_t n = PySequence_Fast_GET_SIZE(seq);
  for (Py_ssize_t i = 0; i < n; ++i) {
    PyObject* inv = PySequence_Fast_GET_ITEM(seq, i);
    for (int part = 0; part < 2; ++part) {
      PyObject* sh = seq_attr(inv, part == 0 ? "model_shards" : "cache_shards");
      if (!sh) {
        Py_DECREF(seq);
        return nullptr;
      }
      const Py_ssize_t m = PySequence_Fast_GET_SIZE(sh);
      const int lo_i = part == 0 ? 1 : 2;
      for (Py_ssize_t k = 0; k < m; ++k) {
        PyObject* t = PySequence_Fast_GET_ITEM(sh, k);
        for (int e = 0; e < 2; ++e) {
          PyObject* x = PySequence_GetItem(t, lo_i + e);
          if (!x) {
            Py_DECREF(sh);
            Py_DECREF(seq);
            return nullptr;
          }
          int64_t nu, de;
          const bool ok = fc.get(x, &nu, &de);
          Py_DECREF(x);
          if (!ok) {
            Py_DECREF(sh);
            Py_DECREF(seq);
            return nullptr;
          }
          const i128 l = (i128)(K / std::gcd(K, de)) * de;
          if (de <= 0 || l >= (i128)kKMax) {
            Py_DECREF(sh);
            Py_DECREF(seq);
            PyErr_SetString(PyExc_ValueError, "common interval denominator exceeds 2^62");
            return nullptr;
          }
          K = (int64_t)l;
        }
      }
      Py_DECREF(sh);
    }
  }
  Py_DECREF(seq);
  return PyLong_FromLongLong(K);
}

// need: dict rid -> list[(d_new, tokens)]
typedef std::unordered_map<std::string, std::vector<std::pair<int32_t, int64_t>>> NeedMap;

bool load_need(PyObject* need, NeedMap* out) {
  if (need == Py_None) return true;
  PyObject *key, *val;
  Py_ssize_t pos = 0;
  while (PyDict_Next(need, &pos, &key, &val)) {
    Py_ssize_t len;
    const char* s = PyUnicode_AsUTF8AndSize(key, &len);
    if (!s) return false;
    auto& v = (*out)[std::string(s, len)];
    PyObject* seq = PySequence_Fast(val, "need entries must be a sequence");
    if (!seq) return false;
    for (Py_ssize_t i = 0; i < PySequence_Fast_GET_SIZE(seq); ++i) {
      PyObject* pr = PySequence_Fast_GET_ITEM(seq, i);
      PyObject* d = PySequence_GetItem(pr, 0);
      PyObject* t = PySequence_GetItem(pr, 1);
      int64_t dv = 0, tv = 0;
      const bool ok = d && t && as_i64(d, &dv) && as_i64(t, &tv);
      Py_XDECREF(d);
      Py_XDECREF(t);
      if (!ok) {
        Py_DECREF(seq);
        return false;
      }
      // pipeline 0 would read as a model segment; callers filter the range
      // 1..D (pack.need_tokens), this keeps the encoding sound regardless
      if (dv >= 1 && dv <= 0x7fffffffLL) v.emplace_back((int32_t)dv, tv);
    }
    Py_DECREF(seq);
  }
  return true;
}

PyObject* py_pack_rows(PyObject*, PyObject* args) {
  PyObject *invs, *need_obj;
  long long K, bpl, kv;
  int force_wide = 0;
  if (!PyArg_ParseTuple(args, "OLLLO|p", &invs, &K, &bpl, &kv, &need_obj, &force_wide)) return nullptr;
  NeedMap need;
  if (!load_need(need_obj, &need)) return nullptr;
  PyObject* seq = PySequence_Fast(invs, "inventories must be a sequence");
  if (!seq) return nullptr;
  FracCache fc;
  const Py_ssize_t R = PySequence_Fast_GET_SIZE(seq);
  std::vector<int32_t> row_ptr(R + 1, 0);
  std::vector<RunSeg> segs;
  bool wide = force_wide != 0 || K > kKRegular;
  const i128 limit53 = (i128)1 << 53;
  const i128 limit127 = (((i128)1 << 126) - 1) * 2 + 1;  // 2^127 - 1
  auto range_error = [&](const char* what) {
    Py_DECREF(seq);
    PyErr_SetString(PyExc_ValueError, what);
    return (PyObject*)nullptr;
  };
  for (Py_ssize_t r = 0; r < R; ++r) {
    PyObject* inv = PySequence_Fast_GET_ITEM(seq, r);
    // model: (a, b, layer) -> multiplicity
    std::map<std::tuple<int64_t, int64_t, int64_t>, int64_t> model;
    PyObject* ms = seq_attr(inv, "model_shards");
    if (!ms) goto fail;
    for (Py_ssize_t k = 0; k < PySequence_Fast_GET_SIZE(ms); ++k) {
      PyObject* t = PySequence_Fast_GET_ITEM(ms, k);
      PyObject *pl = PySequence_GetItem(t, 0), *plo = PySequence_GetItem(t, 1), *phi = PySequence_GetItem(t, 2);
      int64_t layer = 0, a = 0, b = 0;
      const bool ok = pl && plo && phi && as_i64(pl, &layer) && fc.scaled(plo, K, &a) && fc.scaled(phi, K, &b);
      Py_XDECREF(pl);
      Py_XDECREF(plo);
      Py_XDECREF(phi);
      if (!ok) {
        Py_DECREF(ms);
        goto fail;
      }
      model[std::make_tuple(a, b, layer)] += 1;
    }
    Py_DECREF(ms);
    {
      const size_t first = segs.size();
      // runs of consecutive layers with equal (a, b, multiplicity)
      for (auto& kvp : model) {
        const int64_t a = std::get<0>(kvp.first), b = std::get<1>(kvp.first), layer = std::get<2>(kvp.first);
        const i128 u = (i128)bpl * kvp.second;
        if (u > (i128)INT64_MAX) return range_error("segment bytes exceed 2^63: outside the exact range");
        const int64_t unit = (int64_t)u;
        if (segs.size() > first) {
          RunSeg& sg = segs.back();
          if (sg.pipe == 0 && sg.a == a && sg.b == b && sg.unit == unit && sg.l1 == layer) {
            sg.l1 = (int32_t)(layer + 1);
            continue;
          }
        }
        segs.push_back({(int32_t)layer, (int32_t)(layer + 1), 0, a, b, unit});
      }
      if (!need.empty()) {
        std::map<std::tuple<int64_t, int64_t, int32_t, int64_t>, int64_t> cache;
        PyObject* cs = seq_attr(inv, "cache_shards");
        if (!cs) goto fail;
        for (Py_ssize_t k = 0; k < PySequence_Fast_GET_SIZE(cs); ++k) {
          PyObject* t = PySequence_Fast_GET_ITEM(cs, k);
          PyObject* prid = PySequence_GetItem(t, 0);
          if (!prid) {
            Py_DECREF(cs);
            goto fail;
          }
          Py_ssize_t len;
          const char* str = PyUnicode_AsUTF8AndSize(prid, &len);
          if (!str) {
            Py_DECREF(prid);
            Py_DECREF(cs);
            goto fail;
          }
          auto it = need.find(std::string(str, len));
          Py_DECREF(prid);
          if (it == need.end() || it->second.empty()) continue;
          PyObject *pl = PySequence_GetItem(t, 1), *plo = PySequence_GetItem(t, 2),
                   *phi = PySequence_GetItem(t, 3), *ptok = PySequence_GetItem(t, 4);
          int64_t layer = 0, a = 0, b = 0, tok = 0;
          const bool ok = pl && plo && phi && ptok && as_i64(pl, &layer) && fc.scaled(plo, K, &a) &&
                          fc.scaled(phi, K, &b) && as_i64(ptok, &tok);
          Py_XDECREF(pl);
          Py_XDECREF(plo);
          Py_XDECREF(phi);
          Py_XDECREF(ptok);
          if (!ok) {
            Py_DECREF(cs);
            goto fail;
          }
          for (auto& e : it->second) cache[std::make_tuple(a, b, e.first, layer)] += tok < e.second ? tok : e.second;
        }
        Py_DECREF(cs);
        const size_t cfirst = segs.size();
        for (auto& kvp : cache) {
          const int64_t a = std::get<0>(kvp.first), b = std::get<1>(kvp.first), layer = std::get<3>(kvp.first);
          const int32_t d = std::get<2>(kvp.first);
          const int64_t tsum = kvp.second;
          const i128 u = (i128)kv * tsum;
          if (u > (i128)INT64_MAX) return range_error("segment bytes exceed 2^63: outside the exact range");
          const int64_t unit = (int64_t)u;
          if (segs.size() > cfirst) {
            RunSeg& sg = segs.back();
            if (sg.pipe == d && sg.a == a && sg.b == b && sg.unit == unit && sg.l1 == layer && tsum != 0) {
              sg.l1 = (int32_t)(layer + 1);
              continue;
            }
          }
          if (tsum == 0) continue;
          segs.push_back({(int32_t)layer, (int32_t)(layer + 1), d, a, b, unit});
        }
      }
      // every W numerator of this row is <= the sum of its segments' spans:
      // < 2^53 keeps the regular (64-bit) encoding, else 128-bit numerators
      i128 bound = 0;
      for (size_t i = first; i < segs.size(); ++i) {
        const i128 span = (i128)(segs[i].l1 - segs[i].l0) * (segs[i].b - segs[i].a);
        if (span != 0 && (i128)segs[i].unit > limit127 / span) return range_error("edge-weight numerator may exceed 2^127: outside the exact range");
        const i128 term = span * segs[i].unit;
        if (bound > limit127 - term) return range_error("edge-weight numerator may exceed 2^127: outside the exact range");
        bound += term;
      }
      if (bound >= limit53) wide = true;
    }
    row_ptr[r + 1] = (int32_t)segs.size();
  }
  Py_DECREF(seq);
  if (!wide) {
    std::vector<Seg> out(segs.size());  // (scoped: the gotos above jump past it)
    for (size_t i = 0; i < segs.size(); ++i)
      out[i] = {segs[i].l0, segs[i].l1, (int32_t)segs[i].a, (int32_t)segs[i].b, segs[i].pipe, 0, segs[i].unit};
    return Py_BuildValue("(y#y#O)", bptr(row_ptr), (Py_ssize_t)(row_ptr.size() * 4), bptr(out),
                         (Py_ssize_t)(out.size() * sizeof(Seg)), Py_False);
  }
  {
    std::vector<WideSeg> out(segs.size());
    for (size_t i = 0; i < segs.size(); ++i)
      out[i] = {segs[i].l0, segs[i].l1, segs[i].pipe, 0, segs[i].a, segs[i].b, segs[i].unit, {0, 0, 0}};
    for (auto& x : row_ptr) x *= 2;  // two sk_segment slots per wide segment
    return Py_BuildValue("(y#y#O)", bptr(row_ptr), (Py_ssize_t)(row_ptr.size() * 4), bptr(out),
                         (Py_ssize_t)(out.size() * sizeof(WideSeg)), Py_True);
  }
fail:
  Py_DECREF(seq);
  return nullptr;
}

PyObject* py_flatten(PyObject*, PyObject* args) {
  PyObject *invs, *rid_index, *rid_names;
  long long K;
  if (!PyArg_ParseTuple(args, "OLO!O!", &invs, &K, &PyDict_Type, &rid_index, &PyList_Type, &rid_names))
    return nullptr;
  PyObject* seq = PySequence_Fast(invs, "inventories must be a sequence");
  if (!seq) return nullptr;
  FracCache fc;
  const Py_ssize_t G = PySequence_Fast_GET_SIZE(seq);
  std::vector<int32_t> mp(G + 1, 0), cp(G + 1, 0);
  std::vector<int64_t> msh, csh;
  for (Py_ssize_t g = 0; g < G; ++g) {
    PyObject* inv = PySequence_Fast_GET_ITEM(seq, g);
    PyObject* ms = seq_attr(inv, "model_shards");
    if (!ms) goto fail;
    for (Py_ssize_t k = 0; k < PySequence_Fast_GET_SIZE(ms); ++k) {
      PyObject* t = PySequence_Fast_GET_ITEM(ms, k);
      PyObject *pl = PySequence_GetItem(t, 0), *plo = PySequence_GetItem(t, 1), *phi = PySequence_GetItem(t, 2);
      int64_t layer = 0, a = 0, b = 0;
      const bool ok = pl && plo && phi && as_i64(pl, &layer) && fc.scaled(plo, K, &a) && fc.scaled(phi, K, &b);
      Py_XDECREF(pl);
      Py_XDECREF(plo);
      Py_XDECREF(phi);
      if (!ok) {
        Py_DECREF(ms);
        goto fail;
      }
      msh.push_back(layer);
      msh.push_back(a);
      msh.push_back(b);
    }
    Py_DECREF(ms);
    mp[g + 1] = (int32_t)(msh.size() / 3);
    PyObject* cs = seq_attr(inv, "cache_shards");
    if (!cs) goto fail;
    for (Py_ssize_t k = 0; k < PySequence_Fast_GET_SIZE(cs); ++k) {
      PyObject* t = PySequence_Fast_GET_ITEM(cs, k);
      PyObject *prid = PySequence_GetItem(t, 0), *pl = PySequence_GetItem(t, 1), *plo = PySequence_GetItem(t, 2),
               *phi = PySequence_GetItem(t, 3), *ptok = PySequence_GetItem(t, 4);
      int64_t layer = 0, a = 0, b = 0, tok = 0, rid = 0;
      bool ok = prid && pl && plo && phi && ptok && as_i64(pl, &layer) && fc.scaled(plo, K, &a) &&
                fc.scaled(phi, K, &b) && as_i64(ptok, &tok);
      if (ok) {
        PyObject* idx = PyDict_GetItemWithError(rid_index, prid);
        if (idx) {
          ok = as_i64(idx, &rid);
        } else if (PyErr_Occurred()) {
          ok = false;
        } else {
          rid = PyList_GET_SIZE(rid_names);
          PyObject* pi = PyLong_FromLongLong(rid);
          ok = pi && PyDict_SetItem(rid_index, prid, pi) == 0 && PyList_Append(rid_names, prid) == 0;
          Py_XDECREF(pi);
        }
      }
      Py_XDECREF(prid);
      Py_XDECREF(pl);
      Py_XDECREF(plo);
      Py_XDECREF(phi);
      Py_XDECREF(ptok);
      if (!ok) {
        Py_DECREF(cs);
        goto fail;
      }
      csh.insert(csh.end(), {rid, layer, a, b, tok});
    }
    Py_DECREF(cs);
    cp[g + 1] = (int32_t)(csh.size() / 5);
  }
  Py_DECREF(seq);
  return Py_BuildValue("(y#y#y#y#)", bptr(mp), (Py_ssize_t)(mp.size() * 4), bptr(msh),
                       (Py_ssize_t)(msh.size() * 8), bptr(cp), (Py_ssize_t)(cp.size() * 4), bptr(csh),
                       (Py_ssize_t)(csh.size() * 8));
fail:
  Py_DECREF(seq);
  return nullptr;
}

PyMethodDef kMethods[] = {
    {"common_denominator", py_common_denominator, METH_VARARGS, "lcm of M and every interval denominator"},
    {"pack_rows", py_pack_rows, METH_VARARGS, "inventories -> (row_ptr, segments) bytes"},
    {"flatten", py_flatten, METH_VARARGS, "inventories -> planner arrays (bytes)"},
    {nullptr, nullptr, 0, nullptr},
};

PyModuleDef kModule = {PyModuleDef_HEAD_INIT, "_hostpack", "native host-side packing", -1, kMethods};

}  // namespace

PyMODINIT_FUNC PyInit__hostpack(void) {
  g_num = PyUnicode_InternFromString("numerator");
  g_num_slot = PyUnicode_InternFromString("_numerator");
  g_den_slot = PyUnicode_InternFromString("_denominator");
  g_den = PyUnicode_InternFromString("denominator");
  return PyModule_Create(&kModule);
}
