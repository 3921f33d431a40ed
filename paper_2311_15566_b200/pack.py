"""Host packer: GPU context inventories -> exact integer segments (sk_segment).

A row's inventory (model shards (layer, lo, hi) and cache shards (rid, layer,
lo, hi, tokens), reference domain.py:175-220) is rewritten over one common
denominator K as runs of consecutive layers sharing an interval:

* model runs   (l0, l1, a, b, pipe=0, unit = bytes_per_layer * multiplicity)
* cache runs   (l0, l1, a, b, pipe=d, unit = kv * sum_r min(tokens_held, tokens_needed))
  where d is the NEW pipeline whose positions need request r's cache
  (required_context_with_cache, mapping.py:155-169, fed by the inheritance
  map, mapping.py:200-208).

Then the reference's exact overlap (domain.py:299-320) between row u and
position v equals  sum_seg |[l0,l1) & stage(v)| * |[a,b) & I(v)| * unit / K,
which the device evaluates in int64 and converts with one correctly rounded
division.  Nothing here computes a weight; it only re-encodes inventories.
"""

from __future__ import annotations

from math import lcm

import numpy as np

from ._native import SEGMENT, SEGMENT_WIDE

EXACT_LIMIT = 1 << 53       # regular encoding: numerators exact in int64 -> double
K_LIMIT = (1 << 31) - 1     # regular encoding: int32 endpoints
WIDE_LIMIT = 1 << 127       # general-range encoding: 128-bit numerators
K_WIDE_LIMIT = 1 << 62      # general-range encoding: 64-bit endpoints


class PackError(ValueError):
    pass


def _native():
    try:
        from . import _hostpack
    except ImportError as e:  # built by paper_2311_15566_b200.build
        raise RuntimeError("paper_2311_15566_b200._hostpack is not built "
                           "(python -m paper_2311_15566_b200.build)") from e
    return _hostpack


def common_denominator(inventories, tensor_shards: int) -> int:
    """lcm of M and every interval denominator (native)."""
    try:
        return _native().common_denominator(inventories, tensor_shards)
    except ValueError as e:
        raise PackError(str(e)) from None


def py_common_denominator(inventories, tensor_shards: int) -> int:
    """Pure-Python statement of common_denominator (cross-checked in tests)."""
    dens = {tensor_shards}
    for inv in inventories:
        for _, lo, hi in inv.model_shards:
            dens.add(lo.denominator)
            dens.add(hi.denominator)
        for _, _, lo, hi, _ in inv.cache_shards:
            dens.add(lo.denominator)
            dens.add(hi.denominator)
    K = 1
    for d in dens:
        K = lcm(K, d)
        if K >= K_WIDE_LIMIT:
            raise PackError("common interval denominator exceeds 2^62")
    return K


def inherited_by_new(inheritance, requests_by_old_pipeline):
    """new pipeline -> [(rid, tokens)], old pipelines ascending, requests by id
    (mapping.py:200-208)."""
    out: dict[int, list] = {}
    if inheritance and requests_by_old_pipeline:
        for d_old in sorted(requests_by_old_pipeline):
            d_new = inheritance.get(d_old)
            if d_new is None:
                continue
            for req in sorted(requests_by_old_pipeline[d_old], key=lambda r: r.id):
                out.setdefault(d_new, []).append((req.id, req.s_in + req.tokens_generated))
    return out


def need_tokens(inherited: dict, n_pipelines: int | None = None) -> dict:
    """rid -> [(new pipeline, tokens)] for tokens > 0 (the filter of
    mapping.py:167).  Only new pipelines 1..n_pipelines have positions
    (build_graph looks entries up by pos.pipeline, mapping.py:210-213), so an
    inheritance target outside that range contributes nothing and is dropped."""
    out: dict[str, list] = {}
    for d_new in sorted(inherited):
        if n_pipelines is not None and not 1 <= d_new <= n_pipelines:
            continue
        for rid, tok in inherited[d_new]:
            if tok > 0:
                out.setdefault(rid, []).append((d_new, tok))
    return out


def _runs(entries):
    """entries: {(key..., layer): unit}; merge consecutive layers with equal
    (key, unit) -> [(l0, l1, key, unit)]."""
    out = []
    for k in sorted(entries):
        *key, layer = k
        unit = entries[k]
        key = tuple(key)
        if out and out[-1][2] == key and out[-1][3] == unit and out[-1][1] == layer:
            l0, _, kk, uu = out[-1]
            out[-1] = (l0, layer + 1, kk, uu)
        else:
            out.append((layer, layer + 1, key, unit))
    return out


def pack_row(inv, K: int, bpl: int, kv: int, need: dict):
    """One inventory -> list of (l0, l1, a, b, pipe, unit)."""
    scale: dict = {}

    def num(x):
        r = scale.get(x)
        if r is None:
            r = x.numerator * (K // x.denominator)
            scale[x] = r
        return r

    model: dict = {}
    for layer, lo, hi in inv.model_shards:
        k = (num(lo), num(hi), layer)
        model[k] = model.get(k, 0) + 1
    segs = [(l0, l1, a, b, 0, bpl * mult) for l0, l1, (a, b), mult in _runs(model)]
    if need and inv.cache_shards:
        cache: dict = {}
        for rid, layer, lo, hi, tok in inv.cache_shards:
            ents = need.get(rid)
            if not ents:
                continue
            a, b = num(lo), num(hi)
            for d_new, t in ents:
                k = (a, b, d_new, layer)
                cache[k] = cache.get(k, 0) + (tok if tok < t else t)
        segs.extend((l0, l1, a, b, d, kv * tsum) for l0, l1, (a, b, d), tsum in _runs(cache) if tsum)
    return segs


def pack_rows(inventories, K: int, bpl: int, kv: int, need: dict, wide: bool = False):
    """-> (row_ptr int32[R+1], segments, wide) via the native packer
    (csrc/hostpack.cpp), identical to py_pack_rows.  `wide` (returned): the
    rows are encoded as sk_segment_wide (two SEGMENT slots each) for the
    general-range kernels -- forced by the caller, or because K > 2^31 - 1 or
    a numerator may reach 2^53."""
    try:
        rp, sg, w = _native().pack_rows(inventories, K, bpl, kv, need, bool(wide))
    except ValueError as e:
        raise PackError(str(e)) from None
    segs = np.frombuffer(sg, dtype=SEGMENT_WIDE if w else SEGMENT).copy()
    if w:
        segs = segs.view(SEGMENT)
    return np.frombuffer(rp, dtype=np.int32).copy(), segs, bool(w)


def py_pack_rows(inventories, K: int, bpl: int, kv: int, need: dict, wide: bool = False):
    """Pure-Python statement of pack_rows: the readable spec the native packer
    is tested against (tests/test_pack.py)."""
    rows = [pack_row(inv, K, bpl, kv, need) for inv in inventories]
    wide = wide or K > K_LIMIT
    row_ptr = np.zeros(len(rows) + 1, dtype=np.int32)
    total = 0
    for i, segs in enumerate(rows):
        if any(s[5] >= 1 << 63 for s in segs):
            raise PackError("segment bytes exceed 2^63: outside the exact range")
        # every W numerator of this row is <= the sum of its segments' spans
        bound = sum((s[1] - s[0]) * (s[3] - s[2]) * s[5] for s in segs)
        if bound >= WIDE_LIMIT:
            raise PackError("edge-weight numerator may exceed 2^127: outside the exact range")
        wide = wide or bound >= EXACT_LIMIT
        total += len(segs)
        row_ptr[i + 1] = total
    dt = SEGMENT_WIDE if wide else SEGMENT
    out = np.zeros(total, dtype=dt)
    if total:
        arr = np.array([s for segs in rows for s in segs], dtype=object)
        for f, col in (("l0", 0), ("l1", 1), ("a", 2), ("b", 3), ("pipe", 4), ("unit", 5)):
            out[f] = arr[:, col].astype(np.int64)
    if wide:
        return row_ptr * 2, out.view(SEGMENT), True
    return row_ptr, out, False
