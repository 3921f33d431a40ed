"""Migration executor (K3): carry out a MigrationPlan's weight + KV reshard on
the GPUs of one box, in plan order and within the plan's memory budget.

The reference only plans and costs a migration (migration.py:311-384,
costmodel.py:189-260); the paper's engine executes it with batched async NCCL
send/recv, allocating and releasing migration buffers "based on the migration
plan".  Here:

* **Memory follows the plan.**  Each GPU's context lives in one arena.  The
  old shards are placed first; every `Transfer` into the GPU gets a fresh
  piece of arena when its round starts; at the end of each round the GPU's
  bytes the plan `releases` (held - kept, migration.py:283-305) go back to the
  arena's free list and later rounds recycle them.  Kept bytes never move:
  a new shard is the kept pieces of old shards (aliased in place) plus the
  received pieces.  So the arena's high-water mark is the plan's
  `peak_usage` (simulate_buffer_usage, migration.py:387-401) above the old
  footprint, up to alignment and first-fit fragmentation (`ArenaLayout`,
  pure host logic, CPU-tested).
* **Execution follows the plan.**  One persistent `k_exec` launch per rank
  (include/spotkm.h `sk_exec_plan`) copies 1 MiB chunks in round order over
  CUDA-IPC peer mappings (NVLink).  A chunk that lands in recycled space
  waits until every rank has finished the round that freed it -- the only
  cross-rank dependency -- and the device raises each stage's ready flag as
  soon as the round its `start_stage` marker follows is globally complete
  (migration.py:352-371; the paper's per-tensor readiness).

Byte geometry (SURVEY.md finding 8).  A layer's parameters are one flat byte
array of `bytes_per_layer` bytes; tensor shard [lo, hi) owns bytes
[lo*B, hi*B).  A request's KV cache of one layer is one flat array of
kv_bytes_per_token_per_layer * tokens bytes laid out [head][K|V][tok][hd], so
a head-fraction shard [lo, hi) is again the contiguous range [lo*X, hi*X).
Every shard boundary must be a whole number of 8-byte words (checked).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from fractions import Fraction
from math import lcm

import numpy as np
import torch

from . import _native as nat

CHUNK = 1 << 20          # copy granularity: 1 MiB pieces keep every CTA busy
ALIGN = 256              # arena allocation alignment
EXEC_CHUNK = np.dtype([("src", "<u8"), ("dst", "<u8"), ("bytes", "<u8"), ("round", "<i4"),
                       ("wait_round", "<i4")])
assert EXEC_CHUNK.itemsize == 32


def _mix64(z: int) -> int:
    m = (1 << 64) - 1
    z = (z + 0x9E3779B97F4A7C15) & m
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
    return z ^ (z >> 31)


def model_key(seed: int, layer: int) -> int:
    return _mix64((seed << 20) ^ (1 << 60) ^ layer)


def cache_key(seed: int, rid_index: int, layer: int) -> int:
    return _mix64((seed << 20) ^ (2 << 60) ^ (rid_index << 24) ^ layer)


def _span(frac: Fraction, total: int) -> int:
    v = frac * total
    if v.denominator != 1 or v.numerator % 8:
        raise ValueError(f"shard boundary {frac} of a {total}-byte object is not 8-byte aligned")
    return v.numerator


def _align(n: int, a: int = ALIGN) -> int:
    return (n + a - 1) // a * a


# ---------------------------------------------------------------------------
# host-side arena layout (pure Python, no GPU)

MIN_EXTENT = 64 << 10    # smallest piece a received transfer is split into


class Arena:
    """Round-tagged first-fit arena.  Space freed at the end of round d must
    not be written before every rank has finished round d, so every
    allocation reports the latest such round it recycles (`wait`, -1 for
    fresh space).  A received transfer may be placed as several extents
    (scatter-gather: the new context is piecewise anyway), so freed holes are
    reused even when no single one is large enough."""

    def __init__(self):
        self.free: list[list] = []   # [offset, size, round freed] sorted by offset
        self.top = 0                 # end of the highest allocation
        self.high = 0

    def alloc_top(self, n: int) -> int:
        off = _align(self.top)
        self.top = off + n
        self.high = max(self.high, self.top)
        return off

    def _runs(self):
        """maximal address-contiguous runs of free pieces: (i, j, start, end, wait)"""
        fr, i = self.free, 0
        while i < len(fr):
            j, end, wait = i, fr[i][0] + fr[i][1], fr[i][2]
            while j + 1 < len(fr) and fr[j + 1][0] == end:
                j += 1
                end = fr[j][0] + fr[j][1]
                wait = max(wait, fr[j][2])
            yield i, j, fr[i][0], end, wait
            i = j + 1

    def _take(self, a: int, b: int) -> int:
        """remove [a, b) from the free list; -> the latest round it recycles"""
        keep, wait = [], -1
        for off, size, rnd in self.free:
            if off + size <= a or off >= b:
                keep.append([off, size, rnd])
                continue
            wait = max(wait, rnd)
            if off < a:
                keep.append([off, a - off, rnd])
            if off + size > b:
                keep.append([b, off + size - b, rnd])
        self.free = keep
        return wait

    def alloc(self, n: int):
        """-> [(offset, length, wait round)] extents covering n bytes: one
        first-fit block if a hole holds it, else the holes in address order
        (>= MIN_EXTENT each, 256-B aligned), then fresh space at the top."""
        for i, j, a, b, _ in self._runs():
            s = _align(a)
            if b - s >= n:
                return [(s, n, self._take(s, s + n))]
        out, left = [], n
        for i, j, a, b, _ in list(self._runs()):
            s = _align(a)
            room = (b - s) // ALIGN * ALIGN
            if room < MIN_EXTENT and not (b == self.top and left <= room + 0):
                continue
            take = min(room, left)
            if b == self.top and left > room:
                break   # the run ends at the top: extend it below
            out.append((s, take, self._take(s, s + take)))
            left -= take
            if left == 0:
                return out
        # the rest at the top, starting inside a free run that touches it
        start = _align(self.top)
        for i, j, a, b, _ in self._runs():
            if b == self.top and _align(a) < start:
                start = _align(a)
        w = self._take(start, start + left) if start < self.top else -1
        self.top = max(self.top, start + left)
        self.high = max(self.high, self.top)
        out.append((start, left, w))
        return out

    def release(self, off: int, n: int, rnd: int):
        if n <= 0:
            return
        self.free.append([off, n, rnd])
        self.free.sort()
        # coalesce neighbours freed in the same round
        out = []
        for piece in self.free:
            if out and out[-1][0] + out[-1][1] == piece[0] and out[-1][2] == piece[2]:
                out[-1][1] += piece[1]
            else:
                out.append(piece)
        self.free = out


@dataclass
class Region:
    """One contiguous byte range of a context object held in an arena."""

    key: tuple            # ("m", layer) or ("c", rid, layer)
    lo: Fraction          # shard interval of the object
    hi: Fraction
    tokens: int
    unit: int             # object bytes per unit interval (B or kv * tokens)
    off: int              # arena byte offset of lo
    released: list = field(default_factory=list)   # (round, [lo, hi)) sub-intervals freed

    def byte_range(self, lo: Fraction, hi: Fraction):
        return self.off + _span(lo - self.lo, self.unit), _span(hi - lo, self.unit)


@dataclass
class GpuLayout:
    arena: Arena
    old: list                 # Regions of the old context
    pieces: list              # new context: (key, lo, hi, tokens, unit, arena offset)
    incoming: dict            # id(transfer) -> [(arena offset, length, wait round)] extents
    old_bytes: int            # exact bytes of the old context
    old_footprint: int        # arena bytes after placing it (aligned)


class ArenaLayout:
    """Where every byte of a plan's old and new contexts lives, per GPU, and
    which arena space each transfer recycles (see the module docstring).

    `rounds`: the plan's non-start_stage actions in order (round index =
    position); `stage_round[stage]` = the last round before its marker (-1:
    ready at the start)."""

    def __init__(self, plan, old_layout, new_required, model, recycle: bool = True):
        self.plan = plan
        self.recycle = recycle
        self.B, self.kv = model.bytes_per_layer, model.kv_bytes_per_token_per_layer
        self.rounds = [a for a in plan.actions if a.kind != "start_stage"]
        self.stage_round = {}
        r = -1
        for a in plan.actions:
            if a.kind == "start_stage":
                self.stage_round[a.stage] = r
            else:
                r += 1
        gpus = sorted(set(old_layout) | set(new_required))
        self.gpus: dict = {}
        for g in gpus:
            self.gpus[g] = self._place_old(old_layout.get(g))
        # per round: allocate the incoming pieces, then free the releases
        need = {g: new_required.get(g) for g in gpus}
        kept = {g: self._kept(self.gpus[g].old, need[g]) for g in gpus}
        self.freed_bytes: list[dict] = []
        for ri, action in enumerate(self.rounds):
            for t in action.transfers:
                gl = self.gpus[t.dst]
                unit = self.B if t.kind == "model" else self.kv * t.tokens
                n = _span(t.hi - t.lo, unit)
                if n != t.bytes:
                    raise ValueError(f"transfer bytes {t.bytes} != geometry {n}")
                ext = gl.arena.alloc(n)
                gl.incoming[id(t)] = ext
                key = ("m", t.layer) if t.kind == "model" else ("c", t.request, t.layer)
                pos = 0
                for off, ln, _ in ext:
                    lo = t.lo + Fraction(pos, unit)
                    gl.pieces.append((key, lo, lo + Fraction(ln, unit), t.tokens, unit, off))
                    pos += ln
            self.freed_bytes.append(self._release(ri, action, kept))
        for g in gpus:
            gl = self.gpus[g]
            for reg in gl.old:
                for lo, hi in kept[g].get(id(reg), ()):
                    gl.pieces.append((reg.key, lo, hi, reg.tokens, reg.unit, reg.byte_range(lo, hi)[0]))
            self._check_coverage(g, need[g])

    def _place_old(self, inv):
        ar = Arena()
        regs = []
        total = 0
        if inv is not None:
            for layer, lo, hi in inv.model_shards:
                n = _span(hi - lo, self.B)
                regs.append(Region(("m", layer), lo, hi, 0, self.B, ar.alloc_top(n)))
                total += n
            for rid, layer, lo, hi, tok in inv.cache_shards:
                n = _span(hi - lo, self.kv * tok)
                regs.append(Region(("c", rid, layer), lo, hi, tok, self.kv * tok, ar.alloc_top(n)))
                total += n
        return GpuLayout(ar, regs, [], {}, total, _align(ar.top))

    @staticmethod
    def _kept(regs, need):
        """id(region) -> [(lo, hi)] of it the GPU keeps for its own new context
        (the `kept` of migration.py:287-303)."""
        out: dict = {}
        if need is None:
            return out
        want: dict = {}
        for layer, lo, hi in need.model_shards:
            want.setdefault(("m", layer), []).append((lo, hi, 0))
        for rid, layer, lo, hi, tok in need.cache_shards:
            want.setdefault(("c", rid, layer), []).append((lo, hi, tok))
        for reg in regs:
            for lo, hi, tok in want.get(reg.key, ()):
                a, b = max(lo, reg.lo), min(hi, reg.hi)
                if b <= a:
                    continue
                if reg.key[0] == "c" and tok != reg.tokens:
                    raise ValueError("kept KV shard with a different token count: the byte-range "
                                     "executor keeps whole per-token blocks only")
                out.setdefault(id(reg), []).append((a, b))
        return out

    def _release(self, ri, action, kept):
        """Free, at the end of round ri, every old byte the plan releases in
        it: held - kept of the round's layer (migrate_layer) or of all cache
        shards (migrate_cache).  Returns {instance: bytes freed} for the
        cross-check against the plan's `releases`."""
        freed: dict = {}
        for g, gl in self.gpus.items():
            for reg in gl.old:
                if action.kind == "migrate_layer" and reg.key != ("m", action.layer):
                    continue
                if action.kind == "migrate_cache" and reg.key[0] != "c":
                    continue
                pieces = [(reg.lo, reg.hi)]
                for a, b in sorted(kept[g].get(id(reg), ())):
                    nxt = []
                    for lo, hi in pieces:
                        if b <= lo or a >= hi:
                            nxt.append((lo, hi))
                            continue
                        if lo < a:
                            nxt.append((lo, a))
                        if b < hi:
                            nxt.append((b, hi))
                    pieces = nxt
                for lo, hi in pieces:
                    off, n = reg.byte_range(lo, hi)
                    if self.recycle:
                        gl.arena.release(off, n, ri)
                    reg.released.append((ri, lo, hi))
                    freed[g[0]] = freed.get(g[0], 0) + n
        return freed

    def _check_coverage(self, g, need):
        have: dict = {}
        for key, lo, hi, tok, unit, off in self.gpus[g].pieces:
            have.setdefault(key, []).append((lo, hi))
        want = []
        if need is not None:
            want = [(("m", layer), lo, hi) for layer, lo, hi in need.model_shards]
            want += [(("c", rid, layer), lo, hi) for rid, layer, lo, hi, tok in need.cache_shards]
        for key, lo, hi in want:
            ps = sorted(have.get(key, ()))
            pos = lo
            for a, b in ps:
                if a <= pos < b:
                    pos = b
            if pos < hi:
                raise ValueError(f"new context of {g} misses {key} [{pos}, {hi})")

    # -- reports -------------------------------------------------------------
    def check_releases(self):
        """Bytes the arena frees per round and instance == the plan's
        `releases` (relative 1e-12: the plan sums per-shard floats)."""
        for ri, action in enumerate(self.rounds):
            plan_rel = dict(action.releases)
            mine = self.freed_bytes[ri]
            if set(plan_rel) != set(mine):
                raise ValueError(f"round {ri}: released instances {sorted(mine)} != plan {sorted(plan_rel)}")
            for inst, b in plan_rel.items():
                if abs(mine[inst] - b) > 1e-12 * max(1.0, b):
                    raise ValueError(f"round {ri}: {inst} frees {mine[inst]} != plan {b}")

    def memory_report(self):
        """Per instance: old footprint, arena high-water, and the plan's
        peak_usage (migration buffers above the old context)."""
        per_inst: dict = {}
        for g, gl in self.gpus.items():
            d = per_inst.setdefault(g[0], {"old_bytes": 0, "arena_bytes": 0})
            d["old_bytes"] += gl.old_bytes
            d["arena_bytes"] += gl.arena.high
        for inst, d in per_inst.items():
            peak = float(self.plan.peak_usage.get(inst, 0.0))
            d["plan_peak_usage"] = peak
            d["plan_bound_bytes"] = d["old_bytes"] + peak
            d["arena_over_plan"] = d["arena_bytes"] / max(1.0, d["old_bytes"] + peak)
        return per_inst


# ---------------------------------------------------------------------------
# device side

def traffic(plan):
    """bytes in / out per GPU over NVLink (src != dst GPU)."""
    bin_, bout = {}, {}
    for t in plan.transfers():
        if t.src == t.dst:
            continue
        bout[t.src] = bout.get(t.src, 0) + int(t.bytes)
        bin_[t.dst] = bin_.get(t.dst, 0) + int(t.bytes)
    return bin_, bout


class _Mem:
    def __init__(self, nbytes: int):
        self.lib = nat.load()
        p = ctypes.c_void_p()
        nat.check(self.lib.sk_dev_alloc(max(nbytes, 16), ctypes.byref(p)))
        self.ptr = p.value
        self.nbytes = nbytes

    def free(self):
        if self.ptr:
            self.lib.sk_dev_free(self.ptr)
            self.ptr = None


def _exec_lib():
    lib = nat.load()
    if not getattr(lib, "_exec_sigs", False):
        vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
        lib.sk_exec_ctl_bytes.argtypes = [i32, i32]
        lib.sk_exec_ctl_bytes.restype = i64
        lib.sk_exec_plan.argtypes = [vp, i32, vp, i32, vp, i32, vp, vp, i32, vp, i32, ctypes.c_double, vp]
        lib.sk_exec_plan.restype = i32
        lib.sk_memcpy_batched.argtypes = [vp, i32, vp]
        lib.sk_memcpy_batched.restype = i32
        lib.sk_host_register.argtypes = [vp, ctypes.c_uint64, ctypes.POINTER(vp)]
        lib.sk_host_register.restype = i32
        lib.sk_host_unregister.argtypes = [vp]
        lib.sk_host_unregister.restype = i32
        lib.sk_exec_reset.argtypes = [vp, i32, i32, vp]
        lib.sk_exec_reset.restype = i32
        lib.sk_d2h.argtypes = [vp, vp, ctypes.c_uint64]
        lib.sk_d2h.restype = i32
        lib._exec_sigs = True
    return lib


def slab_offsets(layout: "ArenaLayout", owner: dict, rank: int, ctl_bytes: int):
    """This rank's slab: [control block | arena(ref) ...] -> ({ref: offset}, size)."""
    off = _align(ctl_bytes)
    ref_off = {}
    for g in sorted(g for g, r in owner.items() if r == rank):
        ref_off[g] = off
        if g in layout.gpus:
            off = _align(off + layout.gpus[g].arena.high)
    return ref_off, off


def exchange_slabs(rank: int, world: int, slab_ptr: int, handle: bytes, ref_off: dict, opener, group=None):
    """All-gather every rank's (IPC handle, arena offsets) and map the peers'
    slabs with `opener(handle) -> device pointer`.  Returns ({ref: arena base
    usable here}, {rank: control block pointer usable here}, [opened ptrs])."""
    base = {g: slab_ptr + o for g, o in ref_off.items()}
    ctl = {rank: slab_ptr}
    opened = []
    if world > 1:
        import torch.distributed as dist

        gathered = [None] * world
        dist.all_gather_object(gathered, {"handle": handle, "ref_off": ref_off}, group=group)
        for r, doc in enumerate(gathered):
            if r == rank:
                continue
            p = opener(doc["handle"])
            opened.append(p)
            ctl[r] = p
            for g, o in doc["ref_off"].items():
                base[g] = p + o
    return base, ctl, opened


def region_of(layout: "ArenaLayout", g, t) -> Region:
    """The old shard of GPU g a transfer reads from."""
    key = ("m", t.layer) if t.kind == "model" else ("c", t.request, t.layer)
    for reg in layout.gpus[g].old:
        if reg.key == key and reg.lo <= t.lo and t.hi <= reg.hi and (t.kind == "model" or reg.tokens == t.tokens):
            return reg
    raise ValueError(f"transfer {t} has no source shard on {g}")


def issue_list(layout: "ArenaLayout", owner: dict, rank: int, mode: str, base: dict):
    """The copies `rank` issues, in plan order: pull -> the transfers into its
    GPUs, push -> the transfers out of them.  One entry per received extent:
    (round, src ptr, dst ptr, bytes, wait round, transfer)."""
    out = []
    for ri, action in enumerate(layout.rounds):
        for t in action.transfers:
            if owner[t.dst if mode == "pull" else t.src] != rank:
                continue
            s_off, _ = region_of(layout, t.src, t).byte_range(t.lo, t.hi)
            pos = 0
            for d_off, ln, w in layout.gpus[t.dst].incoming[id(t)]:
                out.append((ri, base[t.src] + s_off + pos, base[t.dst] + d_off, ln, w, t))
                pos += ln
    return out


def p2p_ops(layout: "ArenaLayout", owner: dict, rank: int, local_base: dict):
    """`rank`'s side of every transfer extent, in plan order, for a send/recv
    baseline: ("send", peer, local ptr, n), ("recv", peer, local ptr, n), or
    ("local", None, (src, dst), n) when both GPUs are this rank's.  Matching
    send/recv pairs appear in the same order on both ranks."""
    out = []
    for action in layout.rounds:
        for t in action.transfers:
            rs, rd = owner[t.src], owner[t.dst]
            if rank not in (rs, rd):
                continue
            s_off, _ = region_of(layout, t.src, t).byte_range(t.lo, t.hi)
            pos = 0
            for d_off, ln, _ in layout.gpus[t.dst].incoming[id(t)]:
                if rs == rd:
                    out.append(("local", None, (local_base[t.src] + s_off + pos, local_base[t.dst] + d_off), ln))
                elif rs == rank:
                    out.append(("send", rd, local_base[t.src] + s_off + pos, ln))
                else:
                    out.append(("recv", rs, local_base[t.dst] + d_off, ln))
                pos += ln
    return out


class ReshardExecutor:
    """Executes one MigrationPlan on this process's GPU(s).

    `owner[gpu_ref]` = rank hosting that GPU.  Each rank allocates ONE slab
    (control block + one arena per owned GPU ref, sized by ArenaLayout), the
    ranks exchange CUDA IPC handles of their slabs through torch.distributed,
    and each rank's k_exec launch issues its share of the copies: pull = the
    transfers INTO its GPUs (reading peers' old shards over NVLink), push =
    the transfers OUT of its GPUs.  With world == 1 every GPU ref is emulated
    in the local slab (same code path, local pointers) -- used by the tests.
    `recycle=False` keeps released bytes allocated (arena = old + every
    received byte): the layout the order-free comparison paths
    (run_unordered, run_memcpy, NCCL) need.
    """

    def __init__(self, plan, old_layout, new_required, model, owner: dict, rank: int = 0,
                 world: int = 1, seed: int = 1, group=None, mode: str = "pull", chunk: int = CHUNK,
                 timeout_s: float = 30.0, recycle: bool = True):
        if mode not in ("pull", "push"):
            raise ValueError("mode must be 'pull' or 'push'")
        self.lib = _exec_lib()
        self.rank, self.world, self.mode, self.group = rank, world, mode, group
        self.plan = plan
        self.timeout_s = timeout_s
        self.layout = ArenaLayout(plan, old_layout, new_required, model, recycle)
        self.layout.check_releases()
        L = self.layout
        self.n_rounds = len(L.rounds)
        stages = sorted(L.stage_round)
        self.stages = stages
        self.ctl_bytes = int(self.lib.sk_exec_ctl_bytes(self.n_rounds, len(stages)))
        # this rank's slab: [control | arena(ref) ...], peers' slabs IPC-mapped
        self.mine = sorted(g for g, r in owner.items() if r == rank)
        ref_off, size = slab_offsets(L, owner, rank, self.ctl_bytes)
        self.slab = _Mem(size)
        handle = b""
        if world > 1:
            h = ctypes.create_string_buffer(64)
            nat.check(self.lib.sk_ipc_get_handle(self.slab.ptr, h))
            handle = h.raw

        def opener(raw):
            p = ctypes.c_void_p()
            nat.check(self.lib.sk_ipc_open_handle(raw, ctypes.byref(p)))
            return p.value

        base, ctl_ptr, self.opened = exchange_slabs(rank, world, self.slab.ptr, handle, ref_off, opener, group)
        self.base = base
        self.owner = owner
        self.local_base = {g: self.slab.ptr + o for g, o in ref_off.items()}
        dev = torch.device("cuda", torch.cuda.current_device())
        self._dev = dev
        # the copies this rank issues, in plan order, cut into chunks
        rows, rnd, wait = [], [], []
        self.transfers_issued = []
        issued = issue_list(L, owner, rank, mode, base)
        for ri, src_ptr, dst_ptr, ln, w, t in issued:
            self.transfers_issued.append((src_ptr, dst_ptr, ln, owner[t.src], owner[t.dst]))
            for c in range(0, ln, chunk):
                rows.append((src_ptr + c, dst_ptr + c, min(chunk, ln - c)))
                rnd.append(ri)
                wait.append(w)
        self.remote_bytes = sum(e[3] for e in issued)
        ch = np.zeros(len(rows), dtype=EXEC_CHUNK)
        if rows:
            arr = np.array(rows, dtype=np.uint64)
            ch["src"], ch["dst"], ch["bytes"] = arr[:, 0], arr[:, 1], arr[:, 2]
            ch["round"], ch["wait_round"] = rnd, wait
        self.n_chunks = len(ch)
        totals = np.bincount(np.array(rnd, dtype=np.int64), minlength=self.n_rounds).astype(np.uint32) \
            if rnd else np.zeros(self.n_rounds, np.uint32)
        srounds = np.array([L.stage_round[s] for s in stages], dtype=np.int32)
        peers = [ctl_ptr[r] + 4 for r in sorted(ctl_ptr) if r != rank]
        self.d_chunks = torch.from_numpy(ch.view(np.uint8)).to(dev) if len(ch) else None
        self.d_totals = torch.from_numpy(np.ascontiguousarray(totals).view(np.uint8)).to(dev) \
            if self.n_rounds else None
        self.d_stages = torch.from_numpy(srounds.view(np.uint8)).to(dev) if len(stages) else None
        self.d_peers = torch.from_numpy(np.array(peers or [0], dtype=np.uint64).view(np.uint8)).to(dev)
        self.n_peers = len(peers)
        # unordered one-launch copy list (k_copy) and per-transfer copy list (copy engines)
        cp = np.zeros(len(rows), dtype=nat.COPY)
        if rows:
            cp["src"], cp["dst"], cp["bytes"] = ch["src"], ch["dst"], ch["bytes"]
        self.d_copies = torch.from_numpy(cp.view(np.uint8)).to(dev) if len(cp) else None
        tr = np.zeros(len(self.transfers_issued), dtype=nat.COPY)
        for i, (s, d, n, _, _) in enumerate(self.transfers_issued):
            tr[i] = (s, d, n)
        self.h_transfers = tr
        self.seed = seed
        self.d_fill = self._regions(new=False)
        self.d_check = self._regions(new=True)
        self.d_bad = torch.zeros(1, dtype=torch.int64, device=dev)

    def region_rows(self, new: bool, seed: int | None = None):
        """[(gpu ref, (ptr, bytes, pattern key, object byte base))] of this
        rank's old contexts (new=False) or new contexts (every kept and
        received piece, new=True)."""
        seed = self.seed if seed is None else seed
        rids = sorted({k[1] for gl in self.layout.gpus.values() for r in gl.old for k in [r.key] if k[0] == "c"}
                      | {p[0][1] for gl in self.layout.gpus.values() for p in gl.pieces if p[0][0] == "c"})
        rid_index = {r: i for i, r in enumerate(rids)}

        def key_of(key):
            return model_key(seed, key[1]) if key[0] == "m" else cache_key(seed, rid_index[key[1]], key[2])

        rows = []
        for g in self.mine:
            gl = self.layout.gpus.get(g)
            if gl is None:
                continue
            if new:
                for key, lo, hi, tok, unit, off in gl.pieces:
                    rows.append((g, (self.base[g] + off, _span(hi - lo, unit), key_of(key), _span(lo, unit))))
            else:
                for reg in gl.old:
                    rows.append((g, (self.base[g] + reg.off, _span(reg.hi - reg.lo, reg.unit), key_of(reg.key),
                                     _span(reg.lo, reg.unit))))
        return rows

    def _regions(self, new: bool):
        rows = [r for _, r in self.region_rows(new)]
        reg = np.zeros(len(rows), dtype=nat.REGION)
        for i, r in enumerate(rows):
            reg[i] = r
        return (torch.from_numpy(reg.view(np.uint8)).to(self._dev), len(rows)) if rows else (None, 0)

    # -- running -------------------------------------------------------------
    def fill_old(self):
        """(Re)write every old shard's pattern -- needed before each run, since
        a run recycles released old space for received data."""
        t, n = self.d_fill
        if n:
            nat.check(self.lib.sk_fill_regions(t.data_ptr(), n, torch.cuda.current_stream().cuda_stream))

    def run(self, n_ctas: int = 0, flag_mirror: int = 0):
        """The reshard: one k_exec launch over this rank's copies, in plan
        order (resets the control block first; ranks must barrier between
        runs so no peer reads a stale progress word).  flag_mirror: device
        address of host-mapped memory that also receives the stage flags."""
        st = torch.cuda.current_stream().cuda_stream
        nat.check(self.lib.sk_exec_plan(
            self.d_chunks.data_ptr() if self.d_chunks is not None else 0, self.n_chunks,
            self.d_totals.data_ptr() if self.d_totals is not None else 0, self.n_rounds,
            self.d_stages.data_ptr() if self.d_stages is not None else 0, len(self.stages),
            self.slab.ptr, self.d_peers.data_ptr(), self.n_peers, flag_mirror, n_ctas, self.timeout_s, st))

    def reset_control(self):
        """Zero the control block (every stage flag down) on the current stream."""
        nat.check(self.lib.sk_exec_reset(self.slab.ptr, self.n_rounds, len(self.stages),
                                         torch.cuda.current_stream().cuda_stream))

    def run_unordered(self, n_ctas: int = 0):
        """Data path only: the same chunks in one k_copy launch with no round
        order or recycling waits (for NVLink counters; byte-exact only with
        recycle=False)."""
        if self.d_copies is not None:
            nat.check(self.lib.sk_copy_batched(self.d_copies.data_ptr(), self.n_chunks, n_ctas,
                                               torch.cuda.current_stream().cuda_stream))

    def run_memcpy(self):
        """Copy-engine comparison: one cudaMemcpyAsync per issued transfer
        extent, in plan order on the current stream (no recycling waits
        either: byte-exact only with recycle=False)."""
        if len(self.h_transfers):
            nat.check(self.lib.sk_memcpy_batched(self.h_transfers.ctypes.data, len(self.h_transfers),
                                                 torch.cuda.current_stream().cuda_stream))

    def p2p_ops(self):
        """This rank's side of every transfer extent for a send/recv baseline
        (see `p2p_ops`)."""
        return p2p_ops(self.layout, self.owner, self.rank, self.local_base)

    def control(self) -> dict:
        """This rank's control block after a run (synchronizes): error code,
        rounds completed, stage flags and stage-ready times (ms after launch)."""
        torch.cuda.synchronize()
        raw = np.zeros(self.ctl_bytes, dtype=np.uint8)
        nat.check(self.lib.sk_d2h(raw.ctypes.data, self.slab.ptr, self.ctl_bytes))
        w = raw.view(np.uint32)
        R, S = self.n_rounds, len(self.stages)
        flags = w[4 + R:4 + R + S]
        so = ((4 + R + S + 1) & ~1) * 4
        stamps = raw[so:so + 8 * (S + 1)].view(np.uint64).astype(np.float64)
        return {"error": int(w[2]), "progress": int(w[1]), "rounds": R,
                "stage_flags": {s: int(f) for s, f in zip(self.stages, flags)},
                "stage_ready_ms": {s: (stamps[1 + i] - stamps[0]) / 1e6 for i, s in enumerate(self.stages)}}

    def verify(self) -> int:
        """Mismatching 8-byte words in this rank's new contexts (0 = every
        required shard byte-identical, kept and received pieces alike)."""
        t, n = self.d_check
        self.d_bad.zero_()
        if n:
            nat.check(self.lib.sk_verify_regions(t.data_ptr(), n, self.d_bad.data_ptr(),
                                                 torch.cuda.current_stream().cuda_stream))
        return int(self.d_bad.item())

    def close(self, group=None):
        """Unmap the peers' slabs, then free this rank's own.  With world > 1
        every rank must have unmapped a slab before its owner frees it
        (cudaIpcCloseMemHandle before cudaFree), so a barrier separates the
        two halves; all ranks must call close()."""
        torch.cuda.synchronize()
        for p in self.opened:
            self.lib.sk_ipc_close_handle(p)
        self.opened = []
        if self.world > 1:
            import torch.distributed as dist

            dist.barrier(group=group if group is not None else self.group)
        self.slab.free()


def required_layout(mapping, model, inherited_by_pipeline=None, inventory_cls=None):
    """new GpuRef -> required context (required_context_with_cache, mapping.py:155-169)."""
    from .mapping import required_context_with_cache

    out = {}
    for gpu, pos in mapping.assignment.items():
        inh = (inherited_by_pipeline or {}).get(pos.pipeline)
        out[gpu] = required_context_with_cache(mapping.config, pos, model, inh, inventory_cls)
    return out


def common_k(*layouts) -> int:
    K = 1
    for lay in layouts:
        for inv in lay.values():
            for _, lo, hi in inv.model_shards:
                K = lcm(K, lo.denominator, hi.denominator)
    return K


# ---------------------------------------------------------------------------
# synthetic reshard problems (bf16-shaped geometries)

GPT20B_BF16 = ("gpt-20b-bf16", 44, 12 * 6144 * 6144 * 2, 2 * 6144 * 2)
LLAMA30B_BF16 = ("llama-30b-bf16", 60, (4 * 6656 * 6656 + 3 * 6656 * 17920) * 2, 2 * 6656 * 2)
U_MAX = 4e9   # the B_S scenario's migration buffer cap (data/scenario_bs.json:14)


def make_reshard_problem(geom, old_shape, new_shape, batch: int = 8, seq: int = 2048,
                         u_max: float | None = U_MAX, mapper=None, with_mapping: bool = False):
    """One GPU per instance (G=1), old config laid out positionally on i-0..i-(N-1),
    `batch` cached requests of `seq` tokens per old pipeline, identity
    inheritance.  The mapping and plan come from this package's device mapper
    (or `mapper`, same signature) and native planner (memory-optimised layer
    order under `u_max`).
    Returns (plan, old_layout, new_required, model, refs[, mapping])."""
    from . import domain as dm
    from .mapping import default_inheritance, map_devices
    from .planner import plan_migration

    name, L, bpl, kv = geom
    model = dm.ModelSpec(name, L, bpl, kv)
    old = dm.ParallelConfig(*old_shape, batch)
    new = dm.ParallelConfig(*new_shape, batch)
    n = max(old.gpus, new.gpus)
    reqs = {d: [dm.RequestSpec(id=f"r{d}-{j:02d}", arrival_time=0.0, s_in=seq, s_out=seq)
                for j in range(batch)] for d in range(1, old.data_parallel + 1)}
    slots = dm.positions(old)
    insts, layout = [], {}
    for k in range(n):
        ref = (f"i-{k}", 0)
        if k < len(slots):
            pos = slots[k]
            base = dm.required_context(old, pos, model)
            cache = tuple((r.id, layer, lo, hi, seq) for r in reqs[pos.pipeline]
                          for layer, lo, hi in base.model_shards)
            inv = dm.ContextInventory(base.model_shards, cache)
        else:
            inv = dm.ContextInventory()
        layout[ref] = inv
        insts.append(dm.InstanceState(id=f"i-{k}", kind="spot", gpus=1, gpu_inventories=[inv]))
    inh = default_inheritance(old.data_parallel, new.data_parallel)
    mapping = (mapper or map_devices)(insts, new, model, 1, inheritance=inh, requests_by_old_pipeline=reqs)
    inherited = {inh[d]: [(r.id, seq) for r in reqs[d]] for d in sorted(reqs) if d in inh}
    plan = plan_migration(mapping, layout, model, u_max=u_max, inherited_by_pipeline=inherited)
    need = required_layout(mapping, model, inherited, dm.ContextInventory)
    for ref in layout:
        need.setdefault(ref, dm.ContextInventory())
    refs = [(f"i-{k}", 0) for k in range(n)]
    if with_mapping:
        return plan, layout, need, model, refs, mapping
    return plan, layout, need, model, refs
