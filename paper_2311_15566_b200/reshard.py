"""Migration executor (K3): carry out a MigrationPlan's weight + KV reshard on
the GPUs of one box.

The reference only plans and costs a migration (migration.py:311-384,
costmodel.py:189-260); the paper's engine executes it with batched async NCCL
send/recv plus CUDA IPC.  Here every `Transfer` becomes one
contiguous byte-range copy that the DESTINATION GPU pulls from the source
GPU's context slab over NVLink (peer-mapped with CUDA IPC, one process per
GPU), issued by the `k_copy` kernel (`sk_copy_batched`) in plan order; the
destination's own reusable bytes are copied locally into the new layout.

Byte geometry (SURVEY.md finding 8).  A layer's parameters are one flat byte
array of `bytes_per_layer` bytes; tensor shard [lo, hi) owns bytes
[lo*B, hi*B) of it.  A request's KV cache of one layer is one flat array of
kv_bytes_per_token_per_layer * tokens bytes laid out [head][K|V][tok][hd], so
a head-fraction shard [lo, hi) is again the contiguous byte range [lo*X, hi*X).
Every shard boundary must therefore be a whole number of 8-byte words (checked).
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
ALIGN = 256


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


@dataclass
class Slab:
    """Byte layout of one GPU's context: regions in inventory order."""

    model: dict = field(default_factory=dict)   # layer -> [(lo, hi, where)]  (lo, hi: Fractions)
    cache: dict = field(default_factory=dict)   # (rid, layer) -> [(lo, hi, tokens, where)]
    regions: list = field(default_factory=list)  # (where, bytes, key, base); where = (space, offset)
    bytes: int = 0


def _span(frac: Fraction, total: int) -> int:
    v = frac * total
    if v.denominator != 1 or v.numerator % 8:
        raise ValueError(f"shard boundary {frac} of a {total}-byte object is not 8-byte aligned")
    return v.numerator


def build_slab(inv, model, rid_index: dict, seed: int, reuse: "Slab | None" = None) -> Slab:
    """Offsets of an inventory's shards.  With `reuse` (the same GPU's old
    slab), a shard contained in one the GPU already holds is aliased in place
    (("old", offset): no allocation, no copy); everything else gets space in
    the new slab (("new", offset))."""
    s = Slab()
    off = 0
    B, kv = model.bytes_per_layer, model.kv_bytes_per_token_per_layer
    for layer, lo, hi in inv.model_shards:
        a, b = _span(lo, B), _span(hi, B)
        hit = None
        if reuse is not None:
            hit = next((e for e in reuse.model.get(layer, ()) if e[0] <= lo and hi <= e[1]), None)
        where = ("old", hit[2][1] + _span(lo - hit[0], B)) if hit else ("new", off)
        s.model.setdefault(layer, []).append((lo, hi, where))
        s.regions.append((where, b - a, model_key(seed, layer), a))
        if not hit:
            off += (b - a + ALIGN - 1) // ALIGN * ALIGN
    for rid, layer, lo, hi, tok in inv.cache_shards:
        X = kv * tok
        a, b = _span(lo, X), _span(hi, X)
        hit = None
        if reuse is not None:
            hit = next((e for e in reuse.cache.get((rid, layer), ())
                        if e[0] <= lo and hi <= e[1] and e[2] == tok), None)
        where = ("old", hit[3][1] + _span(lo - hit[0], X)) if hit else ("new", off)
        s.cache.setdefault((rid, layer), []).append((lo, hi, tok, where))
        s.regions.append((where, b - a, cache_key(seed, rid_index[rid], layer), a))
        if not hit:
            off += (b - a + ALIGN - 1) // ALIGN * ALIGN
    s.bytes = off
    return s


def _find(entries, lo, hi):
    for e in entries:
        if e[0] <= lo and hi <= e[1]:
            return e
    return None


def plan_copies(plan, old_layout, new_required, model, seed: int = 1, with_rounds: bool = False):
    """Per destination GPU: the ordered byte-range copies that realise `plan`
    (the plan's transfers in plan order, then local reuse).
    Returns (old slabs, new slabs, {dst gpu: [(src gpu, src_off, dst_off, bytes)]}); with
    `with_rounds` also {dst gpu: [plan action index per copy]} (-1 = local reuse)."""
    rids = sorted({r for inv in list(old_layout.values()) + list(new_required.values())
                   for r, *_ in inv.cache_shards})
    rid_index = {r: i for i, r in enumerate(rids)}
    old = {g: build_slab(inv, model, rid_index, seed) for g, inv in old_layout.items()}
    new = {g: build_slab(inv, model, rid_index, seed, old.get(g)) for g, inv in new_required.items()}
    B, kv = model.bytes_per_layer, model.kv_bytes_per_token_per_layer
    copies: dict = {g: [] for g in new}
    rounds: dict = {g: [] for g in new}
    for a_idx, action in enumerate(plan.actions):
        for t in action.transfers:
            if t.kind == "model":
                src = _find(old[t.src].model.get(t.layer, ()), t.lo, t.hi)
                dst = _find(new[t.dst].model.get(t.layer, ()), t.lo, t.hi)
                unit = B
            else:
                src = _find([e for e in old[t.src].cache.get((t.request, t.layer), ()) if e[2] == t.tokens],
                            t.lo, t.hi)
                dst = _find(new[t.dst].cache.get((t.request, t.layer), ()), t.lo, t.hi)
                unit = kv * t.tokens
            if src is None or dst is None:
                raise ValueError(f"transfer {t} does not fit the slab layouts")
            n = _span(t.hi - t.lo, unit)
            if n != t.bytes:
                raise ValueError(f"transfer bytes {t.bytes} != geometry {n}")
            if dst[-1][0] != "new":
                raise ValueError(f"transfer {t} targets a shard its destination already holds")
            copies[t.dst].append((t.src, src[-1][1] + _span(t.lo - src[0], unit),
                                  dst[-1][1] + _span(t.lo - dst[0], unit), n))
            rounds[t.dst].append(a_idx)
    # local reuse: every needed piece the GPU already holds (the plan's "kept" bytes)
    for g, slab in new.items():
        have = old.get(g)
        local = []
        if have is not None:
            for layer, ents in slab.model.items():
                for lo, hi, (space, off) in ents:
                    if space != "new":
                        continue   # aliased in place: nothing to move
                    for olo, ohi, (_, ooff) in have.model.get(layer, ()):
                        a, b = max(lo, olo), min(hi, ohi)
                        if b > a:
                            local.append((g, ooff + _span(a - olo, B), off + _span(a - lo, B),
                                          _span(b - a, B)))
            for key, ents in slab.cache.items():
                for lo, hi, tok, (space, off) in ents:
                    if space != "new":
                        continue
                    for olo, ohi, otok, (_, ooff) in have.cache.get(key, ()):
                        a, b = max(lo, olo), min(hi, ohi)
                        if b > a and otok == tok:
                            X = kv * tok
                            local.append((g, ooff + _span(a - olo, X), off + _span(a - lo, X),
                                          _span(b - a, X)))
        # NVLink pulls first (the scarce link), local reuse copies after them:
        # the copy kernel's CTAs take chunks in list order, so the local HBM
        # copies fill in behind the remote traffic instead of delaying it
        copies[g] = copies[g] + local
        rounds[g] = rounds[g] + [-1] * len(local)
    if with_rounds:
        return old, new, copies, rounds
    return old, new, copies


def issue_lists(copies: dict, owner: dict, mode: str = "pull", rounds: dict | None = None) -> dict:
    """Which rank issues which copy: pull -> the destination GPU's rank, push ->
    the source GPU's rank; local (same-GPU) copies always by the owner.
    Returns {rank: [(src, dst, src_off, dst_off, bytes)]} in plan order (with
    `rounds`, each entry carries its plan action index as a 6th field)."""
    out: dict = {}
    for dst, lst in copies.items():
        for i, (src, soff, doff, n) in enumerate(lst):
            issuer = dst if (mode == "pull" or src == dst) else src
            row = (src, dst, soff, doff, n) if rounds is None else (src, dst, soff, doff, n, rounds[dst][i])
            out.setdefault(owner[issuer], []).append(row)
    return out


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


class ReshardExecutor:
    """Executes one plan on this process's GPU(s).

    `owner[gpu_ref]` = rank hosting that GPU.  With one process per GPU the
    ranks exchange CUDA IPC handles of their old-context slabs through
    torch.distributed (gloo/nccl object all-gather) and each destination pulls
    from peers over NVLink.  With world == 1 every GPU ref is emulated on the
    local device (same code path, local pointers) -- used by the tests.
    """

    def __init__(self, plan, old_layout, new_required, model, owner: dict, rank: int = 0,
                 world: int = 1, seed: int = 1, group=None, mode: str = "pull", chunk: int = CHUNK):
        if mode not in ("pull", "push"):
            raise ValueError("mode must be 'pull' or 'push'")
        self.lib = nat.load()
        self.rank, self.world, self.mode = rank, world, mode
        self.old, self.new, copies, rounds = plan_copies(plan, old_layout, new_required, model, seed,
                                                         with_rounds=True)
        self.plan = plan
        self.mine = [g for g, r in owner.items() if r == rank]
        self.old_mem = {g: _Mem(self.old[g].bytes) for g in self.mine if g in self.old}
        self.new_mem = {g: _Mem(self.new[g].bytes) for g in self.mine if g in self.new}
        # device addresses usable from this GPU: own slabs + peer-mapped slabs
        self.old_ptr = {g: m.ptr for g, m in self.old_mem.items()}
        self.new_ptr = {g: m.ptr for g, m in self.new_mem.items()}
        self.opened = []
        if world > 1:
            import torch.distributed as dist

            handles = {}
            for tag, mems in (("old", self.old_mem), ("new", self.new_mem)):
                for g, m in mems.items():
                    h = ctypes.create_string_buffer(64)
                    nat.check(self.lib.sk_ipc_get_handle(m.ptr, h))
                    handles[(tag, g)] = h.raw
            gathered = [None] * world
            dist.all_gather_object(gathered, handles, group=group)
            for r, hs in enumerate(gathered):
                if r == rank:
                    continue
                for (tag, g), raw in hs.items():
                    if (tag == "old") != (mode == "pull"):
                        continue   # pull maps peers' old slabs, push their new slabs
                    p = ctypes.c_void_p()
                    nat.check(self.lib.sk_ipc_open_handle(raw, ctypes.byref(p)))
                    (self.old_ptr if tag == "old" else self.new_ptr)[g] = p.value
                    self.opened.append(p.value)
        self.peer_ptr = self.old_ptr
        dev = torch.device("cuda", torch.cuda.current_device())
        self._issued = issue_lists(copies, owner, mode, rounds).get(rank, ())
        self._dev = dev
        self.local_bytes = sum(n for src, dst, _, _, n, _ in self._issued if src == dst)
        self.remote_bytes = sum(n for src, dst, _, _, n, _ in self._issued if src != dst)
        self.set_chunk(chunk)
        self.d_fill = self._regions(self.old, self.old_mem, self.old_mem, dev)
        self.d_check = self._regions(self.new, self.new_mem, self.old_mem, dev)
        self.d_bad = torch.zeros(1, dtype=torch.int64, device=dev)

    def set_chunk(self, chunk: int = CHUNK):
        """(Re)build the device copy lists with `chunk`-byte pieces."""
        rows, rnd = [], []
        for src, dst, soff, doff, n, r in self._issued:
            sbase, dbase = self.old_ptr[src], self.new_ptr[dst]
            for c in range(0, n, chunk):
                rows.append((sbase + soff + c, dbase + doff + c, min(chunk, n - c)))
                rnd.append(r)

        def to_dev(rs):
            arr = np.array(rs, dtype=np.uint64).reshape(-1, 3) if rs else np.zeros((0, 3), np.uint64)
            cp = np.zeros(len(arr), dtype=nat.COPY)
            if len(arr):
                cp["src"], cp["dst"], cp["bytes"] = arr[:, 0], arr[:, 1], arr[:, 2]
            return (torch.from_numpy(cp.view(np.uint8)).to(self._dev) if len(cp) else None), len(cp)

        # one-launch order: NVLink transfers in plan order, local reuse last
        self.d_copies, self.n_copies = to_dev(rows)
        # progressive order: local reuse first, then round by round
        order = sorted(range(len(rows)), key=lambda i: (rnd[i], i))
        self.d_prog, _ = to_dev([rows[i] for i in order])
        ro = [rnd[i] for i in order]
        self.round_ranges = []   # (action index, begin, end) in the progressive array
        i = 0
        while i < len(ro):
            j = i
            while j < len(ro) and ro[j] == ro[i]:
                j += 1
            self.round_ranges.append((ro[i], i, j))
            i = j

    @staticmethod
    def _regions(slabs, mems, old_mems, dev):
        rows = []
        for g, m in mems.items():
            for where, n, key, base in slabs[g].regions:
                space, off = where
                ptr = (m.ptr if space == "new" else old_mems[g].ptr) + off
                rows.append((ptr, n, key, base))
        reg = np.zeros(len(rows), dtype=nat.REGION)
        for i, r in enumerate(rows):
            reg[i] = r
        return (torch.from_numpy(reg.view(np.uint8)).to(dev), len(rows)) if rows else (None, 0)

    def fill_old(self):
        t, n = self.d_fill
        if n:
            nat.check(self.lib.sk_fill_regions(t.data_ptr(), n, torch.cuda.current_stream().cuda_stream))

    def run(self, n_ctas: int = 0):
        """The reshard: one launch of k_copy over this rank's copies, in plan order."""
        if self.n_copies:
            nat.check(self.lib.sk_copy_batched(self.d_copies.data_ptr(), self.n_copies, n_ctas,
                                               torch.cuda.current_stream().cuda_stream))

    def run_progressive(self, n_ctas: int = 0) -> dict:
        """Round-by-round execution with a CUDA event per plan round, so a
        stage can start serving as soon as the round its `start_stage` marker
        follows has landed (PAPER.md:497's per-tensor readiness; the marker
        placement is migration.py:352-371).  Returns {stage: event} recorded on
        the current stream: this rank's copies for every round up to that
        marker are complete when the event fires."""
        st = torch.cuda.current_stream()
        begin = torch.cuda.Event(enable_timing=True)
        begin.record(st)
        ptr = self.d_prog.data_ptr() if self.d_prog is not None else 0
        ranges = {r: (b, e) for r, b, e in self.round_ranges}

        def launch(r):
            b, e = ranges[r]
            nat.check(self.lib.sk_copy_batched(ptr + 24 * b, e - b, n_ctas, st.cuda_stream))

        if -1 in ranges:
            launch(-1)  # local reuse first (HBM only)
        last = torch.cuda.Event(enable_timing=True)
        last.record(st)
        ready = {}
        for idx, action in enumerate(self.plan.actions):
            if action.kind == "start_stage":
                ready[action.stage] = last
                continue
            if idx in ranges:
                launch(idx)
            last = torch.cuda.Event(enable_timing=True)
            last.record(st)
        self.progress_begin = begin
        return ready

    def verify(self) -> int:
        """Mismatching 8-byte words in this rank's new slabs (0 = byte-identical)."""
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

            dist.barrier(group=group)
        for m in list(self.old_mem.values()) + list(self.new_mem.values()):
            m.free()


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


def make_reshard_problem(geom, old_shape, new_shape, batch: int = 8, seq: int = 2048):
    """One GPU per instance (G=1), old config laid out positionally on i-0..i-(N-1),
    `batch` cached requests of `seq` tokens per old pipeline, identity
    inheritance.  The mapping and plan come from this package's device mapper
    and native planner.  Returns (plan, old_layout, new_required, model, refs)."""
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
    mapping = map_devices(insts, new, model, 1, inheritance=inh, requests_by_old_pipeline=reqs)
    inherited = {inh[d]: [(r.id, seq) for r in reqs[d]] for d in sorted(reqs) if d in inh}
    plan = plan_migration(mapping, layout, model, inherited_by_pipeline=inherited)
    need = required_layout(mapping, model, inherited, dm.ContextInventory)
    for ref in layout:
        need.setdefault(ref, dm.ContextInventory())
    return plan, layout, need, model, [(f"i-{k}", 0) for k in range(n)]
