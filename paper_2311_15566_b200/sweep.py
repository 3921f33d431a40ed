"""Batched preemption sweep: many device-mapping plans per device call.

This is the batched GPU entry point of the mapping path:
for one target size N, every (old, new) pair of candidate (D,P,M) configs
x S random preemption sets.  A plan is described compactly (sk_sweep_desc:
old config, pool size, an alive-instance bitmask, per-old-pipeline cached
token sums); `sk_sweep_expand` turns it into rows/segments on the device and
`sk_map_batched` solves it.  Host -> device traffic per plan is ~0.2 KB;
device -> host is the assignment (4 B per GPU row) + total_weight.

Synthetic-input semantics: instances i-0..i-(n-1) with
n = ceil(max(old, new GPUs) / G) + 4; the old config laid out positionally on
them; k ~ U{1..4} instances preempted (without replacement); each old
pipeline carries `batch` cached requests of 512 + U{0..128} tokens; identity
inheritance on min(D_old, D_new).
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from math import lcm

import numpy as np
import torch

from . import _native as nat

# (L, bytes_per_layer, kv_bytes_per_token_per_layer) from the reference profiles
GPT20B = (44, 1693181818, 24576)      # data/profile_gpt20b.json:3-7
LLAMA30B = (60, 1863333333, 26624)    # data/profile_llama30b.json:3-7
OPT67B = (32, 781250000, 16384)       # data/profile_opt67b.json:3-7
# candidate (P, M) shapes = the profiles' t_dec keys
GPT20B_SHAPES = ((2, 8), (3, 4), (4, 4), (4, 8), (6, 2), (6, 4))
LLAMA30B_SHAPES = ((2, 8), (4, 4), (4, 8), (8, 2))
OPT67B_SHAPES = ((1, 4), (2, 2), (2, 4), (4, 2))
MODELS = {"gpt-20b": (GPT20B, GPT20B_SHAPES), "llama-30b": (LLAMA30B, LLAMA30B_SHAPES),
          "opt-6.7b": (OPT67B, OPT67B_SHAPES)}


def sweep_configs(n_positions: int, shapes=GPT20B_SHAPES):
    return [(n_positions // (P * M), P, M) for P, M in shapes if n_positions // (P * M) >= 1]


@dataclass
class SweepBatch:
    """Host arrays of one batch of sweep plans (all numpy, ready for one H2D)."""

    desc: np.ndarray    # SWEEP_DESC[Q]
    plans: np.ndarray   # PLAN[Q]
    alive: np.ndarray   # uint32 bitmask words
    tok: np.ndarray     # int64 per old pipeline token sums
    n_positions: int

    @property
    def n_plans(self) -> int:
        return len(self.plans)

    @property
    def rows(self) -> int:
        return int(self.plans["rows"].sum())

    def stats(self):
        g = self.plans["group"].astype(np.int64)
        R = self.plans["rows"].astype(np.int64)
        C = (self.plans["D"] * self.plans["P"] * self.plans["M"]).astype(np.int64)
        nA, nB = R // g, C // g
        return dict(rows=R, cols=C, nA=nA, nB=nB, n=np.maximum(nA, nB), pairs=nA * nB)


def make_sweep(n_positions: int, sets_per_pair: int, seed: int = 0, G: int = 4, batch: int = 4,
               model=GPT20B, shapes=GPT20B_SHAPES, fused_sum: bool = False,
               pairs=None) -> SweepBatch:
    """All (old, new) config pairs x `sets_per_pair` preemption sets."""
    rng = np.random.default_rng(seed)
    cfgs = sweep_configs(n_positions, shapes)
    if pairs is None:
        pairs = [(o, n) for o in cfgs for n in cfgs]
    L, bpl, kv = model
    descs, plans, alive_parts, tok_parts = [], [], [], []
    alive_off = tok_off = 0
    for old, new in pairs:
        oD, oP, oM = old
        nD, nP, nM = new
        S = sets_per_pair
        n_inst = -(-max(oD * oP * oM, nD * nP * nM) // G) + 4
        k = rng.integers(1, 5, size=S)
        ranks = rng.random((S, n_inst)).argsort(axis=1).argsort(axis=1)
        alive = ranks >= k[:, None]                            # drop k instances
        words = (n_inst + 31) // 32
        bits = np.zeros((S, words * 32), dtype=bool)
        bits[:, :n_inst] = alive
        packed = np.packbits(bits.reshape(S, words, 32), axis=2, bitorder="little")
        alive_w = packed.reshape(S, words * 4).view(np.uint32).reshape(S, words)
        toks = rng.integers(512, 641, size=(S, oD, batch)).sum(axis=2).astype(np.int64)
        rows = alive.sum(axis=1).astype(np.int64) * G
        group = min(G, nM)
        K = lcm(oM, nM)
        d = np.zeros(S, dtype=nat.SWEEP_DESC)
        d["oD"], d["oP"], d["oM"], d["G"], d["n_inst"] = oD, oP, oM, G, n_inst
        d["alive_off"] = alive_off + np.arange(S) * words
        d["tok_off"] = tok_off + np.arange(S) * oD
        d["bpl"], d["kv"] = bpl, kv
        p = np.zeros(S, dtype=nat.PLAN)
        p["rows"], p["D"], p["P"], p["M"], p["L"], p["K"] = rows, nD, nP, nM, L, K
        p["group"] = group
        p["flags"] = nat.SK_PLAN_FUSED_SUM if fused_sum else 0
        descs.append(d)
        plans.append(p)
        alive_parts.append(alive_w.reshape(-1))
        tok_parts.append(toks.reshape(-1))
        alive_off += S * words
        tok_off += S * oD
    desc = np.concatenate(descs)
    plan = np.concatenate(plans)
    # largest outer problems first: contiguous size classes for the outer-KM
    # launches and longest-first scheduling inside each launch
    R = plan["rows"].astype(np.int64)
    g = plan["group"].astype(np.int64)
    C = (plan["D"] * plan["P"] * plan["M"]).astype(np.int64)
    n_outer = np.maximum(R // g, C // g)
    order = np.lexsort((np.arange(len(plan)), -(n_outer * (C // g)), -n_outer))
    desc, plan = desc[order], plan[order]
    desc["plan"] = np.arange(len(plan))
    R = plan["rows"].astype(np.int64)
    g = plan["group"].astype(np.int64)
    C = (plan["D"] * plan["P"] * plan["M"]).astype(np.int64)
    pairs_n = (R // g) * (C // g)
    plan["row_base"] = np.concatenate([[0], np.cumsum(R)[:-1]])
    plan["out_off"] = plan["row_base"]
    plan["f_off"] = np.concatenate([[0], np.cumsum(pairs_n)[:-1]])
    if R.sum() * 2 >= 2**31:
        raise ValueError("sweep batch too large for int32 segment indices; split it")
    return SweepBatch(desc, plan, np.concatenate(alive_parts).astype(np.uint32),
                      np.concatenate(tok_parts).astype(np.int64), n_positions)


def _align(n: int, a: int = 256) -> int:
    return (n + a - 1) // a * a


def cpl_bucket(n: int):
    """(warps per plan, columns per thread) of the outer-KM template the
    dispatch picks for size n (mirrors outer_dispatch in spotkm.cu)."""
    if n > 4095:
        return (32, 0)   # k_outer_huge: one 1024-thread CTA per plan
    need = max(1, (n + 31) // 32)
    if need <= 6:
        return (1, need)
    if need <= 8:
        return (1, 8)
    need2 = (n + 63) // 64
    if need2 <= 8:
        return (2, 5 if need2 <= 5 else (6 if need2 <= 6 else 8))
    need4 = (n + 127) // 128
    for c in (3, 4, 5, 6, 8, 12, 16):
        if need4 <= c:
            return (4, c)
    need8 = (n + 255) // 256
    return (8, 12) if need8 <= 12 else (8, 16)


def outer_classes(n_outer: np.ndarray):
    """Contiguous (start, stop, max_n) ranges of plans sharing one outer-KM
    template; plans must be sorted by n descending."""
    out = []
    start = 0
    N = len(n_outer)
    while start < N:
        b = cpl_bucket(int(n_outer[start]))
        stop = start + 1
        while stop < N and cpl_bucket(int(n_outer[stop])) == b:
            stop += 1
        out.append((start, stop, int(n_outer[start:stop].max())))
        start = stop
    return out


class SweepRunner:
    """Device buffers for one SweepBatch; `run()` = one pass of the hot path.

    Inputs live in one pinned host buffer and one device buffer; `upload()`
    is the H2D step, `solve()` the kernels (expand + fused inner KM + outer
    KM), `download()` the D2H of assignments and totals.
    """

    def __init__(self, batch: SweepBatch, device=None, stream=None, scratch=None,
                 reserve=(0, 0)):
        """scratch: another SweepRunner whose device scratch (row_ptr, segments,
        fused weights, permutations) this one reuses when large enough -- for
        sweeps run as consecutive chunks on one stream; reserve: minimum
        (rows, fused pairs) capacity to allocate for such sharing."""
        self.lib = nat.load()
        self.b = batch
        self.dev = torch.device(device or "cuda")
        st = batch.stats()
        self.max_pairs = int(st["pairs"].max())
        self.max_n = int(st["n"].max())
        self.classes = outer_classes(st["n"])
        self.class_rows = [int(st["rows"][a:b].max()) for a, b, _ in self.classes]
        f_off = batch.plans["f_off"].astype(np.int64)
        self.class_na = [int(st["nA"][a:b].max()) for a, b, _ in self.classes]
        self.class_nb = [int(st["nB"][a:b].max()) for a, b, _ in self.classes]
        self.class_gmask = [int(np.bitwise_or.reduce(1 << batch.plans["group"][a:b].astype(np.int64)))
                            for a, b, _ in self.classes]
        self.max_rows = int(st["rows"].max())
        self.gmask = int(np.bitwise_or.reduce(1 << batch.plans["group"].astype(np.int64)))
        parts = [batch.desc, batch.plans, batch.alive, batch.tok]
        self.offs, total = [], 0
        for a in parts:
            self.offs.append(total)
            total = _align(total + a.nbytes)
        self.h_in = torch.empty(total, dtype=torch.uint8, pin_memory=True)
        hv = self.h_in.numpy()
        for a, o in zip(parts, self.offs):
            hv[o:o + a.nbytes] = np.frombuffer(a.tobytes(), dtype=np.uint8)
        self.h2d_bytes = total
        self.d_in = torch.empty(total, dtype=torch.uint8, device=self.dev)
        R = batch.rows
        Q = batch.n_plans
        pairs = max(int(st["pairs"].sum()), 1, reserve[1])
        Rcap = max(R, reserve[0])

        def buf(name, n, dtype):
            old = getattr(scratch, name, None)
            if old is not None and old.numel() >= n:
                return old
            return torch.empty(n, dtype=dtype, device=self.dev)

        self.row_ptr = buf("row_ptr", Rcap + 1, torch.int32)
        self.segs = buf("segs", 2 * Rcap * 32, torch.uint8)
        self.fused = buf("fused", pairs, torch.float64)
        self.perm = buf("perm", pairs, torch.int32)
        self.out_bytes = _align(8 * Q + 4 * R)
        self.d_out = torch.empty(self.out_bytes, dtype=torch.uint8, device=self.dev)
        self.h_out = torch.empty(self.out_bytes, dtype=torch.uint8, pin_memory=True)
        self.d2h_bytes = 8 * Q + 4 * R
        # per class: the byte ranges of its totals and assignments in d_out
        rb = batch.plans["row_base"].astype(np.int64)
        rows = batch.plans["rows"].astype(np.int64)
        self._class_out = [((8 * a, 8 * b),
                            (8 * Q + 4 * int(rb[a]), 8 * Q + 4 * int(rb[b - 1] + rows[b - 1])))
                           for a, b, _ in self.classes]
        # global code scratch for the big size classes (sk_outer_codes_bytes);
        # the classes run concurrently, so each gets its own slice
        # coded K2: k_fuse writes one-byte codes + a per-plan dictionary instead
        # of the double matrix (every codable class then needs the code scratch
        # and dictionaries) -- for sweeps whose largest outer problem has n >= 96 (measured per
        # sweep size, all classes coded vs none: -6% at 64 positions (n <= 38),
        # -2% at 128 (n <= 70), +4% at 256, +7.5% at 512, +5% at 1,024; per-class
        # mixes measured no better).  SK_PRECODED=0 / 1 forces it off / on.
        mode = os.environ.get("SK_PRECODED", "auto")
        self.precoded = mode == "1" or (mode != "0" and self.max_n >= 96)
        need, dneed, coded = [], [], []
        for (a, b, mn), rows in zip(self.classes, self.class_rows):
            d = ctypes.c_int64(0)
            use = self.precoded
            pc = int(self.lib.sk_precoded_bytes(b - a, mn, ctypes.byref(d))) if use else 0
            coded.append(pc > 0)
            need.append(pc if pc > 0 else int(self.lib.sk_outer_codes_bytes(b - a, mn, rows)))
            dneed.append(_align(int(d.value)) if pc > 0 else 0)
        self.class_coded = coded
        self.codes_off = np.concatenate([[0], np.cumsum(need)]).astype(np.int64)
        self.codes_need = need
        self.codes = buf("codes", max(int(self.codes_off[-1]), 1), torch.uint8)
        self.dict_off = np.concatenate([[0], np.cumsum(dneed)]).astype(np.int64)
        self.dict_need = dneed
        self.dict = buf("dict", max(int(self.dict_off[-1]) // 8, 1), torch.int64)
        self.stream = stream
        # one side stream per outer-KM size class so the classes' tails overlap
        self.side = [torch.cuda.Stream(self.dev) for _ in self.classes]
        # SK_EXPAND_PER_CLASS=1: expand each class on its own stream (measured:
        # +2% at 64 positions, -2% at 256; default: one expansion, then fork)
        self.expand_per_class = os.environ.get("SK_EXPAND_PER_CLASS", "0") == "1"

    @property
    def launches_per_solve(self) -> int:
        """Kernel launches of one solve(): expand and fuse split the plans into
        chunks of at most 65,535 (grid y); one fuse launch per group size; a
        coded class adds the overflow list and one overflow re-fuse per regular
        group size."""
        ch = lambda q: -(-q // 65535)  # noqa: E731
        n = 0 if self.expand_per_class else ch(self.b.n_plans)
        for (a, b, _), m, coded in zip(self.classes, self.class_gmask, self.class_coded):
            n += bin(m).count("1") * ch(b - a) + 1 + (ch(b - a) if self.expand_per_class else 0)
            if coded:
                n += 1 + bin(m & 0x1fe).count("1")
        return n

    def _s(self) -> int:
        return (self.stream or torch.cuda.current_stream(self.dev)).cuda_stream

    def upload(self):
        self.d_in.copy_(self.h_in, non_blocking=True)

    def solve(self, steps=None, profile=None, download: bool = False):
        """One pass of the hot path on the runner's stream: expand, then per
        outer-KM size class the fused inner KMs and the outer KM, each class
        on its own stream so the classes' tails overlap.

        steps: optional int64 device tensor [2*Q] receiving {Dijkstra steps,
        cost loads} per plan.  profile: optional dict; when given, the launches
        are serialised on the main stream and bracketed with CUDA events so
        per-kernel times can be read back (profile["events"]).  download: also
        copy each class's results to the pinned host buffer on its stream as
        soon as its outer KM ends (overlaps the D2H with the other classes)."""
        base = self.d_in.data_ptr()
        p_desc, p_plans, p_alive, p_tok = (base + o for o in self.offs)
        Q = self.b.n_plans
        main = self.stream or torch.cuda.current_stream(self.dev)
        evs = []

        def mark(tag):
            if profile is not None:
                e = torch.cuda.Event(enable_timing=True)
                e.record(main)
                evs.append((tag, e))

        mark("start")
        if not self.expand_per_class:
            rc = self.lib.sk_sweep_expand(p_desc, Q, p_alive, p_tok, p_plans, self.row_ptr.data_ptr(),
                                          self.segs.data_ptr(), self.max_rows, main.cuda_stream)
            nat.check(rc)
            mark("k_sweep_expand")
        out = self.d_out.data_ptr()
        fork = torch.cuda.Event()
        fork.record(main)
        for c, ((a, b, mn), side) in enumerate(zip(self.classes, self.side)):
            st = side
            if profile is None:
                side.wait_event(fork)
            else:
                st = main
            if self.expand_per_class:
                # this class's rows only, on its own stream: the first class
                # starts after its own expansion, later ones overlap it
                rc = self.lib.sk_sweep_expand(p_desc + 48 * a, b - a, p_alive, p_tok, p_plans,
                                              self.row_ptr.data_ptr(), self.segs.data_ptr(),
                                              self.class_rows[c], st.cuda_stream)
                nat.check(rc)
                mark(f"k_sweep_expand[{c}]")
            codes = self.codes.data_ptr() + int(self.codes_off[c])
            dct = self.dict.data_ptr() + int(self.dict_off[c])
            if self.class_coded[c]:
                rc = self.lib.sk_map_fuse_coded(p_plans + 64 * a, b - a, self.row_ptr.data_ptr(),
                                                self.segs.data_ptr(), self.fused.data_ptr(),
                                                self.perm.data_ptr(), self.class_na[c], self.class_nb[c],
                                                self.class_gmask[c], codes, self.codes_need[c], dct,
                                                self.dict_need[c], st.cuda_stream)
            else:
                rc = self.lib.sk_map_fuse(p_plans + 64 * a, b - a, self.row_ptr.data_ptr(),
                                          self.segs.data_ptr(), self.fused.data_ptr(),
                                          self.perm.data_ptr(), self.class_na[c], self.class_nb[c],
                                          self.class_gmask[c], 0, 0, st.cuda_stream)
            nat.check(rc)
            mark(f"k_fuse[{c}]")
            outer = self.lib.sk_map_outer_coded if self.class_coded[c] else self.lib.sk_map_outer_codes
            extra = (dct,) if self.class_coded[c] else ()
            rc = outer(p_plans + 64 * a, b - a, self.row_ptr.data_ptr(), self.segs.data_ptr(),
                       self.fused.data_ptr(), self.perm.data_ptr(), out + 8 * Q, out + 8 * a,
                       0 if steps is None else steps.data_ptr() + 16 * a, mn, self.class_rows[c],
                       codes, self.codes_need[c], *extra, st.cuda_stream)
            nat.check(rc)
            mark(f"k_outer[{c}]")
            if download:
                with torch.cuda.stream(st):
                    for lo, hi in self._class_out[c]:
                        self.h_out[lo:hi].copy_(self.d_out[lo:hi], non_blocking=True)
            if profile is None:
                done = torch.cuda.Event()
                done.record(side)
                main.wait_event(done)
        if profile is not None:
            profile["events"] = evs

    @staticmethod
    def kernel_ms(profile, per_class: bool = False):
        """Per-kernel milliseconds from a profiled solve (after synchronize)."""
        evs = profile["events"]
        out: dict[str, float] = {}
        for (_, e0), (tag, e1) in zip(evs, evs[1:]):
            if not per_class:
                tag = tag.split("[")[0]
            out[tag] = out.get(tag, 0.0) + e0.elapsed_time(e1)
        return out

    def download(self):
        self.h_out.copy_(self.d_out, non_blocking=True)

    def results(self):
        """(assign int32[sum R], totals float64[Q]) -- call after synchronize."""
        h = self.h_out.numpy()
        Q, R = self.b.n_plans, self.b.rows
        return h[8 * Q:8 * Q + 4 * R].view(np.int32).copy(), h[:8 * Q].view(np.float64).copy()

    def run(self):
        self.upload()
        self.solve(download=True)
        torch.cuda.current_stream(self.dev).synchronize()
        return self.results()
