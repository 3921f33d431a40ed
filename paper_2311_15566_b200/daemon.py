"""Context daemon: a per-GPU process that owns the context
slabs, receives migration plans on the wire and executes them, and a client
for the serving process that consumes the migrated context.

SpotServe runs its inference engine and a context daemon as separate
processes that share context pointers through CUDA IPC and block inference
per tensor until its context has arrived; plans travel as
JSON (`plan_to_dict`, migration.py:407-431).  Here:

* `ContextDaemon` listens on a Unix socket.  A `migrate` request carries the
  plan's wire form plus the old layout, the required new layout and the
  mapping (stage of every GPU).  The daemon builds the executor
  (reshard.ReshardExecutor: arena layout + one persistent k_exec launch),
  fills the old contexts, and answers `ready` with its slab's CUDA IPC handle,
  the byte offsets of the per-stage ready flags in its control block and,
  per stage, the byte regions of the new context.  On `go` it runs the
  migration and answers `done` with the control block (error, rounds,
  stage-ready times) and its own byte check.
* The stage flags are mirrored by the daemon's kernel into a POSIX
  shared-memory segment registered as mapped host memory (`sk_host_register`,
  written with system-scope stores), because the two processes' contexts
  time-slice on one GPU: a consumer that waits ON THE GPU (a spinning kernel,
  or a stream semaphore wait) can hold the GPU away from the producer.
* `DaemonClient` (the serving side) maps the slab with CUDA IPC, polls the
  shared flags from its host thread, and launches each stage's work the moment
  that stage's flag is up -- here a byte check of the stage's context, standing
  in for the first decode step -- while later rounds are still moving.

Messages are JSON lines.  Intervals travel as [num, den].
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import socket
import sys
from fractions import Fraction

import numpy as np
import torch

from . import _native as nat
from . import domain as dm
from . import reshard
from .planner import plan_from_dict, plan_to_dict


def enc_inv(inv):
    return {"m": [[l, lo.numerator, lo.denominator, hi.numerator, hi.denominator] for l, lo, hi in inv.model_shards],
            "c": [[r, l, lo.numerator, lo.denominator, hi.numerator, hi.denominator, t]
                  for r, l, lo, hi, t in inv.cache_shards]}


def dec_inv(doc):
    return dm.ContextInventory(
        tuple((l, Fraction(a, b), Fraction(c, d)) for l, a, b, c, d in doc["m"]),
        tuple((r, l, Fraction(a, b), Fraction(c, d), t) for r, l, a, b, c, d, t in doc["c"]))


def migrate_request(plan, old_layout, new_required, model, assignment) -> dict:
    """The wire form of one migration (plan_to_dict + layouts + mapping)."""
    return {"op": "migrate", "plan": plan_to_dict(plan),
            "model": [model.num_layers, model.bytes_per_layer, model.kv_bytes_per_token_per_layer],
            "old": [[g[0], g[1], enc_inv(inv)] for g, inv in old_layout.items()],
            "new": [[g[0], g[1], enc_inv(inv)] for g, inv in new_required.items()],
            "assignment": [[g[0], g[1], p.pipeline, p.stage, p.shard] for g, p in assignment.items()]}


def _send(f, doc):
    f.write((json.dumps(doc) + "\n").encode())
    f.flush()


def _recv(f):
    line = f.readline()
    if not line:
        raise ConnectionError("peer closed the connection")
    return json.loads(line)


class ContextDaemon:
    """Owns this GPU's context slabs and executes migration plans."""

    def __init__(self, path: str, device: int = 0):
        self.path = path
        self.device = device
        torch.cuda.set_device(device)
        nat.load()

    def serve(self, max_requests: int | None = None):
        if os.path.exists(self.path):
            os.unlink(self.path)
        srv = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
        srv.bind(self.path)
        srv.listen(1)
        served = 0
        try:
            while max_requests is None or served < max_requests:
                conn, _ = srv.accept()
                with conn, conn.makefile("rwb") as f:
                    if not self._session(f):
                        return
                served += 1
        finally:
            srv.close()
            if os.path.exists(self.path):
                os.unlink(self.path)

    def _session(self, f) -> bool:
        ex = None
        self.shm = None
        try:
            while True:
                msg = _recv(f)
                op = msg["op"]
                if op == "shutdown":
                    _send(f, {"op": "bye"})
                    return False
                if op == "migrate":
                    if ex is not None:
                        ex.close()
                    ex, reply = self._prepare(msg)
                    _send(f, reply)
                elif op == "go":
                    if ex is None:
                        _send(f, {"op": "error", "message": "go before migrate"})
                        continue
                    ex.run(flag_mirror=self.mirror_dev)
                    torch.cuda.synchronize()
                    ctl = ex.control()
                    _send(f, {"op": "done", "error": ctl["error"], "progress": ctl["progress"],
                              "rounds": ctl["rounds"],
                              "stage_ready_ms": {str(k): v for k, v in ctl["stage_ready_ms"].items()},
                              "mismatched_words": ex.verify()})
                elif op == "release":
                    # the slab goes; the session stays open for the next plan
                    if ex is not None:
                        ex.close()
                        ex = None
                    self._drop_shm()
                    _send(f, {"op": "released"})
                else:
                    _send(f, {"op": "error", "message": f"unknown op {op!r}"})
        except ConnectionError:
            return True
        finally:
            if ex is not None:
                ex.close()
            self._drop_shm()

    def _drop_shm(self):
        if self.shm is not None:
            torch.cuda.synchronize()
            ex_lib = nat.load()
            ex_lib.sk_host_unregister(ctypes.c_void_p(self.shm_addr))
            self.shm.close()
            self.shm.unlink()
            self.shm = None

    def _prepare(self, msg):
        model = dm.ModelSpec("wire", *msg["model"])
        plan = plan_from_dict(msg["plan"])
        old = {(i, g): dec_inv(v) for i, g, v in msg["old"]}
        new = {(i, g): dec_inv(v) for i, g, v in msg["new"]}
        stage_of = {(i, g): p for i, g, d, p, m in msg["assignment"]}
        owner = {g: 0 for g in set(old) | set(new)}
        ex = reshard.ReshardExecutor(plan, old, new, model, owner)
        ex.fill_old()
        ex.reset_control()   # flags down before the consumer can see the handle
        torch.cuda.synchronize()
        # host-mapped mirror of the stage flags, shared with the consumer process
        from multiprocessing import shared_memory

        self._drop_shm()
        self.shm = shared_memory.SharedMemory(create=True, size=max(4096, 4 * len(ex.stages)))
        self.shm.buf[:] = bytes(len(self.shm.buf))
        self.shm_addr = ctypes.addressof(ctypes.c_char.from_buffer(self.shm.buf))
        d = ctypes.c_void_p()
        nat.check(ex.lib.sk_host_register(ctypes.c_void_p(self.shm_addr), len(self.shm.buf), ctypes.byref(d)))
        self.mirror_dev = d.value
        handle = ctypes.create_string_buffer(64)
        nat.check(ex.lib.sk_ipc_get_handle(ex.slab.ptr, handle))
        R = ex.n_rounds
        flag_off = {str(s): 4 * (4 + R + i) for i, s in enumerate(ex.stages)}
        regions = {}   # stage -> [[slab offset, bytes, key, object base]]
        rows = ex.region_rows(new=True)
        for g, row in rows:
            st = stage_of.get(g)
            if st is None:
                continue
            ptr, n, key, base = row
            regions.setdefault(str(st), []).append([ptr - ex.slab.ptr, n, str(key), base])
        return ex, {"op": "ready", "handle": handle.raw.hex(), "slab_bytes": ex.slab.nbytes,
                    "flag_shm": self.shm.name,
                    "flag_offset": flag_off, "regions": regions, "rounds": R,
                    "stages": [int(s) for s in ex.stages]}


class DaemonClient:
    """The serving side: submits a migration, maps the daemon's slab, and
    starts each stage's work on the device as soon as its flag is raised."""

    def __init__(self, path: str):
        self.sock = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
        self.sock.connect(path)
        self.f = self.sock.makefile("rwb")
        self.lib = nat.load()
        self.lib.sk_wait_flag.argtypes = [ctypes.c_void_p, ctypes.c_uint32, ctypes.c_double, ctypes.c_void_p,
                                          ctypes.c_void_p]
        self.lib.sk_wait_flag.restype = ctypes.c_int32
        self.lib.sk_stream_wait_flag.argtypes = [ctypes.c_void_p, ctypes.c_uint32, ctypes.c_void_p]
        self.lib.sk_stream_wait_flag.restype = ctypes.c_int32
        self.mapped = None

    def migrate(self, request: dict, timeout_s: float = 30.0) -> dict:
        """Submit, map, run; launch each stage's work (a byte check of its new
        context) as soon as its flag appears in the shared mirror.  Returns the
        daemon's `done` report plus, per stage, the mismatching words this
        process saw in that stage's context, and the order stages started in."""
        import time
        from multiprocessing import shared_memory

        _send(self.f, request)
        ready = _recv(self.f)
        if ready["op"] != "ready":
            raise RuntimeError(ready)
        p = ctypes.c_void_p()
        nat.check(self.lib.sk_ipc_open_handle(bytes.fromhex(ready["handle"]), ctypes.byref(p)))
        self.mapped = p.value
        shm = shared_memory.SharedMemory(name=ready["flag_shm"])
        try:
            flags = np.ndarray((len(ready["stages"]),), dtype=np.uint32, buffer=shm.buf)
            st = torch.cuda.current_stream()
            stages = ready["stages"]
            bad = torch.zeros(max(len(stages), 1), dtype=torch.int64, device="cuda")
            keep, started = [], []
            _send(self.f, {"op": "go"})
            t0 = time.perf_counter()
            pending = set(range(len(stages)))
            while pending and time.perf_counter() - t0 < timeout_s:
                for i in sorted(pending):
                    if flags[i] == 0:
                        continue
                    pending.discard(i)
                    started.append(stages[i])
                    rows = ready["regions"].get(str(stages[i]), [])
                    if rows:
                        reg = np.zeros(len(rows), dtype=nat.REGION)
                        for k, (off, n, key, base) in enumerate(rows):
                            reg[k] = (self.mapped + off, n, int(key), base)
                        d = torch.from_numpy(reg.view(np.uint8)).cuda()
                        keep.append(d)
                        nat.check(self.lib.sk_verify_regions(d.data_ptr(), len(rows), bad.data_ptr() + 8 * i,
                                                             st.cuda_stream))
            done = _recv(self.f)
            torch.cuda.synchronize()
            done["client_stage_mismatched_words"] = {str(s): int(b) for s, b in zip(stages, bad.tolist())}
            done["client_wait_timeouts"] = len(pending)
            done["client_stage_order"] = started
            del keep, flags
        finally:
            shm.close()
        return done

    def release(self):
        if self.mapped:
            torch.cuda.synchronize()
            self.lib.sk_ipc_close_handle(self.mapped)
            self.mapped = None
        _send(self.f, {"op": "release"})
        _recv(self.f)

    def shutdown(self):
        try:
            _send(self.f, {"op": "shutdown"})
            _recv(self.f)
        except (ConnectionError, OSError):
            pass  # the daemon already closed the session
        self.f.close()
        self.sock.close()


def main(argv=None):
    ap = argparse.ArgumentParser(description="SpotServe context daemon (one per GPU)")
    ap.add_argument("--socket", required=True)
    ap.add_argument("--device", type=int, default=0)
    args = ap.parse_args(argv)
    ContextDaemon(args.socket, args.device).serve()
    return 0


if __name__ == "__main__":
    sys.exit(main())
