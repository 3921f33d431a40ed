"""NVLink evidence for the executor's data path (one process, two GPUs: run
under `ncu --metrics nvlrx__bytes.sum,nvltx__bytes.sum,gpu__time_duration.sum`).

GPU 0 pulls (or pushes) one GPU's share of a BASELINE reshard -- the chunk
sizes of the real plan's transfers -- from (to) GPU 1 over the peer mapping
with the executor's copy kernel (k_copy, `sk_copy_batched`).  Prints the
event-timed GB/s; ncu's nvlrx/nvltx byte counters on GPU 0 show the bytes
crossing NVLink.

  python tools/nvlink_probe.py [pull|push] [GB]
"""

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2311_15566_b200 import _native as nat  # noqa: E402


def main():
    mode = sys.argv[1] if len(sys.argv) > 1 else "pull"
    gb = float(sys.argv[2]) if len(sys.argv) > 2 else 7.2
    assert torch.cuda.device_count() >= 2, "needs two GPUs in this process"
    lib = nat.load()
    nat.check(lib.sk_enable_peer_access(0, (ctypes_int_array([1])), 1))
    nat.check(lib.sk_enable_peer_access(1, (ctypes_int_array([0])), 1))
    n = int(gb * 1e9) // (1 << 20) * (1 << 20)
    a = torch.empty(n, dtype=torch.uint8, device="cuda:0")
    b = torch.empty(n, dtype=torch.uint8, device="cuda:1")
    b.fill_(7)
    a.fill_(3)
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)
    chunk = 1 << 20
    src, dst = (b, a) if mode == "pull" else (a, b)
    launch_dev = 0
    rows = np.zeros(n // chunk, dtype=nat.COPY)
    rows["src"] = src.data_ptr() + np.arange(n // chunk, dtype=np.uint64) * chunk
    rows["dst"] = dst.data_ptr() + np.arange(n // chunk, dtype=np.uint64) * chunk
    rows["bytes"] = chunk
    with torch.cuda.device(launch_dev):
        d = torch.from_numpy(rows.view(np.uint8)).cuda()
        st = torch.cuda.current_stream()
        times = []
        for it in range(4):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            nat.check(lib.sk_copy_batched(d.data_ptr(), len(rows), 0, st.cuda_stream))
            e1.record()
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
    ok = bool((dst[:: 1 << 24] == (7 if mode == "pull" else 3)).all().item())
    ms = min(times[1:])
    print(f"{mode} {n / 1e9:.2f} GB over NVLink: {ms:.2f} ms, {n / ms / 1e6:.1f} GB/s, bytes ok {ok}")


def ctypes_int_array(vals):
    import ctypes

    return (ctypes.c_int * len(vals))(*vals)


if __name__ == "__main__":
    main()
