"""Per size-class breakdown of one sweep batch: plans, n range, Dijkstra
steps, serialised k_fuse / k_outer ms.  usage: python tools/sweep_classes.py N SETS"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2311_15566_b200 import sweep  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
S = int(sys.argv[2]) if len(sys.argv) > 2 else 32
b = sweep.make_sweep(N, S, seed=5)
r = sweep.SweepRunner(b)
r.run()
steps = torch.zeros(2 * b.n_plans, dtype=torch.int64, device="cuda")
prof = {}
r.upload()
r.solve(steps=steps, profile=prof)
torch.cuda.synchronize()
ms = r.kernel_ms(prof, per_class=True)
st = steps.cpu().numpy().reshape(-1, 2)
n = b.stats()["n"]
out = []
for c, (a, e, mn) in enumerate(r.classes):
    out.append({"class": c, "plans": e - a, "n": [int(n[a:e].min()), int(n[a:e].max())],
                "bucket": sweep.cpl_bucket(mn), "steps_mean": float(st[a:e, 0].mean()),
                "steps_max": int(st[a:e, 0].max()), "k_fuse_ms": ms.get(f"k_fuse[{c}]"),
                "k_outer_ms": ms.get(f"k_outer[{c}]")})
print(json.dumps(out, indent=1))
