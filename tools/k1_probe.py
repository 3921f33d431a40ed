"""K1 (build_graph's dense W) alone, for ncu: bench.k1_leg at 256 and 1,024
positions.  python tools/k1_probe.py"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2311_15566_b200 import sweep  # noqa: E402

geom, shapes = sweep.MODELS["gpt-20b"]
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
pk, _ = bench.peaks()
print(json.dumps(bench.k1_leg(geom, shapes, flush, float(pk.get("hbm_gbs", 6650.0)), reps=2)))
