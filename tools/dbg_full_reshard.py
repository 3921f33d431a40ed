"""Debug: the plan-ordered executor at growing sizes (one GPU, emulated refs)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import torch
from paper_2311_15566_b200 import reshard

SMALL = ("toy-bf16", 8, 8 * 1024 * 64, 1024)
geom_name, batch, seq = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
geom = {"small": SMALL, "gpt": reshard.GPT20B_BF16}[geom_name]
t = time.time()
plan, layout, need, model, refs = reshard.make_reshard_problem(geom, (1, 4, 2), (1, 2, 4), batch, seq)
owner = {g: 0 for g in set(layout) | set(need)}
ex = reshard.ReshardExecutor(plan, layout, need, model, owner, timeout_s=5)
ch = ex.d_chunks.cpu().numpy().view(reshard.EXEC_CHUNK)
print("chunks", len(ch), "rounds", ex.n_rounds, "waits", int((ch["wait_round"] >= 0).sum()),
      "bad waits", int((ch["wait_round"] >= ch["round"]).sum()),
      "misaligned", int(((ch["src"] | ch["dst"]) % 16 != 0).sum()), "slab GB", ex.slab.nbytes / 1e9, flush=True)
ex.fill_old(); torch.cuda.synchronize()
t = time.time()
ex.run(); torch.cuda.synchronize()
print("run s", time.time() - t, flush=True)
c = ex.control()
print({k: v for k, v in c.items() if k != "stage_ready_ms"}, flush=True)
print("verify", ex.verify(), flush=True)
ex.close()
