"""Build libspotkm.so with extra nvcc flags into altlib/ for A/B timing
(SPOTKM_LIB=altlib/NAME.so selects it).  usage: python tools/build_variant.py NAME [-DFOO ...]"""
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2311_15566_b200 import build as b  # noqa: E402

out = Path(b.ROOT) / "altlib" / f"{sys.argv[1]}.so"
out.parent.mkdir(exist_ok=True)
cmd = [b.nvcc(), *b.NVCC_FLAGS, *sys.argv[2:], "-o", str(out), *map(str, b.SRC)]
subprocess.run(cmd, check=True)
print(out)
