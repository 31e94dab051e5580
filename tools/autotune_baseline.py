"""Run smmc_autotune_f32 on the small BASELINE layers (table plans vs tuner candidates)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2411_15659_b200 import _native  # noqa: E402
from paper_2411_15659_b200.workloads import CONFIGS  # noqa: E402
for c in (2, 3, 5):
    for name, n, g in CONFIGS[c]["layers"]:
        if n > 8 and c != 3:
            continue
        for rep in range(2):
            _native.autotune_clear()
            print(c, name, _native.autotune(g, n, iters=20), flush=True)
