"""Run one GEMM configuration a few times (for ncu captures)."""
import sys
import os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import gemm_bench as G  # noqa: E402

name = sys.argv[1]
tile = int(sys.argv[2]) if len(sys.argv) > 2 else 0
pair = int(sys.argv[3]) if len(sys.argv) > 3 else 0
shapes = list(G.SHAPES) + [("big8k", 8192, 8192, 8192, 1, 1, 0), ("big8k_wg", 8192, 8192, 8192, 0, 0, 0)]
sh = [s for s in shapes if s[0] == name][0]
tf, ms = G.run(*sh, tile_n=tile, iters=5, pair=pair)
print(name, tile, round(tf, 1), "TFLOP/s", round(ms * 1e3, 1), "us")
