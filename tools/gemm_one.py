"""Run one GEMM configuration a few times (for ncu captures)."""
import sys
import os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import gemm_bench as G  # noqa: E402

name = sys.argv[1]
tile = int(sys.argv[2]) if len(sys.argv) > 2 else 0
sh = [s for s in G.SHAPES if s[0] == name][0]
tf, ms = G.run(*sh, tile_n=tile, iters=5)
print(name, tile, round(tf, 1), "TFLOP/s", round(ms * 1e3, 1), "us")
