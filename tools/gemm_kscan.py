"""GEMM time vs K and vs tile count (back-to-back launches, warm L2): the slope
in K is the mainloop cost per k-block, the intercept the fixed per-launch /
per-tile cost (prologue, pipeline fill, epilogue, wave tail)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
os.environ["GB_BACK2BACK"] = "1"
import gemm_bench as G  # noqa: E402

for pair, tile in ((1, 256), (0, 256)):
    for n in (1024, 4096):
        for k in (512, 1024, 2048, 4096, 8192):
            tf, ms = G.run("scan", 3584, n, k, 1, 1, 0, tile_n=tile, iters=30, pair=pair)
            tiles = (3584 // (256 if pair else 128)) * (n // tile)
            print(f"pair={pair} tile={tile} M=3584 N={n:5d} K={k:5d} tiles={tiles:4d} {ms*1e3:8.2f} us {tf:7.1f} TF/s",
                  flush=True)
