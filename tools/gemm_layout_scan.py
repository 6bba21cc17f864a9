"""Mainloop cost per k-block by operand layout (back-to-back launches, warm
L2): K-major x K-major (forward), K-major x MN-major (activation gradient),
MN-major x MN-major (weight gradient), CTA-pair 256 x 256 tiles. The slope of
time vs K over one wave of tiles is the per-k-block mainloop time."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
os.environ["GB_BACK2BACK"] = "1"
import gemm_bench as G  # noqa: E402

for name, ak, bk in (("fwd  K x K  ", 1, 1), ("dgrad K x MN", 1, 0), ("wgrad MN x MN", 0, 0)):
    prev = None
    for k in (1024, 2048, 4096, 8192):
        tf, ms = G.run("scan", 3584, 1024, k, ak, bk, 0, tile_n=256, iters=30, pair=1)
        us = ms * 1e3
        slope = "" if prev is None else f"  slope {(us - prev[1]) / ((k - prev[0]) / 64):.3f} us/k-block"
        print(f"{name} M=3584 N=1024 K={k:5d} (56 pair tiles) {us:8.2f} us {tf:7.1f} TF/s{slope}", flush=True)
        prev = (k, us)
