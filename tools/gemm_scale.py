"""Per-SM vs chip-wide limits of the tcgen05 GEMM mainloop: one long-k tile per
CTA, varying the number of CTAs (37 / 74 / 148) and the tile kind. Reports
TF/s, TF/s per active SM and the SM clock seen by nvidia-smi right after."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import gemm_bench as G  # noqa: E402

os.environ["GB_BACK2BACK"] = "1"
K = 16384
for name, tn, pair, rows_per_cta, ncta in [
        ("1cta_256", 256, -1, 128, 37), ("1cta_256", 256, -1, 128, 74), ("1cta_256", 256, -1, 128, 148),
        ("1cta_128", 128, -1, 128, 74), ("1cta_128", 128, -1, 128, 148),
        ("2cta_256", 256, 1, 128, 37 * 2), ("2cta_256", 256, 1, 128, 74 * 2)]:
    if pair > 0:
        m, n = 256 * (ncta // 2), 256
    else:
        m, n = rows_per_cta * ncta, tn
    tf, ms = G.run(name, m, n, K, 1, 1, 0, tile_n=tn, pair=pair, iters=10)
    clk = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits"],
                         capture_output=True, text=True).stdout.strip()
    floor = 8192 * float(clk) * 1e6 / 1e12 if clk else 0
    print(f"{name} ctas={ncta:3d} m={m} n={n} k={K}: {tf:7.1f} TF/s  {tf / ncta:6.2f} TF/s/SM "
          f"(floor/SM at {clk} MHz = {floor:.2f})", flush=True)
