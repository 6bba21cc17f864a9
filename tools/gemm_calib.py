"""Calibration: cuBLAS (torch.matmul fp16) vs our tcgen05 GEMM on the C4 step shapes
and on 8192^3, back-to-back launches between CUDA events (L2 warm)."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import torch  # noqa: E402
import gemm_bench as G  # noqa: E402


def cublas(m, n, k, ak, bk, iters=20):
    dt = torch.float16
    a = torch.randn(m, k, device="cuda", dtype=dt) if ak else torch.randn(k, m, device="cuda", dtype=dt).t()
    b = torch.randn(n, k, device="cuda", dtype=dt) if bk else torch.randn(k, n, device="cuda", dtype=dt).t()
    c = torch.empty(m, n, device="cuda", dtype=dt)
    for _ in range(3):
        torch.matmul(a, b.t(), out=c)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        torch.matmul(a, b.t(), out=c)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    return 2.0 * m * n * k / (ms * 1e-3) / 1e12, ms


def main():
    os.environ["GB_BACK2BACK"] = "1"
    shapes = list(G.SHAPES) + [("big8k", 8192, 8192, 8192, 1, 1, 0), ("big8k_wg", 8192, 8192, 8192, 0, 0, 0)]
    for sh in shapes:
        name, m, n, k, ak, bk, fl = sh
        cb, cms = cublas(m, n, k, ak, bk)
        ours = {}
        for tn, pr in ((256, -1), (128, -1), (256, 1)):
            tf, ms = G.run(*sh, tile_n=tn, pair=pr)
            ours[f"{'p' if pr > 0 else ''}{tn}"] = round(tf, 1)
        print(f"{name:10s} m={m:5d} n={n:5d} k={k:5d} cublas={cb:7.1f} TF/s ({cms*1e3:7.1f} us) ours={ours}", flush=True)


if __name__ == "__main__":
    main()
