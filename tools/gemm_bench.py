"""Microbenchmark of the tcgen05 GEMM on the C4 (Transformer-big) step shapes:
TFLOP/s per (shape, layout, tile width), CUDA events on the launch stream,
L2 flushed between launches (inputs > L2 for the big shapes anyway)."""
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1904_01038_b200 import _lib as L  # noqa: E402

M = 3584
SHAPES = [  # (name, m, n, k, a_kmajor, b_kmajor, flags)
    ("fwd_qkv", M, 3072, 1024, 1, 1, 3), ("fwd_out", M, 1024, 1024, 1, 1, 19), ("fwd_ffn1", M, 4096, 1024, 1, 1, 7),
    ("fwd_ffn2", M, 1024, 4096, 1, 1, 19), ("fwd_ckv", M, 2048, 1024, 1, 1, 3), ("fwd_vocab", M, 32768, 1024, 1, 1, 1),
    ("dg_qkv", M, 1024, 3072, 1, 0, 32), ("dg_out", M, 1024, 1024, 1, 0, 0), ("dg_ffn1", M, 1024, 4096, 1, 0, 32),
    ("dg_ffn2", M, 4096, 1024, 1, 0, 8), ("dg_vocab", M, 1024, 32768, 1, 0, 0),
    ("wg_qkv", 3072, 1024, M, 0, 0, 32), ("wg_out", 1024, 1024, M, 0, 0, 32), ("wg_ffn1", 4096, 1024, M, 0, 0, 32),
    ("wg_ffn2", 1024, 4096, M, 0, 0, 32), ("wg_vocab", 32768, 1024, M, 0, 0, 32),
]


def run(name, m, n, k, ak, bk, flags, tile_n, iters=20, pair=0):
    dt = torch.float16
    a = torch.randn(m * k, device="cuda").to(dt)
    b = torch.randn(n * k, device="cuda").to(dt)
    c = torch.randn(m * n, device="cuda").to(dt)
    bias = torch.randn(n, device="cuda").to(dt)
    res = torch.randn(m * n, device="cuda").to(dt)
    args = L.GemmArgs(m=m, n=n, k=k, dtype=1, a=a.data_ptr(), lda=k if ak else m, a_kmajor=ak, b=b.data_ptr(),
                      ldb=k if bk else n, b_kmajor=bk, c=c.data_ptr(), ldc=n, bias=bias.data_ptr(),
                      res=res.data_ptr(), ldr=n, mask=res.data_ptr(), ldm=n, flags=flags, tile_n=tile_n, pair=pair)
    st = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        L.check(L.sfk_gemm(C.byref(args), C.c_void_p(st.cuda_stream)), True)
    if os.environ.get("GB_BACK2BACK"):
        # back-to-back launches between two events: GPU time per GEMM with the
        # host ahead of the device (L2 warm: steady-state in-step conditions)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(iters):
            L.sfk_gemm(C.byref(args), C.c_void_p(st.cuda_stream))
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / iters
        return 2.0 * m * n * k / (ms * 1e-3) / 1e12, ms
    ts = []
    for _ in range(iters):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        L.sfk_gemm(C.byref(args), C.c_void_p(st.cuda_stream))
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    ms = ts[len(ts) // 2]
    return 2.0 * m * n * k / (ms * 1e-3) / 1e12, ms


def main():
    out = {}
    # GB_VARIANTS="p256,256": subset of {0,128,256,p128,p256} (default all)
    variants = os.environ.get("GB_VARIANTS", "0,128,256,p128,p256").split(",")
    for sh in SHAPES:
        row = {}
        for v in variants:
            pair = 1 if v.startswith("p") else 0
            tf, ms = run(*sh, tile_n=int(v.lstrip("p")), pair=pair)
            row[v] = (round(tf, 1), round(ms * 1e3, 1))
        out[sh[0]] = row
        print(sh[0], json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
