"""Is the per-GEMM fixed cost on the device or on the host? The same GEMM
launched back to back (a) directly and (b) replayed from a CUDA graph (no host
work per launch), plus the host wall time per sfk_gemm call."""
import ctypes as C
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1904_01038_b200 import _lib as L  # noqa: E402


def one(m, n, k, pair, tile=256, iters=40, sk=False, flags=1):
    dt = torch.float16
    a = torch.randn(m * k, device="cuda").to(dt)
    b = torch.randn(n * k, device="cuda").to(dt)
    c = torch.zeros(m * n, device="cuda").to(dt)
    bias = torch.zeros(n, device="cuda").to(dt)
    args = L.GemmArgs(m=m, n=n, k=k, dtype=1, a=a.data_ptr(), lda=k, a_kmajor=1, b=b.data_ptr(), ldb=k, b_kmajor=1,
                      c=c.data_ptr(), ldc=n, flags=flags, bias=bias.data_ptr(), tile_n=tile, pair=pair,
                      stream_k=0 if sk else -1)
    if sk:
        sms = L.sfk_num_sms()
        ws = torch.zeros(sms * 2 * 128 * 256, device="cuda")
        ctr = torch.zeros(2 * sms, dtype=torch.int32, device="cuda")
        args.workspace, args.workspace_floats = ws.data_ptr(), ws.numel()
        args.counters, args.n_counters = ctr.data_ptr(), ctr.numel()
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for _ in range(3):
            L.check(L.sfk_gemm(C.byref(args), C.c_void_p(st.cuda_stream)), True)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(st)
        for _ in range(iters):
            L.sfk_gemm(C.byref(args), C.c_void_p(st.cuda_stream))
        e1.record(st)
        host_us = (time.perf_counter() - t0) / iters * 1e6
        torch.cuda.synchronize()
        direct = e0.elapsed_time(e1) / iters * 1e3
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(iters):
                L.sfk_gemm(C.byref(args), C.c_void_p(st.cuda_stream))
        g.replay()
        torch.cuda.synchronize()
        e0.record(st)
        g.replay()
        e1.record(st)
        torch.cuda.synchronize()
        graph = e0.elapsed_time(e1) / iters * 1e3
    fl = 2.0 * m * n * k
    print(f"M={m} N={n} K={k} pair={pair} sk={int(sk)}: direct {direct:7.2f} us ({fl/direct/1e6:6.1f} TF/s)  graph {graph:7.2f} us "
          f"({fl/graph/1e6:6.1f} TF/s)  host {host_us:6.2f} us/call", flush=True)


for pair, sk in ((1, False), (1, True), (0, False)):
    for n, k in ((1024, 512), (1024, 1024), (1024, 4096), (4096, 1024), (3072, 1024)):
        one(3584, n, k, pair, sk=sk)
