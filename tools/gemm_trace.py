"""Device timeline of single pair-GEMM launches (trace build: SQF_LIB=.../trace/libsqf_b200.so):
%globaltimer stamps of CTA 0 and the last CTA relative to CTA 0's entry."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1904_01038_b200 import _lib as L  # noqa: E402

NAMES = ["entry", "prologue", "pdl_wait", "tma0", "stage0", "mma_end", "acc_ready", "epi_done", "all_done", "tmem_free"]


def trace(m, n, k, prev=None, sk=False):
    dt = torch.float16
    a = torch.randn(m * k, device="cuda").to(dt)
    b = torch.randn(n * k, device="cuda").to(dt)
    c = torch.zeros(m * n, device="cuda").to(dt)
    args = L.GemmArgs(m=m, n=n, k=k, dtype=1, a=a.data_ptr(), lda=k, a_kmajor=1, b=b.data_ptr(), ldb=k, b_kmajor=1,
                      c=c.data_ptr(), ldc=n, flags=int(os.environ.get('GT_FLAGS', '1')), tile_n=256, pair=1,
                      stream_k=0 if sk else -1)
    if sk:
        sms = L.sfk_num_sms()
        ws = torch.zeros(sms * 2 * 128 * 256, device="cuda")
        ctr = torch.zeros(2 * sms, dtype=torch.int32, device="cuda")
        args.workspace, args.workspace_floats = ws.data_ptr(), ws.numel()
        args.counters, args.n_counters = ctr.data_ptr(), ctr.numel()
    st = torch.cuda.current_stream()
    for rep in range(3):
        L.check(L.sfk_gemm(C.byref(args), C.c_void_p(st.cuda_stream)), True)
        L.check(L.sfk_gemm(C.byref(args), C.c_void_p(st.cuda_stream)), True)  # back to back: the second is traced
        torch.cuda.synchronize()
    out = np.zeros(48, np.uint64)
    L.check(L.sfk_debug_gemm_trace(out.ctypes.data), True)
    t = out.reshape(2, 24).astype(np.int64)
    base = t[0, 0]
    print(f"M={m} N={n} K={k} sk={int(sk)}")
    for r, who in enumerate(("cta0", "last")):
        print("  " + who + ": " + " ".join(f"{NAMES[i]}={(t[r, i] - base) / 1e3:.2f}" for i in range(10)))
        if r == 0:
            print("    sk: partial_stored/fixup_start/fixup_done: " + " ".join(
                f"{(t[0, i] - base) / 1e3:.2f}" for i in (11, 22, 23)))
            print("    warp2 chunk ld done: " + " ".join(f"c{i}={(t[0, 10 + i] - base) / 1e3:.2f}" for i in range(8))
                  + "  block stores: " + " ".join(f"b{i}={(t[0, 18 + i] - base) / 1e3:.2f}" for i in range(4)))


for n, k in ((1024, 4096), (4096, 1024)):
    trace(3584, n, k)
    trace(3584, n, k, sk=True)
