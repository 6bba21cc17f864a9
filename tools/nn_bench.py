"""Back-to-back GPU timing of the memory-bound kernels at C4 step shapes."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1904_01038_b200 import _lib as L  # noqa: E402


def timeit(fn, iters=50):
    st = torch.cuda.current_stream()
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(iters):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters * 1e3


def main():
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    R, d = 3584, 1024
    x = torch.randn(R, d, device="cuda").half()
    dy = torch.randn(R, d, device="cuda").half()
    g = torch.ones(d, device="cuda").half()
    b = torch.zeros(d, device="cuda").half()
    y = torch.empty_like(x)
    dx = torch.empty_like(x)
    st = torch.zeros(R, 2, device="cuda")
    part = torch.zeros(2 * 592 * 4096, device="cuda")
    dg, db = torch.zeros(d, device="cuda").half(), torch.zeros(d, device="cuda").half()
    p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    mb = R * d * 2 / 1e6
    t = timeit(lambda: L.sfk_layernorm_fwd(1, p(x), R, d, p(g), p(b), p(y), p(st), s))
    print(f"ln_fwd      {t:7.1f} us  {2 * mb / t:6.2f} TB/s")
    t = timeit(lambda: L.sfk_layernorm_bwd_fused(1, p(x), p(dy), R, d, p(g), p(st), p(dx), 1, p(part), None, p(dg),
                                                 p(db), s))
    print(f"ln_bwd      {t:7.1f} us  {4 * mb / t:6.2f} TB/s")
    t = timeit(lambda: L.sfk_layernorm_bwd_dx_acc(1, p(x), p(dy), R, d, p(g), p(st), p(dx), p(dx), s))
    print(f"ln_dx(acc)  {t:7.1f} us  {4 * mb / t:6.2f} TB/s  (reads x, dy, acc; writes dx)")
    npart = C.c_int()
    t = timeit(lambda: L.sfk_layernorm_bwd_params_partial(1, p(x), p(dy), R, d, p(st), p(part), C.byref(npart), s))
    print(f"ln_gb_part  {t:7.1f} us  {2 * mb / t:6.2f} TB/s  ({npart.value} partials)")
    for n in (1024, 3072, 4096, 32768):
        a = torch.randn(R, n, device="cuda").half()
        o = torch.zeros(n, device="cuda").half()
        t = timeit(lambda: L.sfk_colsum(1, p(a), R, n, n, p(part), None, p(o), s))
        print(f"colsum n={n:6d} {t:7.1f} us  {R * n * 2 / t * 1e-6:6.2f} TB/s")
    lg = torch.randn(R, 32768, device="cuda").half()
    gold = torch.randint(4, 32768, (R,), device="cuda", dtype=torch.int32)
    ro = torch.zeros(R, 4, device="cuda")
    t = timeit(lambda: L.sfk_xent_fwd_bwd(1, p(lg), R, 32768, 32768, p(gold), 1, 0.1, 1.0, p(lg), p(ro), s), 10)
    print(f"xent        {t:7.1f} us  {2 * R * 32768 * 2 / t * 1e-6:6.2f} TB/s")
    n = 277_000_000
    g16 = torch.zeros(n, device="cuda").half()
    flag = torch.zeros(4, dtype=torch.int32, device="cuda")
    t = timeit(lambda: L.sfk_nonfinite(1, p(g16), n, p(flag), s), 5)
    print(f"nonfinite   {t:7.1f} us  {n * 2 / t * 1e-6:6.2f} TB/s")


def attention():
    """Attention fwd / bwd at C4 shapes: self-attention on fused QKV rows
    (ld 3d), 16 heads of 64; batches of 3584 tokens at widths 16..200."""
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    H, dh = 16, 64
    d = H * dh
    shapes = [(3584 // w, w, c) for w in (16, 30, 48, 64, 96, 120, 200) for c in (False, True)]
    for batch, w, causal in shapes:
        rows = batch * w
        qkv = (torch.randn(rows, 3 * d, device="cuda") * 0.5).half()
        o = torch.zeros(rows, d, device="cuda").half()
        do = torch.randn(rows, d, device="cuda").half()
        dq, dk, dv = (torch.zeros(rows, d, device="cuda").half() for _ in range(3))
        st = torch.zeros(rows * H, 2, device="cuda")
        sc = torch.zeros(rows * H, device="cuda")
        lens = torch.randint(w // 2, w + 1, (batch,), device="cuda", dtype=torch.int32)
        base = qkv.data_ptr()
        a = L.AttnArgs(dtype=1, batch=batch, q_width=w, k_width=w, heads=H, dh=dh, causal=int(causal),
                       k_len=p(lens), q=base, ldq=3 * d, k=base + 2 * d, ldk=3 * d, v=base + 4 * d, ldv=3 * d,
                       o=p(o), ldo=d, stats=p(st), dout=p(do), lddo=d, dq=p(dq), lddq=d, dk=p(dk), lddk=d,
                       dv=p(dv), lddv=d, scratch=p(sc))
        tf = timeit(lambda: L.sfk_attention_fwd(C.byref(a), s))
        tb = timeit(lambda: L.sfk_attention_bwd(C.byref(a), s))
        mb = rows * d * 2 / 1e6
        print(f"attention batch={batch} width={w} causal={int(causal)}: fwd {tf:6.1f} us ({4 * mb / tf:.2f} TB/s) "
              f"bwd {tb:6.1f} us ({8 * mb / tb:.2f} TB/s)")


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "attention":
        attention()
        sys.exit(0)
    main()
