"""GPU parity of each sm_100a kernel through the C ABI (include/sqf_kernels.h)
against the reference oracle (the seqforge tape ops, oracle/_ref) or, for the
GEMM, an fp64 product of the same (rounded) operands. Tolerances are stated
per test; integer/index outputs are compared exactly."""
import ctypes as C

import numpy as np
import pytest

from oracle import ref

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def L():
    from paper_1904_01038_b200 import _lib
    return _lib


def stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


TDT = {0: torch.float32, 1: torch.float16, 2: torch.bfloat16}


def run_gemm(m, n, k, dtype, a_kmajor, b_kmajor, flags=0, seed=0, force_simt=False, with_c=None, pair=0, tile_n=0,
             stream_k=-1, ws=None):
    lib = L()
    g = torch.Generator(device="cuda").manual_seed(seed)
    td = TDT[dtype]
    A = (torch.randn(m, k, device="cuda", generator=g) * 0.5).to(td)  # logical A(i,k)
    B = (torch.randn(n, k, device="cuda", generator=g) * 0.5).to(td)  # logical B(j,k)
    a_store = A.contiguous() if a_kmajor else A.t().contiguous()
    b_store = B.contiguous() if b_kmajor else B.t().contiguous()
    bias = (torch.randn(n, device="cuda", generator=g)).to(td)
    res = (torch.randn(m, n, device="cuda", generator=g)).to(td)
    mask = (torch.randn(m, n, device="cuda", generator=g)).to(td)
    c = with_c.clone() if with_c is not None else torch.randn(m, n, device="cuda", generator=g).to(td)
    c0 = c.clone()
    args = lib.GemmArgs(m=m, n=n, k=k, dtype=dtype, a=ptr(a_store), lda=a_store.shape[1], a_kmajor=int(a_kmajor),
                        b=ptr(b_store), ldb=b_store.shape[1], b_kmajor=int(b_kmajor), c=ptr(c), ldc=n,
                        bias=ptr(bias), res=ptr(res), ldr=n, mask=ptr(mask), ldm=n, flags=flags,
                        force_simt=int(force_simt), pair=pair, tile_n=tile_n, stream_k=stream_k)
    if ws is not None:
        args.workspace, args.workspace_floats = ptr(ws[0]), ws[0].numel()
        args.counters, args.n_counters = ptr(ws[1]), ws[1].numel()
    lib.check(lib.sfk_gemm(C.byref(args), stream()), kernel=True)
    torch.cuda.synchronize()
    acc = (A.double() @ B.double().t()).float()
    q = (lambda x: x.to(td).float()) if dtype != 0 else (lambda x: x)
    v = acc
    if flags & lib.EPI_ACCUM:
        v = q(c0.float() + acc)
    else:
        if flags & lib.EPI_PREROUND:
            v = q(v)
        if flags & lib.EPI_BIAS:
            v = q(v + bias.float())
        if flags & lib.EPI_RELU:
            v = torch.clamp_min(v, 0)
        if flags & lib.EPI_MASK:
            v = torch.where(mask.float() > 0, q(v), torch.zeros_like(v))
        if flags & lib.EPI_RESIDUAL:
            v = q(res.float() + v)
    return c.float(), q(v)


@pytest.mark.parametrize("dtype", [1, 2])
@pytest.mark.parametrize("layout", [(True, True), (True, False), (False, False), (False, True)])
@pytest.mark.parametrize("shape", [(128, 256, 64), (200, 320, 96), (1000, 72, 520), (4096, 3072, 1024),
                                   (3584, 1024, 4096), (17, 24, 16)])
def test_gemm_tc_layouts(dtype, layout, shape):
    m, n, k = shape
    lda = k if layout[0] else m
    ldb = k if layout[1] else n
    if lda % 8 or ldb % 8:
        # TMA needs 16-byte row pitches: the library must refuse, not compute garbage
        with pytest.raises(Exception, match="16-byte"):
            run_gemm(m, n, k, dtype, *layout)
        return
    got, want = run_gemm(m, n, k, dtype, *layout)
    tol = 4e-3 if dtype == 1 else 2e-2
    torch.testing.assert_close(got, want, rtol=tol, atol=tol * max(1.0, k ** 0.5 * 0.25))


@pytest.mark.parametrize("tile_n", [128, 256])
@pytest.mark.parametrize("layout", [(True, True), (True, False), (False, False), (False, True)])
@pytest.mark.parametrize("shape", [(256, 256, 64), (300, 200, 96), (1000, 136, 520), (3584, 1024, 1024),
                                   (4096, 3072, 1024), (64, 40, 32)])
def test_gemm_tc_cta_pair(tile_n, layout, shape):
    # cta_group::2 tiles (256 x tile_n per CTA pair), fp16 and a fused epilogue
    m, n, k = shape
    lda = k if layout[0] else m
    ldb = k if layout[1] else n
    if lda % 8 or ldb % 8:
        pytest.skip("TMA pitch")
    flags = (1 | 2 | 16) if layout == (True, True) else (32 if layout == (False, False) else 0)
    got, want = run_gemm(m, n, k, 1, *layout, flags=flags, pair=1, tile_n=tile_n)
    torch.testing.assert_close(got, want, rtol=4e-3, atol=4e-3 * max(1.0, k ** 0.5 * 0.25))


@pytest.mark.parametrize("flags", [1 | 2, 1 | 2 | 4, 1 | 2 | 16, 8, 32, 1 | 2 | 4 | 16])
def test_gemm_tc_epilogues(flags):
    got, want = run_gemm(300, 200, 128, 1, True, flags != 32, flags)
    torch.testing.assert_close(got, want, rtol=4e-3, atol=8e-3)


@pytest.mark.parametrize("layout", [(True, True), (True, False), (False, False)])
def test_gemm_simt_fp32(layout):
    got, want = run_gemm(133, 70, 95, 0, *layout, flags=1 | 2 | 16)
    torch.testing.assert_close(got, want, rtol=1e-5, atol=1e-5)


def test_gemm_rejects_misaligned_tc_operands():
    lib = L()
    a = torch.zeros(64, 30, dtype=torch.float16, device="cuda")
    c = torch.zeros(64, 64, dtype=torch.float16, device="cuda")
    args = lib.GemmArgs(m=64, n=64, k=30, dtype=1, a=ptr(a), lda=30, a_kmajor=1, b=ptr(a), ldb=30, b_kmajor=1,
                        c=ptr(c), ldc=64)
    assert lib.sfk_gemm(C.byref(args), stream()) == -1


@pytest.mark.parametrize("fp16", [False, True])
@pytest.mark.parametrize("rows,vocab,eps", [(7, 11, 0.1), (64, 1000, 0.1), (33, 32768, 0.1), (20, 10000, 0.0)])
def test_xent_matches_reference(fp16, rows, vocab, eps):
    lib = L()
    rng = np.random.default_rng(rows)
    lg = (rng.standard_normal((rows, vocab)) * 3).astype(np.float32)
    if fp16:
        lg = ref.quantize_array(lg)
    gold = rng.integers(0, vocab, rows).astype(np.int32)
    gold[::5] = 1  # pad rows
    seed = 256.0 if fp16 else 1.0
    loss, nll, corr, dl = ref.xent(lg, gold, eps, fp16, seed)
    dt = 1 if fp16 else 0
    t = torch.tensor(lg, device="cuda").to(TDT[dt])
    g = torch.tensor(gold, device="cuda")
    rows_out = torch.zeros(rows, 4, device="cuda")
    acc = torch.zeros(4, dtype=torch.float64, device="cuda")
    lib.check(lib.sfk_xent_fwd_bwd(dt, ptr(t), rows, vocab, vocab, ptr(g), 1, eps, seed, ptr(t), ptr(rows_out),
                                   stream()), kernel=True)
    lib.check(lib.sfk_xent_reduce(ptr(rows_out), rows, ptr(acc), stream()), kernel=True)
    torch.cuda.synchronize()
    ro = rows_out.cpu().numpy()
    active = gold != 1
    np.testing.assert_array_equal(ro[:, 3], active.astype(np.float32))
    np.testing.assert_array_equal(ro[:, 2], corr.astype(np.float32))  # argmax (first max) exact
    np.testing.assert_allclose(ro[:, 1], nll, rtol=2e-6, atol=2e-5)
    np.testing.assert_allclose(ro[:, 0], loss, rtol=1e-3 if fp16 else 2e-6, atol=2e-5)
    # fp32: the reference folds sum-exp sequentially over V terms, the kernel
    # uses a tree; lse differs by O(1e-6) relative, p by O(1e-5) (tolerance 1e-4)
    np.testing.assert_allclose(t.float().cpu().numpy(), dl, rtol=1e-3 if fp16 else 1e-4, atol=1e-6 * seed)
    a = acc.cpu().numpy()
    assert a[2] == active.sum() and a[3] == corr.sum()
    np.testing.assert_allclose(a[0], float(loss.astype(np.float64).sum()), rtol=1e-3 if fp16 else 1e-5)


@pytest.mark.parametrize("fp16", [False, True])
@pytest.mark.parametrize("rows,d", [(5, 16), (300, 512), (129, 1024), (64, 64)])
def test_layernorm_matches_reference(fp16, rows, d):
    lib = L()
    rng = np.random.default_rng(d)
    x = (rng.standard_normal((rows, d)) * 2 + 0.5).astype(np.float32)
    gm = (1 + 0.1 * rng.standard_normal(d)).astype(np.float32)
    bt = (0.1 * rng.standard_normal(d)).astype(np.float32)
    dy = rng.standard_normal((rows, d)).astype(np.float32)
    if fp16:
        x, gm, bt, dy = (ref.quantize_array(a) for a in (x, gm, bt, dy))
    y, dx, dg, db = ref.layer_norm(x, gm, bt, dy, fp16)
    dt = 1 if fp16 else 0
    T = lambda a: torch.tensor(a, device="cuda").to(TDT[dt])  # noqa: E731
    tx, tg, tb, tdy = T(x), T(gm), T(bt), T(dy)
    ty = torch.zeros_like(tx)
    stats = torch.zeros(rows, 2, device="cuda")
    lib.check(lib.sfk_layernorm_fwd(dt, ptr(tx), rows, d, ptr(tg), ptr(tb), ptr(ty), ptr(stats), stream()), True)
    tdx = torch.zeros_like(tx)
    part = torch.zeros(2 * 592 * d, device="cuda")
    npart = C.c_int()
    lib.check(lib.sfk_layernorm_bwd(dt, ptr(tx), ptr(tdy), rows, d, ptr(tg), ptr(stats), ptr(tdx), 0, ptr(part),
                                    C.byref(npart), stream()), True)
    dgt = torch.zeros(d, device="cuda").to(TDT[dt])
    dbt = torch.zeros(d, device="cuda").to(TDT[dt])
    lib.check(lib.sfk_colsum_finish(dt, ptr(part), npart.value, d, ptr(dgt), stream()), True)
    lib.check(lib.sfk_colsum_finish(dt, C.c_void_p(part.data_ptr() + 4 * npart.value * d), npart.value, d,
                                    ptr(dbt), stream()), True)
    torch.cuda.synchronize()
    rt = 2e-3 if fp16 else 1e-5
    np.testing.assert_allclose(ty.float().cpu().numpy(), y, rtol=rt, atol=rt)
    np.testing.assert_allclose(tdx.float().cpu().numpy(), dx, rtol=rt * 5, atol=rt * 5)
    np.testing.assert_allclose(dgt.float().cpu().numpy(), dg, rtol=rt * 5, atol=rt * 5 * rows ** 0.5)
    np.testing.assert_allclose(dbt.float().cpu().numpy(), db, rtol=rt * 5, atol=rt * 5 * rows ** 0.5)


def _spans(batch, qw, kw, lens, causal):
    kb, kl = [], []
    for b in range(batch):
        for t in range(qw):
            kb.append(b * kw)
            kl.append(t + 1 if causal else lens[b])
    return kb, kl


@pytest.mark.parametrize("fp16", [False, True])
@pytest.mark.parametrize("batch,qw,kw,heads,dh,causal", [(3, 7, 7, 2, 8, False), (2, 9, 9, 4, 16, True),
                                                        (4, 6, 11, 8, 64, False), (2, 40, 40, 4, 128, True),
                                                        (3, 25, 31, 16, 64, False),
                                                        # <= 16 wide, heads % 4 == 0: four heads per CTA
                                                        (5, 16, 16, 8, 64, True), (3, 12, 16, 16, 32, False),
                                                        (2, 16, 30, 4, 64, False),
                                                        # widths 65..128: one 8-warp CTA per (sentence, head)
                                                        (2, 100, 100, 4, 64, True), (2, 70, 90, 4, 64, False),
                                                        (2, 128, 128, 2, 128, False), (3, 120, 97, 4, 32, False),
                                                        # widths > 128: the two-kernel (dQ | dK,dV) backward
                                                        (1, 200, 200, 2, 32, True), (2, 64, 65, 2, 64, False)])
def test_attention_matches_reference(fp16, batch, qw, kw, heads, dh, causal):
    lib = L()
    rng = np.random.default_rng(qw * kw)
    d = heads * dh
    lens = rng.integers(1, kw + 1, batch).astype(np.int32)
    q = rng.standard_normal((batch * qw, d)).astype(np.float32)
    k = rng.standard_normal((batch * kw, d)).astype(np.float32)
    v = rng.standard_normal((batch * kw, d)).astype(np.float32)
    do = rng.standard_normal((batch * qw, d)).astype(np.float32)
    if fp16:
        q, k, v, do = (ref.quantize_array(a) for a in (q, k, v, do))
    kb, kl = _spans(batch, qw, kw, lens, causal)
    out, dq, dk, dv = ref.attention(q, k, v, heads, kb, kl, do, fp16)
    dt = 1 if fp16 else 0
    T = lambda a: torch.tensor(a, device="cuda").to(TDT[dt])  # noqa: E731
    tq, tk, tv, tdo = T(q), T(k), T(v), T(do)
    to, tdq, tdk, tdv = (torch.zeros_like(x) for x in (tq, tk, tk, tv))
    to = torch.zeros_like(tq)
    tdq = torch.zeros_like(tq)
    stats = torch.zeros(batch * qw * heads, 2, device="cuda")
    scratch = torch.zeros(batch * qw * heads, device="cuda")
    tl = torch.tensor(lens, device="cuda")
    a = lib.AttnArgs(dtype=dt, batch=batch, q_width=qw, k_width=kw, heads=heads, dh=dh, causal=int(causal),
                     k_len=ptr(tl), q=ptr(tq), ldq=d, k=ptr(tk), ldk=d, v=ptr(tv), ldv=d, o=ptr(to), ldo=d,
                     stats=ptr(stats), dout=ptr(tdo), lddo=d, dq=ptr(tdq), lddq=d, dk=ptr(tdk), lddk=d,
                     dv=ptr(tdv), lddv=d, scratch=ptr(scratch))
    lib.check(lib.sfk_attention_fwd(C.byref(a), stream()), True)
    lib.check(lib.sfk_attention_bwd(C.byref(a), stream()), True)
    torch.cuda.synchronize()
    rt = 4e-3 if fp16 else 2e-5
    for got, want in ((to, out), (tdq, dq), (tdk, dk), (tdv, dv)):
        np.testing.assert_allclose(got.float().cpu().numpy(), want, rtol=rt, atol=rt * 4)


@pytest.mark.parametrize("n,scale,ntok,lr,t,seed", [(10000, 512.0, 3333.0, 7e-4, 5, 3),
                                                   (1 << 20, 128.0, 51239.0, 5e-4, 1, 4),
                                                   (1 << 20, 0.5, 430117.0, 1e-3, 977, 5),
                                                   (1 << 20, 2.0 ** -14, 7.0, 2e-3, 40000, 6)])
def test_adam_bit_exact_with_reference(n, scale, ntok, lr, t, seed):
    """The fused unscale + 1/ntokens + Adam kernel against the reference's
    double-math update (optim.cpp:48-66): bit-identical master, moments and
    16-bit shadow over a million elements whose gradients and moments span
    many orders of magnitude (the constant divisions use a reciprocal plus one
    FMA correction, which must round exactly like a true division)."""
    lib = L()
    rng = np.random.default_rng(seed)
    p = rng.standard_normal(n).astype(np.float32)
    mag = 10.0 ** rng.uniform(-6, 3, n)
    g = ref.quantize_array((rng.standard_normal(n) * mag).astype(np.float32))
    m = (rng.standard_normal(n) * 10.0 ** rng.uniform(-9, -1, n)).astype(np.float32)
    v = (rng.random(n) * 10.0 ** rng.uniform(-14, -1, n)).astype(np.float32)
    g_pre = ((g / np.float32(scale)).astype(np.float32) / np.float32(ntok)).astype(np.float32)
    want_p, want_m, want_v = ref.adam(p, g_pre, m, v, t - 1, lr)
    tp, tm, tv = (torch.tensor(a, device="cuda") for a in (p, m, v))
    tg = torch.tensor(g, device="cuda").half()
    sh = torch.zeros(n, dtype=torch.float16, device="cuda")
    bc1, bc2 = 1 - 0.9 ** t, 1 - 0.98 ** t
    lib.check(lib.sfk_adam(1, ptr(tp), ptr(sh), 1, ptr(tg), ptr(tm), ptr(tv), n, lr, 0.9, 0.98, 1e-8, bc1, bc2,
                           scale, 1, ntok, None, stream()), True)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(tp.cpu().numpy().view(np.uint32), want_p.view(np.uint32))
    np.testing.assert_array_equal(tm.cpu().numpy().view(np.uint32), want_m.view(np.uint32))
    np.testing.assert_array_equal(tv.cpu().numpy().view(np.uint32), want_v.view(np.uint32))
    np.testing.assert_array_equal(sh.float().cpu().numpy(), ref.quantize_array(want_p))


def test_nonfinite_flag():
    lib = L()
    g = torch.zeros(1 << 20, dtype=torch.float16, device="cuda")
    flag = torch.zeros(4, dtype=torch.int32, device="cuda")
    lib.check(lib.sfk_nonfinite(1, ptr(g), g.numel(), ptr(flag), stream()), True)
    torch.cuda.synchronize()
    assert flag[0].item() == 0
    g[777777] = float("inf")
    lib.check(lib.sfk_nonfinite(1, ptr(g), g.numel(), ptr(flag), stream()), True)
    torch.cuda.synchronize()
    assert flag[0].item() == 1


@pytest.mark.parametrize("dt", [0, 1, 2])
@pytest.mark.parametrize("rows,n,ld", [(3584, 1024, 1024), (77, 3072, 3072), (5, 40, 48), (1000, 32768, 32768)])
def test_colsum_single_launch(dt, rows, n, ld):
    lib = L()
    g = torch.Generator(device="cuda").manual_seed(rows)
    x = torch.randn(rows, ld, device="cuda", generator=g).to(TDT[dt])
    out = torch.randn(n, device="cuda", generator=g).to(TDT[dt])
    want = (out.double() + x[:, :n].double().sum(0))
    part = torch.zeros(min(512 * n, 4 << 20), device="cuda")
    ctr = torch.zeros((n + 255) // 256, dtype=torch.int32, device="cuda")
    for _ in range(2):  # counters must re-arm
        o = out.clone()
        lib.check(lib.sfk_colsum(dt, ptr(x), rows, n, ld, ptr(part), ptr(ctr), ptr(o), stream()), True)
        torch.cuda.synchronize()
        tol = 1e-5 if dt == 0 else (4e-3 if dt == 1 else 2e-2)
        torch.testing.assert_close(o.double(), want.to(TDT[dt]).double(), rtol=tol, atol=tol * rows ** 0.5)
        assert int(ctr.abs().sum()) == 0


@pytest.mark.parametrize("rows,d", [(300, 512), (3584, 1024), (7, 64)])
def test_layernorm_bwd_fused_equals_two_phase(rows, d):
    lib = L()
    g = torch.Generator(device="cuda").manual_seed(d)
    x = torch.randn(rows, d, device="cuda", generator=g).half()
    dy = torch.randn(rows, d, device="cuda", generator=g).half()
    gm = (1 + 0.1 * torch.randn(d, device="cuda", generator=g)).half()
    bt = torch.zeros(d, device="cuda").half()
    y = torch.zeros_like(x)
    stats = torch.zeros(rows, 2, device="cuda")
    lib.check(lib.sfk_layernorm_fwd(1, ptr(x), rows, d, ptr(gm), ptr(bt), ptr(y), ptr(stats), stream()), True)
    part = torch.zeros(2 * 592 * d, device="cuda")
    dx1, dx2 = torch.zeros_like(x), torch.zeros_like(x)
    dg1, db1 = torch.zeros(d, device="cuda").half(), torch.zeros(d, device="cuda").half()
    dg2, db2 = dg1.clone(), db1.clone()
    npart = C.c_int()
    lib.check(lib.sfk_layernorm_bwd(1, ptr(x), ptr(dy), rows, d, ptr(gm), ptr(stats), ptr(dx1), 0, ptr(part),
                                    C.byref(npart), stream()), True)
    lib.check(lib.sfk_colsum_finish(1, ptr(part), npart.value, d, ptr(dg1), stream()), True)
    lib.check(lib.sfk_colsum_finish(1, C.c_void_p(part.data_ptr() + 4 * npart.value * d), npart.value, d, ptr(db1),
                                    stream()), True)
    ctr = torch.zeros(4, dtype=torch.int32, device="cuda")
    part2 = torch.zeros_like(part)
    lib.check(lib.sfk_layernorm_bwd_fused(1, ptr(x), ptr(dy), rows, d, ptr(gm), ptr(stats), ptr(dx2), 0, ptr(part2),
                                          ptr(ctr), ptr(dg2), ptr(db2), stream()), True)
    torch.cuda.synchronize()
    # dx identical; dgamma/dbeta fold the same partials in a different fixed
    # association (8-way ILP), so they agree to fp32 rounding before the fp16 store
    assert torch.equal(dx1, dx2)
    torch.testing.assert_close(dg1.float(), dg2.float(), rtol=2e-3, atol=2e-3)
    torch.testing.assert_close(db1.float(), db2.float(), rtol=2e-3, atol=2e-3)
    # split form (dx on the critical path, gamma/beta as a column reduction)
    dx4, dg4, db4 = torch.zeros_like(x), torch.zeros(d, device="cuda").half(), torch.zeros(d, device="cuda").half()
    lib.check(lib.sfk_layernorm_bwd_dx(1, ptr(x), ptr(dy), rows, d, ptr(gm), ptr(stats), ptr(dx4), 0, stream()), True)
    lib.check(lib.sfk_layernorm_bwd_params(1, ptr(x), ptr(dy), rows, d, ptr(stats), ptr(part2), None, ptr(dg4),
                                           ptr(db4), stream()), True)
    # single-launch form (arrival counter, fused fold): same sums, fixed order
    ctr5 = torch.zeros((d + 255) // 256, dtype=torch.int32, device="cuda")
    dg5, db5 = torch.zeros(d, device="cuda").half(), torch.zeros(d, device="cuda").half()
    for _ in range(2):
        dg5.zero_(), db5.zero_()
        lib.check(lib.sfk_layernorm_bwd_params(1, ptr(x), ptr(dy), rows, d, ptr(stats), ptr(part2), ptr(ctr5),
                                               ptr(dg5), ptr(db5), stream()), True)
        torch.cuda.synchronize()
        torch.testing.assert_close(dg1.float(), dg5.float(), rtol=2e-3, atol=2e-3)
        torch.testing.assert_close(db1.float(), db5.float(), rtol=2e-3, atol=2e-3)
        assert int(ctr5.abs().sum()) == 0
    torch.cuda.synchronize()
    assert torch.equal(dx1, dx4)
    torch.testing.assert_close(dg1.float(), dg4.float(), rtol=2e-3, atol=2e-3)
    torch.testing.assert_close(db1.float(), db4.float(), rtol=2e-3, atol=2e-3)
    # one-pass form: dx plus per-block gamma/beta partials, folded in block order
    dx6, dg6, db6 = torch.zeros_like(x), torch.zeros(d, device="cuda").half(), torch.zeros(d, device="cuda").half()
    part6 = torch.zeros(2 * ((rows + 15) // 16) * d, device="cuda")
    np6 = C.c_int()
    lib.check(lib.sfk_layernorm_bwd_dx_part(1, ptr(x), ptr(dy), rows, d, ptr(gm), ptr(stats), ptr(dx6), 0, ptr(part6),
                                            C.byref(np6), stream()), True)
    lib.check(lib.sfk_layernorm_bwd_fold(1, ptr(part6), np6.value, d, ptr(dg6), ptr(db6), stream()), True)
    torch.cuda.synchronize()
    assert torch.equal(dx1, dx6)
    torch.testing.assert_close(dg1.float(), dg6.float(), rtol=2e-3, atol=2e-3)
    torch.testing.assert_close(db1.float(), db6.float(), rtol=2e-3, atol=2e-3)
    # deterministic: a second run is bitwise identical
    dx3, dg3, db3 = torch.zeros_like(x), torch.zeros(d, device="cuda").half(), torch.zeros(d, device="cuda").half()
    lib.check(lib.sfk_layernorm_bwd_fused(1, ptr(x), ptr(dy), rows, d, ptr(gm), ptr(stats), ptr(dx3), 0, ptr(part2),
                                          ptr(ctr), ptr(dg3), ptr(db3), stream()), True)
    torch.cuda.synchronize()
    assert torch.equal(dx2, dx3) and torch.equal(dg2, dg3) and torch.equal(db2, db3)


def _segments(ids, chunk=16):
    """Host segment + chunk tables exactly as PackedBatch::pack builds them."""
    order = np.argsort(ids, kind="stable").astype(np.int32)
    uniq, off = [], []
    for i, r in enumerate(order):
        if i == 0 or ids[r] != ids[order[i - 1]]:
            uniq.append(int(ids[r]))
            off.append(i)
    off.append(len(order))
    chunks, multi, nslots = [], [], 0
    for u in range(len(uniq)):
        s0, s1 = off[u], off[u + 1]
        n = (s1 - s0 + chunk - 1) // chunk
        if n == 1:
            chunks += [uniq[u], s0, s1, -1]
            continue
        multi += [uniq[u], nslots, n, 0]
        for c in range(n):
            chunks += [uniq[u], s0 + c * chunk, min(s1, s0 + (c + 1) * chunk), nslots]
            nslots += 1
    return order, np.array(uniq, np.int32), np.array(off, np.int32), chunks, multi, nslots


@pytest.mark.parametrize("dt", [1, 2])
@pytest.mark.parametrize("rows,d,vocab", [(3584, 1024, 32768), (300, 64, 50), (33, 512, 5)])
def test_embedding_backward_chunked(dt, rows, d, vocab):
    """Embedding backward (tape.cpp:311-323): the chunked form (frequent ids
    split into <= 16-row chunks, chunk sums folded in order) equals the
    per-id sequential form to fp32 rounding and an fp64 reference within the
    storage tolerance; ids follow a Zipf head (eos/pad-like repeats)."""
    lib = L()
    rng = np.random.default_rng(rows)
    ids = np.minimum(rng.zipf(1.1, rows) - 1, vocab - 1).astype(np.int32)
    ids[::7] = 1  # a pad-like id repeated rows/7 times
    order, uniq, off, chunks, multi, nslots = _segments(ids)
    g = torch.Generator(device="cuda").manual_seed(d)
    dx = torch.randn(rows, d, device="cuda", generator=g).to(TDT[dt])
    table0 = (torch.randn(vocab, d, device="cuda", generator=g) * 0.1).to(TDT[dt])
    scale = float(np.sqrt(d))
    T = lambda a: torch.tensor(a, dtype=torch.int32, device="cuda")  # noqa: E731
    t_order, t_uniq, t_off = T(order), T(uniq), T(off)
    t_chunks, t_multi = T(chunks), T(multi if multi else [0, 0, 0, 0])
    scratch = torch.zeros(max(1, nslots) * d, device="cuda")
    a, b = table0.clone(), table0.clone()
    lib.check(lib.sfk_embed_bwd(dt, ptr(t_uniq), ptr(t_off), ptr(t_order), len(uniq), d, ptr(dx), scale, ptr(a),
                                stream()), True)
    lib.check(lib.sfk_embed_bwd_chunked(dt, ptr(t_chunks), len(chunks) // 4, ptr(t_multi), len(multi) // 4,
                                        ptr(t_order), d, ptr(dx), scale, ptr(scratch), ptr(b), stream()), True)
    torch.cuda.synchronize()
    q = lambda x: x.to(TDT[dt]).double()  # noqa: E731
    want = table0.double().index_add(0, torch.tensor(ids, device="cuda").long(), q(dx.double() * scale))
    tol = 4e-3 if dt == 1 else 2e-2
    torch.testing.assert_close(b.double(), q(want), rtol=tol, atol=tol)
    torch.testing.assert_close(a.double(), b.double(), rtol=tol, atol=tol)
    c = table0.clone()
    lib.check(lib.sfk_embed_bwd_chunked(dt, ptr(t_chunks), len(chunks) // 4, ptr(t_multi), len(multi) // 4,
                                        ptr(t_order), d, ptr(dx), scale, ptr(scratch), ptr(c), stream()), True)
    torch.cuda.synchronize()
    assert torch.equal(b, c)  # deterministic


def sk_workspace():
    sms = L().sfk_num_sms()
    return (torch.zeros(sms * 2 * 128 * 256, device="cuda"), torch.zeros(2 * sms, dtype=torch.int32, device="cuda"))


@pytest.mark.parametrize("layout", [(True, True), (True, False), (False, False)])
@pytest.mark.parametrize("shape", [(1024, 1024, 3584), (3584, 1024, 1024), (3000, 4096, 1024), (200, 296, 640),
                                   (3584, 3072, 1024), (136, 248, 4096)])
@pytest.mark.parametrize("flags", [0, 7, 32])
def test_gemm_stream_k(layout, shape, flags):
    """Stream-K (k-loop of the last wave split across all SMs, parts summed
    in k order by the last arriving CTA) against fp64; deterministic, and the
    arrival counters are re-armed for the next launch."""
    ws = sk_workspace()
    m, n, k = shape
    got, want = run_gemm(m, n, k, 1, *layout, flags=flags, seed=3, stream_k=1, ws=ws)
    tol = 2e-3 * (k ** 0.5)
    torch.testing.assert_close(got, want, rtol=4e-3, atol=tol)
    assert int(ws[1].abs().sum()) == 0
    again, _ = run_gemm(m, n, k, 1, *layout, flags=flags, seed=3, stream_k=1, ws=ws)
    assert torch.equal(got, again)


@pytest.mark.parametrize("dtype", [1, 2])
@pytest.mark.parametrize("shape", [(1024, 1024, 3584), (3072, 1024, 3000), (200, 296, 640), (4096, 1024, 37),
                                   (1024, 4096, 2048), (600, 512, 700)])
@pytest.mark.parametrize("pair", [0, 1])
def test_gemm_fused_bias_grad(dtype, shape, pair):
    """Weight-gradient GEMM with the bias gradient fused (add_bias backward,
    tape.cpp:347-358): dW = q(dW + dY^T X) as before and db = q(db + sum_rows dY)
    from the same A tiles; fp64 reference, deterministic."""
    lib = L()
    m, n, k = shape  # m = out features, n = in features, k = rows
    g = torch.Generator(device="cuda").manual_seed(m + k)
    td = TDT[dtype]
    dy = (torch.randn(k, m, device="cuda", generator=g) * 0.5).to(td)   # A(i,kk) = dy[kk, i]: MN-major
    x = (torch.randn(k, n, device="cuda", generator=g) * 0.5).to(td)    # B(j,kk) = x[kk, j]: MN-major
    dw0 = torch.randn(m, n, device="cuda", generator=g).to(td)
    db0 = torch.randn(m, device="cuda", generator=g).to(td)
    outs = []
    for _ in range(2):
        dw, db = dw0.clone(), db0.clone()
        args = lib.GemmArgs(m=m, n=n, k=k, dtype=dtype, a=ptr(dy), lda=m, a_kmajor=0, b=ptr(x), ldb=n, b_kmajor=0,
                            c=ptr(dw), ldc=n, flags=lib.EPI_ACCUM, stream_k=-1, bias_grad=ptr(db), pair=pair,
                            tile_n=256 if pair else 0)
        lib.check(lib.sfk_gemm(C.byref(args), stream()), kernel=True)
        torch.cuda.synchronize()
        outs.append((dw, db))
    q = lambda v: v.to(td).double()  # noqa: E731
    want_w = q(dw0.double() + dy.double().t() @ x.double())
    want_b = q(db0.double() + dy.double().sum(0))
    tol = (4e-3 if dtype == 1 else 2e-2)
    torch.testing.assert_close(outs[0][0].double(), want_w, rtol=tol, atol=tol * k ** 0.5)
    torch.testing.assert_close(outs[0][1].double(), want_b, rtol=tol, atol=tol * k ** 0.5)
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])


# ---------------------------------------------------------------- generation kernels

def test_gather_rows_reorders_every_matrix():
    lib = L()
    rows, row_elems, nmat = 37, 96, 5
    src = torch.randn(nmat, rows, row_elems, device="cuda")
    dst = torch.empty_like(src)
    idx = torch.randint(0, rows, (rows,), device="cuda", dtype=torch.int32)
    lib.check(lib.sfk_gather_rows(ptr(src), ptr(dst), ptr(idx), rows, row_elems * 4, row_elems * 4, nmat,
                                  rows * row_elems * 4, stream()), kernel=True)
    torch.cuda.synchronize()
    assert torch.equal(dst, src[:, idx.long()])
    # prefix copy: only the first 40 elements of each row move
    dst2 = torch.zeros_like(src)
    lib.check(lib.sfk_gather_rows(ptr(src), ptr(dst2), ptr(idx), rows, row_elems * 4, 40 * 4, nmat,
                                  rows * row_elems * 4, stream()), kernel=True)
    torch.cuda.synchronize()
    assert torch.equal(dst2[..., :40], src[:, idx.long(), :40]) and not dst2[..., 40:].any()
    assert lib.sfk_gather_rows(ptr(src), ptr(src), ptr(idx), rows, row_elems * 4, row_elems * 4, nmat, 0,
                               stream()) != 0


@pytest.mark.parametrize("row_elems,copy", [(97, 50), (33, 33), (10, 3)])
def test_gather_rows_any_row_size(row_elems, copy):
    """fp32 caches of an odd model width have rows that are not 16-byte
    multiples: the gather falls back to 4-byte (or byte) copies instead of
    refusing."""
    lib = L()
    rows, nmat = 21, 3
    src = torch.randn(nmat, rows, row_elems, device="cuda")
    dst = torch.zeros_like(src)
    idx = torch.randint(0, rows, (rows,), device="cuda", dtype=torch.int32)
    lib.check(lib.sfk_gather_rows(ptr(src), ptr(dst), ptr(idx), rows, row_elems * 4, copy * 4, nmat,
                                  rows * row_elems * 4, stream()), kernel=True)
    torch.cuda.synchronize()
    assert torch.equal(dst[..., :copy], src[:, idx.long(), :copy]) and not dst[..., copy:].any()


def test_beam_topk_ranks_minus_inf_candidates():
    """A row with fewer than kk finite log-probs still returns kk distinct
    tokens: the -inf ones in token order (the reference's stable sort lists
    them), never padding with repeated eos."""
    lib = L()
    V, kk, rows = 50, 8, 2
    lg = torch.full((rows, V), float("-inf"), device="cuda")
    lg[0, [3, 7, 11]] = torch.tensor([1.0, 2.0, 0.5], device="cuda")
    lg[1, :] = torch.randn(V, device="cuda")
    lse = torch.zeros(rows, device="cuda")
    eos_lp = torch.zeros(rows, device="cuda")
    tok = torch.zeros(rows, kk, dtype=torch.int32, device="cuda")
    lp = torch.zeros(rows, kk, device="cuda")
    cum = torch.zeros(rows, dtype=torch.float64, device="cuda")
    lib.check(lib.sfk_beam_topk(0, ptr(lg), V, rows, V, ptr(cum), kk, 2, ptr(lse), ptr(eos_lp), ptr(tok), ptr(lp),
                                stream()), kernel=True)
    torch.cuda.synchronize()
    t0 = tok[0].tolist()
    assert t0[:3] == [7, 3, 11]
    assert t0[3:] == [0, 1, 2, 4, 5]  # -inf candidates, lowest token first
    assert len(set(tok[1].tolist())) == kk


@pytest.mark.parametrize("dt,V,kk", [(0, 1000, 8), (1, 32768, 8), (2, 5000, 10), (0, 7, 7)])
def test_beam_topk_order_and_values(dt, V, kk):
    """sfk_beam_topk against a host ranking of every candidate: key = cum +
    (logit - lse) descending, token ascending on ties (generate.cpp:246-249);
    ties are forced by repeating logit values."""
    lib = L()
    rows = 12
    g = torch.Generator(device="cuda").manual_seed(dt * 7 + kk)
    logits = (torch.randn(rows, V, device="cuda", generator=g) * 3).to(TDT[dt])
    logits[:, 1::3] = logits[:, 0:1]  # many exact ties in every row
    ld = V
    cum = torch.randn(rows, device="cuda", dtype=torch.float64, generator=g) * 10
    lse = torch.empty(rows, device="cuda")
    eos_lp = torch.empty(rows, device="cuda")
    tok = torch.empty(rows, kk, device="cuda", dtype=torch.int32)
    lp = torch.empty(rows, kk, device="cuda")
    lib.check(lib.sfk_beam_topk(dt, ptr(logits), ld, rows, V, ptr(cum), kk, 2, ptr(lse), ptr(eos_lp), ptr(tok),
                                ptr(lp), stream()), kernel=True)
    torch.cuda.synchronize()
    x = logits.float().cpu().numpy()
    c = cum.cpu().numpy()
    want_lse = np.log(np.exp(x.astype(np.float64) - x.max(1, keepdims=True)).sum(1)) + x.max(1)
    np.testing.assert_allclose(lse.cpu().numpy(), want_lse, rtol=0, atol=1e-4)
    got_lse = lse.cpu().numpy()
    np.testing.assert_allclose(eos_lp.cpu().numpy(), x[:, 2] - got_lse, atol=1e-6)
    for r in range(rows):
        lpr = (x[r] - got_lse[r]).astype(np.float32)
        key = c[r] + lpr.astype(np.float64)
        order = sorted(range(V), key=lambda v: (-key[v], v))[:kk]
        assert tok[r].cpu().tolist() == order, r
        np.testing.assert_array_equal(lp[r].cpu().numpy(), lpr[order])


@pytest.mark.parametrize("dt,V,kk", [(0, 1000, 5), (1, 32768, 20)])
def test_topk_raw_mode_for_sampling(dt, V, kk):
    """cum == NULL: rank by the raw logit (ties to the lower id, as
    sample_from_topk's stable sort, generate.cpp:360-365) and return raw logits."""
    lib = L()
    rows = 6
    g = torch.Generator(device="cuda").manual_seed(11 + dt)
    logits = (torch.randn(rows, V, device="cuda", generator=g) * 2).to(TDT[dt])
    logits[:, 5::7] = logits[:, 3:4]
    lse, eos_lp, lp = (torch.empty(rows, device="cuda") for _ in range(3))
    tok = torch.empty(rows, kk, device="cuda", dtype=torch.int32)
    lp = torch.empty(rows, kk, device="cuda")
    lib.check(lib.sfk_beam_topk(dt, ptr(logits), V, rows, V, None, kk, 2, ptr(lse), ptr(eos_lp), ptr(tok), ptr(lp),
                                stream()), kernel=True)
    torch.cuda.synchronize()
    x = logits.float().cpu().numpy()
    for r in range(rows):
        order = sorted(range(V), key=lambda v: (-x[r, v], v))[:kk]
        assert tok[r].cpu().tolist() == order
        np.testing.assert_array_equal(lp[r].cpu().numpy(), x[r, order])


class LnFoldJob(C.Structure):
    _fields_ = [("part", C.c_void_p), ("dgamma", C.c_void_p), ("dbeta", C.c_void_p), ("nparts", C.c_int),
                ("d", C.c_int)]


@pytest.mark.parametrize("dt", [1, 2])
def test_layernorm_params_partial_and_batched_fold_match_reference(dt):
    """gamma/beta gradients as the trainer computes them: one partial pass per
    LayerNorm node, then a single fold launch for several nodes (different
    widths and row counts), each gradient accumulated q(old + sum) into a
    non-zero buffer -- against the reference's layer_norm backward
    (tape.cpp:383-418), summed over rows."""
    lib = L()
    rng = np.random.default_rng(11)
    jobs, want, outs, keep = [], [], [], []
    for rows, d in ((3584, 1024), (1234, 512), (37, 64), (900, 1024)):
        x = ref.quantize_array((rng.standard_normal((rows, d)) * 2 + 0.5).astype(np.float32))
        gm = ref.quantize_array((1 + 0.1 * rng.standard_normal(d)).astype(np.float32))
        bt = ref.quantize_array((0.1 * rng.standard_normal(d)).astype(np.float32))
        dy = ref.quantize_array(rng.standard_normal((rows, d)).astype(np.float32))
        _, _, dg, db = ref.layer_norm(x, gm, bt, dy, False)
        g0 = ref.quantize_array((0.5 * rng.standard_normal(d)).astype(np.float32))
        b0 = ref.quantize_array((0.5 * rng.standard_normal(d)).astype(np.float32))
        tx, tg, tb, tdy = (torch.tensor(a, device="cuda").to(TDT[dt]) for a in (x, gm, bt, dy))
        ty, stats = torch.zeros_like(tx), torch.zeros(rows, 2, device="cuda")
        lib.check(lib.sfk_layernorm_fwd(dt, ptr(tx), rows, d, ptr(tg), ptr(tb), ptr(ty), ptr(stats), stream()), True)
        part = torch.full((2 * 148 * d,), float("nan"), device="cuda")
        npart = C.c_int()
        lib.check(lib.sfk_layernorm_bwd_params_partial(dt, ptr(tx), ptr(tdy), rows, d, ptr(stats), ptr(part),
                                                       C.byref(npart), stream()), True)
        assert 1 <= npart.value <= 148
        og, ob = torch.tensor(g0, device="cuda").to(TDT[dt]), torch.tensor(b0, device="cuda").to(TDT[dt])
        jobs.append(LnFoldJob(part.data_ptr(), og.data_ptr(), ob.data_ptr(), npart.value, d))
        want.append((g0.astype(np.float64) + dg, b0.astype(np.float64) + db))
        outs.append((og, ob))
        keep += [tx, tdy, stats, part]
    arr = (LnFoldJob * len(jobs))(*jobs)
    lib.check(lib.sfk_layernorm_bwd_params_fold(dt, arr, len(jobs), stream()), True)
    torch.cuda.synchronize()
    rt = 4e-3 if dt == 1 else 1.6e-2
    for (og, ob), (wg, wb), j in zip(outs, want, jobs):
        sc = np.sqrt(j.nparts * 1.0)
        np.testing.assert_allclose(og.float().cpu().numpy(), wg, rtol=rt, atol=rt * 10 * sc)
        np.testing.assert_allclose(ob.float().cpu().numpy(), wb, rtol=rt, atol=rt * 10 * sc)


@pytest.mark.parametrize("dtype", [1, 2])
@pytest.mark.parametrize("tile_n", [256, 128])
@pytest.mark.parametrize("layout,flags", [((True, True), 1 | 2 | 16), ((True, True), 1 | 2 | 4), ((True, False), 0),
                                          ((True, False), 32), ((True, False), 8), ((False, False), 32)])
@pytest.mark.parametrize("shape", [(3584, 1024, 1024), (3584, 1024, 4096), (3584, 3072, 1024), (3584, 4096, 1024),
                                   (1024, 1024, 3584), (3000, 1000, 2000)])
def test_gemm_pair_stream_k(dtype, tile_n, layout, flags, shape):
    """CTA-pair GEMM with the auto stream-K split of the last wave (fp32
    partials per CTA, summed in k order by the last arriving part, TMA-store
    epilogue) against fp64; deterministic, counters re-armed."""
    ws = sk_workspace()
    m, n, k = shape
    got, want = run_gemm(m, n, k, dtype, *layout, flags=flags, seed=5, stream_k=0, ws=ws, pair=1, tile_n=tile_n)
    tol = (4e-3 if dtype == 1 else 2e-2)
    torch.testing.assert_close(got, want, rtol=tol, atol=tol * max(1.0, k ** 0.5 * 0.25))
    assert int(ws[1].abs().sum()) == 0
    again, _ = run_gemm(m, n, k, dtype, *layout, flags=flags, seed=5, stream_k=0, ws=ws, pair=1, tile_n=tile_n)
    assert torch.equal(got, again)


@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("heads,dh", [(16, 64), (4, 32)])
def test_attention_parts_match_single_calls(causal, heads, dh):
    """sfk_attention_{fwd,bwd}_parts (the parts of a multi-part pass, one
    launch per width class) give bitwise the results of one call per part:
    parts of 12/16 (four heads per CTA), 30/25 (32-row CTAs), 50, 100 and 150
    positions, all inside one fused-QKV buffer."""
    lib = L()
    rng = np.random.default_rng(7 + heads + int(causal))
    d = heads * dh
    shapes = [(6, 12), (5, 16), (4, 30), (3, 25), (2, 50), (2, 100), (1, 150)]  # (sentences, width)
    rows = sum(b * w for b, w in shapes)
    qkv = torch.tensor(rng.standard_normal((rows, 3 * d)) * 0.5, device="cuda").half()
    do = torch.tensor(rng.standard_normal((rows, d)), device="cuda").half()
    lens = [torch.tensor(rng.integers(1, w + 1, b).astype(np.int32), device="cuda") for b, w in shapes]

    def run(split):
        o = torch.zeros(rows, d, device="cuda").half()
        dqkv = torch.zeros(rows, 3 * d, device="cuda").half()
        st = torch.zeros(rows * heads, 2, device="cuda")
        sc = torch.zeros(rows * heads, device="cuda")
        args, r0 = [], 0
        for (b, w), ln in zip(shapes, lens):
            q = qkv.data_ptr() + r0 * 3 * d * 2
            dq = dqkv.data_ptr() + r0 * 3 * d * 2
            args.append(lib.AttnArgs(dtype=1, batch=b, q_width=w, k_width=w, heads=heads, dh=dh, causal=int(causal),
                                     k_len=ptr(ln), q=q, ldq=3 * d, k=q + 2 * d, ldk=3 * d, v=q + 4 * d, ldv=3 * d,
                                     o=o.data_ptr() + r0 * d * 2, ldo=d, stats=st.data_ptr() + r0 * heads * 8,
                                     dout=do.data_ptr() + r0 * d * 2, lddo=d, dq=dq, lddq=3 * d, dk=dq + 2 * d,
                                     lddk=3 * d, dv=dq + 4 * d, lddv=3 * d, scratch=sc.data_ptr() + r0 * heads * 4))
            r0 += b * w
        if split:
            for a in args:
                lib.check(lib.sfk_attention_fwd(C.byref(a), stream()), True)
            for a in args:
                lib.check(lib.sfk_attention_bwd(C.byref(a), stream()), True)
        else:
            arr = (lib.AttnArgs * len(args))(*args)
            lib.check(lib.sfk_attention_fwd_parts(arr, len(args), stream()), True)
            nf = lib.sfk_attention_last_launches()
            lib.check(lib.sfk_attention_bwd_parts(arr, len(args), stream()), True)
            assert 0 < nf < len(args)  # width classes share launches
        torch.cuda.synchronize()
        return o, dqkv, st

    for x, y in zip(run(True), run(False)):
        assert torch.equal(x, y)
