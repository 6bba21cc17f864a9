"""Pin the numpy restatement (oracle/restate.py) against the compiled reference
(oracle/_ref): integer/bitwise pieces exactly, floating-point ops within 1e-5."""
import math

import numpy as np
import pytest

import paper_1904_01038_b200 as sqf
from oracle import ref, restate


def test_rng_and_shuffles_exact():
    for seed, stream, ctr in [(1, 4242, 0), (7, 9, 5), (2 ** 40 + 3, 2 ** 33, 77)]:
        r = restate.RngStream(seed, stream, ctr)
        assert [r.next_u64() for _ in range(16)] == [int(x) for x in ref.rng_u64(seed, stream, ctr, 16)]
        r = restate.RngStream(seed, stream, ctr)
        assert [r.next_double() for _ in range(8)] == ref.rng_double(seed, stream, ctr, 8).tolist()
        r = restate.RngStream(seed, stream, ctr)
        assert [r.next_below(1000003) for _ in range(8)] == [int(x) for x in
                                                              ref.rng_below(seed, stream, ctr, 1000003, 8)]
    for n, seed, ep in [(1, 1, 1), (37, 1, 3), (500, 11, 2)]:
        assert restate.shuffle_epoch(n, seed, ep) == ref.shuffle_epoch(n, seed, ep)


def test_batching_exact():
    c = sqf.synthetic_corpus(400, 1000, 1000, 1.1, 5)
    pairs = [c.pair(i) for i in range(c.npairs)]
    for budget, ms in [(512, 0), (2048, 9), (30, 0)]:
        assert restate.make_batches(pairs, budget, ms) == ref.make_batches(c, budget, ms, 1)
    mem = ref.make_batches(c, 1024, 0, 1)[3]
    a, b = restate.make_minibatch(pairs, mem), ref.make_minibatch(c, mem)
    for k in ("source", "target_in", "target_out", "src_lens", "tgt_lens"):
        np.testing.assert_array_equal(a[k], b[k])
    assert a["ntokens"] == b["ntokens"]
    rng = np.random.default_rng(0)
    sizes = rng.integers(1, 3000, 40).tolist()
    assert restate.bucket_gradients(sizes, 5000) == ref.bucket_gradients(sizes, 5000)


def test_fp16_scaler_schedule_adam_exact():
    x = np.random.default_rng(1).standard_normal(5000).astype(np.float32) * 1e3
    np.testing.assert_array_equal(restate.quantize_fp16(x), ref.quantize_array(x))
    ov = (np.random.default_rng(2).random(200) < 0.1).astype(int).tolist()
    assert restate.scaler_run(128.0, 5, 0.03125, 32768.0, ov) == ref.scaler_run(128.0, 5, 0.03125, 32768.0, ov)
    for step in (1, 10, 4000, 9999):
        assert restate.inverse_sqrt(5e-4, 4000, 0.0, step) == ref.inverse_sqrt(5e-4, 4000, 0.0, step)
    rng = np.random.default_rng(3)
    p, g = rng.standard_normal(999).astype(np.float32), rng.standard_normal(999).astype(np.float32)
    m, v = (rng.standard_normal(999) * 0.01).astype(np.float32), (rng.random(999) * 0.01).astype(np.float32)
    a, b = restate.adam(p, g, m, v, 4, 1e-3), ref.adam(p, g, m, v, 4, 1e-3)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x.view(np.uint32), y.view(np.uint32))


def test_xent_layernorm_attention_match_reference():
    rng = np.random.default_rng(4)
    lg = (rng.standard_normal((6, 50)) * 2).astype(np.float32)
    gold = np.array([3, 1, 7, 49, 0, 1], np.int32)
    for eps in (0.0, 0.1):
        a, b = restate.xent(lg, gold, eps, 2.0), ref.xent(lg, gold, eps, False, 2.0)
        np.testing.assert_allclose(a[0], b[0], rtol=1e-5, atol=1e-6)
        np.testing.assert_array_equal(a[2], b[2])
        np.testing.assert_allclose(a[3], b[3], rtol=1e-5, atol=1e-6)
    x = rng.standard_normal((9, 32)).astype(np.float32)
    gm, bt = (1 + 0.1 * rng.standard_normal(32)).astype(np.float32), (0.1 * rng.standard_normal(32)).astype(np.float32)
    dy = rng.standard_normal((9, 32)).astype(np.float32)
    for u, w in zip(restate.layer_norm(x, gm, bt, dy), ref.layer_norm(x, gm, bt, dy)):
        np.testing.assert_allclose(u, w, rtol=1e-5, atol=1e-5)
    q, k, v, do = (rng.standard_normal((8, 16)).astype(np.float32) for _ in range(4))
    kb = [0, 0, 0, 0, 4, 4, 4, 4]
    kl = [1, 2, 3, 4, 4, 4, 4, 4]
    for u, w in zip(restate.attention(q, k, v, 2, kb, kl, do), ref.attention(q, k, v, 2, kb, kl, do)):
        np.testing.assert_allclose(u, w, rtol=1e-5, atol=1e-5)
    assert math.isinf(float(restate.quantize_fp16(65520.0)))


def test_known_answers_hold_for_restatement():
    # test_criterions.cpp:120-142 / test_optim.cpp:45-53
    loss, nll, _, _ = restate.xent(np.array([[0.0, 0.0, math.log(2.0)]]), np.array([2]), 0.1)
    assert abs(loss[0] - 0.7393573) < 1e-6
    p, _, _ = restate.adam([1.0], [1.0], [0.0], [0.0], 0, 0.1, 0.9, 0.999, 1e-8)
    assert abs(p[0] - 0.9) < 1e-6
    assert restate.split_counts(10, 2, 2) == [3, 3, 2, 2]
    with pytest.raises(ValueError):
        restate.shuffle_epoch(3, 1, 0)
