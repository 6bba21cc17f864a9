"""Pin the oracle (the reference built from its own sources) against the
known-answer values the reference's own test-suite holds for this path
(SURVEY.md §8(c)), and against the committed golden fixtures."""
import json
import math
import os

import numpy as np
import pytest

from oracle import ref

pytestmark = pytest.mark.skipif(not ref.available() and not os.path.isdir(ref.REFERENCE),
                                reason="oracle library not built")

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_fp16_known_answers():
    # proj/tests/test_numerics.cpp:45-63
    q = ref.quantize_fp16
    assert q(0.5) == 0.5
    assert math.isinf(q(1.0e5))
    assert q(2.0 ** -25) == 0.0 and math.copysign(1, q(2.0 ** -25)) > 0
    assert math.copysign(1, q(-2.0 ** -25)) < 0
    assert q(65504.0) == 65504.0
    assert q(65519.0) == 65504.0
    assert math.isinf(q(65520.0))
    assert q(6.0e-8) == 2.0 ** -24
    assert q(np.float32(1.0) / np.float32(3.0)) == 0.333251953125
    assert q(345.678) == 345.75
    assert q(0.1) == 0.0999755859375
    assert math.isnan(q(float("nan")))


def test_fp16_matches_numpy_binary16_sweep():
    # test_numerics.cpp:65-98: agreement with an independent binary16 conversion
    rng = np.random.default_rng(0)
    bits = rng.integers(0, 2 ** 32, 200_000, dtype=np.uint64).astype(np.uint32)
    x = bits.view(np.float32)
    x = x[np.isfinite(x)]
    got = ref.quantize_array(x)
    want = x.astype(np.float16).astype(np.float32)
    np.testing.assert_array_equal(got.view(np.uint32), want.view(np.uint32))


def test_criterion_known_answers():
    # test_criterions.cpp:55-142
    loss, nll, corr, _ = ref.xent(np.zeros((1, 4), np.float32), [2], 0.0)
    assert abs(loss[0] - math.log(4)) < 1e-6
    loss, nll, _, _ = ref.xent(np.zeros((1, 8), np.float32), [5], 0.3)
    assert abs(loss[0] - math.log(8)) < 1e-6
    lg = np.array([[0.0, 0.0, math.log(2.0)]], np.float32)
    loss, nll, _, _ = ref.xent(lg, [2], 0.1)
    assert abs(loss[0] - 0.7393573) < 1e-5 * 0.7393573
    assert abs(nll[0] - math.log(2.0)) < 1e-6
    lg = np.zeros((1, 4), np.float32)
    lg[0, 2] = 1e4
    loss, _, corr, _ = ref.xent(lg, [2], 0.0)
    assert loss[0] < 1e-3 and corr[0] == 1


def test_optimizer_known_answers():
    # test_optim.cpp:45-53 (Adam t=1 moves by ~lr), 122-147 (inverse sqrt)
    p, m, v = ref.adam([1.0], [1.0], [0.0], [0.0], 0, 0.1, 0.9, 0.999, 1e-8)
    assert abs(p[0] - 0.9) < 1e-6
    assert ref.inverse_sqrt(5e-4, 4000, 0.0, 4000) == 5e-4
    assert ref.inverse_sqrt(5e-4, 4000, 0.0, 16000) == 5e-4 / 2
    assert abs(ref.inverse_sqrt(5e-4, 4000, 0.0, 1) - 5e-4 / 4000) < 1e-18


def test_minibatch_known_answer():
    # test_data.cpp:306-331
    from paper_1904_01038_b200 import Corpus
    c = Corpus.from_pairs([([5, 2], [8, 9, 2]), ([6, 7, 2], [4, 2])])
    mb = ref.make_minibatch(c, [0, 1])
    assert mb["source"].ravel().tolist() == [5, 2, 1, 6, 7, 2]
    assert mb["target_in"].ravel().tolist() == [0, 8, 9, 0, 4, 1]
    assert mb["target_out"].ravel().tolist() == [8, 9, 2, 4, 2, 1]
    assert mb["ntokens"] == 5


def test_packing_known_answers():
    # test_data.cpp:176-212
    from paper_1904_01038_b200 import Corpus

    def mk(s, t):
        return ([4] * (s - 1) + [2], [4] * (t - 1) + [2])
    c = Corpus.from_pairs([mk(3, 3), mk(3, 3), mk(7, 7)])
    assert ref.make_batches(c, 6, 0, 7) == [[0, 1], [2]]
    c = Corpus.from_pairs([mk(4, 4)] * 10)
    assert [len(b) for b in ref.make_batches(c, 40, 5, 7)] == [5, 5]
    c = Corpus.from_pairs([mk(9, 2), mk(2, 2)])
    assert ref.make_batches(c, 5, 0, 7) == [[1], [0]]


def test_golden_fixtures_replay():
    """Committed fixtures (tests/golden/*.json, made by tests/golden/make_golden.py
    from the reference) still match the oracle built here."""
    path = os.path.join(GOLDEN, "oracle_golden.json")
    if not os.path.exists(path):
        pytest.skip("golden fixtures not generated")
    g = json.load(open(path))
    assert [int(x) for x in ref.rng_u64(1, 4242, 0, 8)] == g["rng_u64_1_4242"]
    assert ref.shuffle_epoch(37, 1, 3) == g["shuffle_37_1_3"]
    from paper_1904_01038_b200 import synthetic_corpus
    c = synthetic_corpus(200, 1000, 1000, 1.1, 1)
    assert ref.make_batches(c, 512, 0, 1) == g["batches_200_512"]
    for case in g["xent"]:
        lg = np.array(case["logits"], np.float32)
        loss, nll, corr, dl = ref.xent(lg, case["gold"], case["eps"], case["fp16"], case["seed"])
        np.testing.assert_array_equal(loss, np.array(case["loss"], np.float32))
        np.testing.assert_array_equal(dl, np.array(case["dlogits"], np.float32))
