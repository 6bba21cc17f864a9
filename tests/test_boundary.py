"""CPU tests of the drop-in boundary: the C-ABI library loads and exports every
symbol include/*.h declares, and the host-side pieces of the hot path (batch
composition, padding masks, epoch shuffles, split dispatch, buckets, parameter
layout + init, loss-scaler policy, LR schedules, binary16 rounding) are
bit-exact with the reference oracle on the same seeded inputs."""
import ctypes
import math
import os
import re

import numpy as np
import pytest

import paper_1904_01038_b200 as sqf
from paper_1904_01038_b200 import _lib
from oracle import ref

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    names = []
    for h in ("sqf_kernels.h", "sqf_trainer.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names += re.findall(r"\b((?:sfk|sqf)_[a-z0-9_]+)\s*\(", src)
    return sorted(set(names))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [n for n in declared_symbols() if not hasattr(lib, n)]
    assert not missing, missing
    assert len(declared_symbols()) >= 40


@pytest.mark.parametrize("npairs,vocab,budget", [(300, 1000, 1024), (2000, 32768, 4096), (500, 10000, 256)])
def test_batches_shuffles_minibatches_bit_exact(npairs, vocab, budget):
    c = sqf.synthetic_corpus(npairs, vocab, vocab, 1.1, 1)
    mine = sqf.make_batches(c, budget, 0, 1)
    theirs = ref.make_batches(c, budget, 0, 1)
    assert mine == theirs
    assert sorted(x for b in mine for x in b) == list(range(npairs))  # partition
    for epoch in (1, 2, 5):
        assert sqf.shuffle_epoch(len(mine), 1, epoch) == ref.shuffle_epoch(len(theirs), 1, epoch)
    for b in mine[:: max(1, len(mine) // 7)]:
        a, r = sqf.make_minibatch(c, b), ref.make_minibatch(c, b)
        for k in ("source", "target_in", "target_out", "src_lens", "tgt_lens"):
            np.testing.assert_array_equal(a[k], r[k])
        assert (a["rows"], a["src_width"], a["tgt_width"], a["ntokens"]) == \
               (r["rows"], r["src_width"], r["tgt_width"], r["ntokens"])
        # padding mask: pad exactly beyond each length, eos at len-1
        for i, (sl, tl) in enumerate(zip(a["src_lens"], a["tgt_lens"])):
            assert (a["source"][i, sl:] == sqf.PAD).all() and a["source"][i, sl - 1] == sqf.EOS
            assert (a["target_out"][i, tl:] == sqf.PAD).all() and a["target_in"][i, 0] == sqf.BOS


def test_max_sentences_and_edge_cases():
    c = sqf.synthetic_corpus(400, 1000, 1000, 1.1, 3)
    assert sqf.make_batches(c, 2048, 7, 1) == ref.make_batches(c, 2048, 7, 1)
    # budget smaller than any pair: every pair is an oversized singleton
    assert sqf.make_batches(c, 1, 0, 1) == ref.make_batches(c, 1, 0, 1)
    empty = sqf.Corpus(*(np.zeros(0, np.int32) for _ in range(4)))
    assert sqf.make_batches(empty, 100) == []
    with pytest.raises(sqf.NativeError) as e:
        sqf.make_batches(c, 0)
    assert e.value.kind == "ConfigError"
    with pytest.raises(sqf.NativeError):
        sqf.shuffle_epoch(5, 1, 0)


def test_split_counts_follow_trainer_split_batch():
    # trainer.cpp:186-202: base = rows/(W*A), first rem groups take one more
    for rows, w, a in [(10, 2, 2), (3, 2, 2), (37, 4, 3), (1, 1, 8)]:
        c = sqf.split_counts(rows, w, a)
        g = w * a
        assert c == [rows // g + (1 if i < rows % g else 0) for i in range(g)]


def test_buckets_bit_exact():
    rng = np.random.default_rng(0)
    for _ in range(20):
        sizes = rng.integers(1, 5000, rng.integers(1, 60)).tolist()
        for th in (1, 100, 16384, 10 ** 9):
            assert sqf.bucket_gradients(sizes, th) == ref.bucket_gradients(sizes, th)


CONFIGS = [
    ("tiny_transformer", {"src_vocab": 37, "tgt_vocab": 41}),
    ("transformer_base_defaults", {"src_vocab": 1000, "tgt_vocab": 1000}),
    ("transformer_base_defaults", {"src_vocab": 1000, "tgt_vocab": 1000, "share_embeddings": True, "seed": 7}),
]


@pytest.mark.parametrize("arch,ov", CONFIGS)
def test_parameter_layout_and_init_bit_exact(arch, ov):
    mine = sqf.model_init(arch, ov)
    c = sqf.synthetic_corpus(20, ov["src_vocab"], ov["tgt_vocab"], 1.1, 1)
    rt = ref.RefTrainer(arch, ov, c, ov["src_vocab"], ov["tgt_vocab"])
    theirs = rt.params()
    assert mine.shape == theirs.shape
    np.testing.assert_array_equal(mine.view(np.uint32), theirs.view(np.uint32))


def test_scaler_policy_matches_reference():
    rng = np.random.default_rng(1)
    for _ in range(10):
        ov = (rng.random(300) < 0.05).astype(np.uint8).tolist()
        assert sqf.scaler_run(128.0, 8, 0.03125, 32768.0, ov) == ref.scaler_run(128.0, 8, 0.03125, 32768.0, ov)
    # divergence at the floor
    assert sqf.scaler_run(1.0, 4, 0.25, 4.0, [1, 1, 1]) == ref.scaler_run(1.0, 4, 0.25, 4.0, [1, 1, 1])


def test_schedules_match_reference():
    for step in (1, 2, 399, 400, 401, 4000, 16000, 123457):
        assert sqf.schedule_lr("inverse_sqrt", step, 5e-4, 4000, 0.0) == ref.inverse_sqrt(5e-4, 4000, 0.0, step)
        assert sqf.schedule_lr("inverse_sqrt", step, 1e-3, 0, 1e-7) == ref.inverse_sqrt(1e-3, 0, 1e-7, step)
        assert sqf.schedule_lr("cosine_restart", step, 1e-3, 0, 0.0, 1e-5, 1000, 2.0) == \
               ref.cosine_restart(1e-3, 1e-5, 1000, 2.0, step)
        assert sqf.schedule_lr("fixed", step, 3e-4) == 3e-4
    with pytest.raises(sqf.NativeError):
        sqf.schedule_lr("inverse_sqrt", 0)


def test_quantize_fp16_matches_reference():
    rng = np.random.default_rng(2)
    xs = np.concatenate([rng.standard_normal(2000) * 10.0 ** rng.integers(-9, 6, 2000),
                         [65519.0, 65520.0, 2.0 ** -25, -2.0 ** -25, 6e-8, 0.1, 1 / 3]]).astype(np.float32)
    for x in xs:
        a, b = sqf.quantize_fp16(float(x)), ref.quantize_fp16(float(x))
        assert (math.isnan(a) and math.isnan(b)) or np.float32(a).view(np.uint32) == np.float32(b).view(np.uint32)


def test_registry_errors_surface_as_reference_classes():
    with pytest.raises(sqf.NativeError) as e:
        sqf.model_init("no_such_arch", {})
    assert e.value.kind == "RegistryError"
    with pytest.raises(sqf.NativeError) as e:
        sqf.model_init("tiny_transformer", {"src_vocab": 10, "tgt_vocab": 10, "heads": 3})
    assert e.value.kind == "RegistryError" and "d_model must be a positive multiple" in str(e.value)
    with pytest.raises(sqf.NativeError) as e:
        sqf.model_init("tiny_transformer", {"nonexistent_key": 1})
    assert e.value.kind == "ConfigError"


def test_oracle_side_corpus_equals_product_corpus():
    """The bench's CPU reference arm builds its corpus from the oracle
    (reference RngStream) without loading the product library: it must be the
    product's synthetic corpus, id for id."""
    for npairs, sv, tv, s in ((500, 1000, 1000, 1.1), (300, 32768, 32768, 1.1), (50, 10000, 8000, 0.0)):
        a = sqf.synthetic_corpus(npairs, sv, tv, s, 1)
        b = ref.synthetic_corpus(npairs, sv, tv, s, 1)
        for f in ("src_len", "tgt_len", "src_ids", "tgt_ids"):
            assert np.array_equal(getattr(a, f), getattr(b, f)), f
