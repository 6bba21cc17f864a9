"""Checkpoints in the reference's SQFG v2 container (docs/checkpoint_format.md,
checkpoint.cpp:87-391; the reference's own tests test_checkpoint.cpp:98-174).

CPU: a checkpoint written by the reference itself parses with our reader
(magic, table, FNV-1a checksums, meta, canonical-order payloads) and a
corrupted byte is rejected. GPU: save -> load resumes training bitwise; the
reference's checkpoint restores into the B200 trainer and training continues
within the fp32 tolerance; our file parses with the reference's reader."""
import numpy as np
import pytest

import paper_1904_01038_b200 as sqf
from oracle import ref

V = 1000
OV = {"max_tokens": 512, "seed": 1, "lr": 2e-3, "warmup": 20, "max_epochs": 50,
      "criterion": "label_smoothed_cross_entropy", "label_smoothing": 0.1}


def corpus():
    return sqf.synthetic_corpus(120, V, V, 1.1, 1)


def test_reference_checkpoint_parses_with_our_reader(tmp_path):
    if not ref.available():
        pytest.skip("oracle not built")
    c = corpus()
    rt = ref.RefTrainer("transformer_base_defaults", dict(OV, fp16=True), c, V, V)
    for _ in range(2):
        rt.train_one()
    path = tmp_path / "ref.ckpt"
    rt.save(path)
    version, meta, params, opt = sqf.read_checkpoint(path)
    assert version == 2
    assert np.array_equal(params, rt.params())
    m, v, t = rt.adam_state()
    assert np.array_equal(opt, np.concatenate([m, v]))
    assert int(meta["opt.step_count"]) == t == 2
    assert int(meta["progress.step"]) == 2 and meta["loss_scaler.window"] == "256"
    assert meta["config.arch"] == "transformer_base_defaults" and meta["origin.fp16"] == "user"
    # a flipped payload byte fails its section checksum
    raw = bytearray(path.read_bytes())
    raw[-5] ^= 0x40
    bad = tmp_path / "bad.ckpt"
    bad.write_bytes(bytes(raw))
    with pytest.raises(Exception, match="checksum"):
        sqf.read_checkpoint(bad)


@pytest.mark.gpu
def test_save_load_resumes_bitwise(tmp_path):
    c = corpus()
    a = sqf.Trainer("transformer_base_defaults", dict(OV, fp16=True), corpus=c, src_vocab=V, tgt_vocab=V)
    for _ in range(3):
        a.train_one()
    path = tmp_path / "b200.ckpt"
    a.save(path)
    b = sqf.Trainer("transformer_base_defaults", dict(OV, fp16=True), corpus=c, src_vocab=V, tgt_vocab=V)
    assert b.load(path) == 2
    assert np.array_equal(a.params(), b.params()) and a.progress() == b.progress() and a.scaler() == b.scaler()
    for _ in range(3):
        assert a.train_one() == b.train_one()
    assert np.array_equal(a.params(), b.params())
    ma, va, ta = a.adam_state()
    mb, vb, tb = b.adam_state()
    assert np.array_equal(ma, mb) and np.array_equal(va, vb) and ta == tb
    # the file also parses with the reference's own reader
    if ref.available():
        ver, params, opt = ref.checkpoint_read(path)
        a2 = sqf.Trainer("transformer_base_defaults", dict(OV, fp16=True), corpus=c, src_vocab=V, tgt_vocab=V)
        a2.load(path)
        assert ver == 2 and np.array_equal(params, a2.params())
        assert ref.checkpoint_meta(path, "progress.step") == "3"


@pytest.mark.gpu
def test_reference_checkpoint_restores_into_b200_trainer(tmp_path):
    if not ref.available():
        pytest.skip("oracle not built")
    c = corpus()
    rt = ref.RefTrainer("transformer_base_defaults", OV, c, V, V)
    for _ in range(3):
        rt.train_one()
    path = tmp_path / "ref.ckpt"
    rt.save(path)
    mine = sqf.Trainer("transformer_base_defaults", OV, corpus=c, src_vocab=V, tgt_vocab=V)
    mine.load(path)
    assert np.array_equal(mine.params(), rt.params())
    assert mine.progress()["step"] == 3
    for _ in range(3):
        a, b = mine.train_one(), rt.train_one()
        assert a["ntokens"] == b["ntokens"] and a["step"] == b["step"]
        assert abs(a["loss"] - b["loss"]) <= 1e-4 * abs(b["loss"])
    p, q = mine.params(), rt.params()
    assert float(np.max(np.abs(p - q) / np.maximum(1.0, np.abs(p)))) < 1e-4
