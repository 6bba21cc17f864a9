"""Oracle parity for the headline architectures (BASELINE.json configs C3 and
C4), through the whole training step at the real widths -- d=512/1024,
8/16 heads of 64, ffn 2048/4096, 6+6 layers, V=32,768 -- at a budget the
single-threaded reference finishes in seconds (two short sentences per step):

  * fp32: one sub-batch's gradient within 1e-4 (|a-b|/max(1,|a|),
    test_trainer.cpp:69-78) of the reference's Tape gradient;
  * fp16: two optimizer steps with loss within 1e-2 and identical skip
    decisions, then the masters within 1e-2 (L2) of the reference's.

Architectures are registered over the reference's pre-norm `transformer`
(registry.cpp:76-110, model.cpp:199-275)."""
import numpy as np
import pytest

from oracle import ref

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

V = 32768
BASE = {"criterion": "label_smoothed_cross_entropy", "label_smoothing": 0.1, "lr": 2e-3, "warmup": 20, "seed": 1,
        "max_tokens": 64}
ARCHS = ["transformer_wmt_en_de", "transformer_vaswani_wmt_en_de_big"]


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(1.0, np.abs(a))))


def short_members(c, n, cap):
    out = []
    for i in range(c.npairs):
        s, t = c.pair(i)
        if len(s) <= cap and len(t) <= cap:
            out.append(i)
        if len(out) == n:
            return out
    raise AssertionError("corpus has too few short pairs")


@pytest.fixture(scope="module")
def corpus():
    import paper_1904_01038_b200 as sqf
    return sqf.synthetic_corpus(400, V, V, 1.1, 1)


def make(arch, ov, c):
    import paper_1904_01038_b200 as sqf
    o = dict(BASE, **ov)
    return (sqf.Trainer(arch, o, corpus=c, src_vocab=V, tgt_vocab=V), ref.RefTrainer(arch, o, c, V, V))


@pytest.mark.parametrize("arch", ARCHS)
def test_headline_fp32_gradient_matches_reference(arch, corpus):
    mine, theirs = make(arch, {"optimizer": "sgd", "scheduler": "fixed", "lr": 1e-9}, corpus)
    assert len(mine.params()) == len(theirs.params())
    members = short_members(corpus, 2, 12)
    g_ref, st = theirs.subbatch_grad(members)
    s = mine.train_step([[members]])
    assert s["ntokens"] == st["ntokens"]
    assert abs(s["loss"] - st["loss"]) <= 1e-4 * abs(st["loss"]), (s, st)
    g = mine.last_grads()
    assert np.abs(g_ref).max() > 1e-3
    assert rel(g, g_ref) < 1e-4


@pytest.mark.parametrize("arch", ARCHS)
def test_headline_fp16_steps_track_reference(arch, corpus):
    mine, theirs = make(arch, {"fp16": True}, corpus)
    members = short_members(corpus, 4, 12)
    for step in range(2):
        sub = [[members[2 * step:2 * step + 2]]]
        a, b = mine.train_step(sub), theirs.train_step(sub)
        assert a["ntokens"] == b["ntokens"] and a["skipped"] == b["skipped"] and a["scale"] == b["scale"], (a, b)
        assert abs(a["loss"] - b["loss"]) <= 1e-2 * abs(b["loss"]), (step, a, b)
    p, q = mine.params(), theirs.params()
    assert np.linalg.norm(p - q) <= 1e-2 * np.linalg.norm(q)
