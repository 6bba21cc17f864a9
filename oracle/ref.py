"""TEST INFRASTRUCTURE ONLY — the parity oracle.

ctypes binding of ``oracle/_ref/libseqforge_ref.so``: the unmodified C++
reference (seqforge, /root/reference/proj) compiled from its own sources by
``oracle/Makefile`` plus the marshalling shim ``oracle/ref_capi.cpp``. Only
tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline leg may import
this module; the product path never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_ref", "libseqforge_ref.so")
REFERENCE = "/root/reference/proj"


def build(force: bool = False) -> bool:
    """Compile the reference sources (only possible where /root/reference exists)."""
    if os.path.exists(LIB) and not force:
        return True
    if not os.path.isdir(REFERENCE):
        return os.path.exists(LIB)
    subprocess.run(["make", "-C", HERE, "-j8"], check=True, capture_output=True)
    return os.path.exists(LIB)


def available() -> bool:
    return os.path.exists(LIB)


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not available():
            build()
        _lib = C.CDLL(LIB)
        _declare(_lib)
    return _lib


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p)


vp, i32, i64, u64, f32, f64, cp = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_float, C.c_double, C.c_char_p
P = C.POINTER


class StatsC(C.Structure):
    _fields_ = [("step", i64), ("loss", f64), ("nll", f64), ("ntokens", i64), ("ncorrect", i64), ("lr", f64),
                ("skipped", i32), ("_pad", i32), ("scale", f64)]

    def as_dict(self):
        return {"step": self.step, "loss": self.loss, "nll": self.nll, "ntokens": self.ntokens,
                "ncorrect": self.ncorrect, "lr": self.lr, "skipped": bool(self.skipped), "scale": self.scale}


def _declare(L):
    def s(name, res, *args):
        f = getattr(L, name)
        f.restype = res
        f.argtypes = list(args)
    s("sqfref_last_error", cp)
    s("sqfref_quantize_fp16", f32, f32)
    s("sqfref_f32_to_f16_bits", C.c_uint16, f32)
    s("sqfref_quantize_many", None, vp, i64)
    for n in ("sqfref_rng_u64", "sqfref_rng_double", "sqfref_rng_normal"):
        s(n, None, u64, u64, u64, C.c_int, vp)
    s("sqfref_rng_below", None, u64, u64, u64, u64, C.c_int, vp)
    s("sqfref_positional_row", None, C.c_int, C.c_int, vp)
    s("sqfref_corpus_create", vp, C.c_int, vp, vp, vp, vp)
    s("sqfref_synthetic_corpus", C.c_int, C.c_int, C.c_int, C.c_int, f64, u64, u64, vp, vp, vp, vp, vp, vp)
    s("sqfref_corpus_free", None, vp)
    s("sqfref_make_batches", C.c_int, vp, i64, C.c_int, u64, P(i32), vp, vp)
    s("sqfref_shuffle_epoch", C.c_int, C.c_int, u64, C.c_int, vp)
    s("sqfref_make_minibatch", C.c_int, vp, vp, C.c_int, vp, vp, vp, vp, vp, vp, P(i64))
    s("sqfref_bucket_gradients", C.c_int, vp, C.c_int, i64, P(i32), vp, vp)
    s("sqfref_inverse_sqrt", C.c_int, f64, i64, f64, i64, P(f64))
    s("sqfref_cosine_restart", C.c_int, f64, f64, i64, f64, i64, P(f64))
    s("sqfref_adam", C.c_int, vp, vp, i64, vp, vp, i64, f64, f64, f64, f64)
    s("sqfref_scaler_run", C.c_int, f64, i64, f64, f64, vp, C.c_int, vp, P(i32))
    s("sqfref_xent", C.c_int, vp, C.c_int, C.c_int, vp, vp, f32, C.c_int, f32, vp, vp, vp, vp)
    s("sqfref_layer_norm", C.c_int, vp, C.c_int, C.c_int, vp, vp, C.c_int, vp, vp, vp, vp, vp)
    s("sqfref_attention", C.c_int, vp, C.c_int, vp, vp, C.c_int, C.c_int, C.c_int, vp, vp, C.c_int, vp, vp, vp,
      vp, vp)
    s("sqfref_linear", C.c_int, vp, C.c_int, C.c_int, vp, vp, C.c_int, C.c_int, vp, vp, vp, vp, vp)
    s("sqfref_trainer_create", vp, cp, P(cp), P(cp), C.c_int, vp, C.c_int, C.c_int)
    s("sqfref_trainer_free", None, vp)
    s("sqfref_trainer_set_injector", C.c_int, vp, vp, C.c_int)
    s("sqfref_trainer_train_one", C.c_int, vp, P(StatsC))
    s("sqfref_trainer_train_step", C.c_int, vp, vp, vp, vp, C.c_int, C.c_int, P(StatsC))
    s("sqfref_trainer_num_params", i64, vp)
    s("sqfref_trainer_params", C.c_int, vp, vp)
    s("sqfref_trainer_set_params", C.c_int, vp, vp)
    s("sqfref_trainer_manifest_size", C.c_int, vp)
    s("sqfref_trainer_manifest_entry", C.c_int, vp, C.c_int, cp, C.c_int, P(i64), P(i64))
    s("sqfref_trainer_adam_state", C.c_int, vp, vp, vp, P(i64))
    s("sqfref_trainer_scaler", C.c_int, vp, P(f64), P(i64))
    s("sqfref_trainer_progress", C.c_int, vp, P(i64), P(i32), P(i32), P(i32))
    s("sqfref_trainer_buckets", C.c_int, vp, P(i32), vp, vp)
    s("sqfref_trainer_subbatch_grad", C.c_int, vp, vp, vp, C.c_int, f32, vp, P(StatsC))
    s("sqfref_trainer_evaluate", C.c_int, vp, vp, P(f64), P(f64), P(i64), P(i64))
    s("sqfref_trainer_save", C.c_int, vp, cp)
    s("sqfref_generate", C.c_int, vp, C.c_int, vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, f64,
      f64, f64, C.c_uint64, vp, C.c_int, P(vp))
    s("sqfref_gen_count", C.c_int, vp, C.c_int)
    s("sqfref_gen_hyp", C.c_int, vp, C.c_int, C.c_int, vp, vp, C.c_int, P(i32), P(f64), P(f64), P(i32), P(i32))
    s("sqfref_gen_free", None, vp)
    s("sqfref_sample_from_topk", C.c_int, vp, C.c_int, C.c_int, f64, f64, P(i32))
    s("sqfref_batch_for_inference", C.c_int, vp, C.c_int, i64, P(i32), vp, vp)
    s("sqfref_simulate_timeline", C.c_int, C.c_int, C.c_int, C.c_int, vp, vp, C.c_int, vp, C.c_int)
    s("sqfref_checkpoint_read", C.c_int, cp, P(i32), P(i64), vp, P(i64), vp)
    s("sqfref_checkpoint_meta", C.c_int, cp, cp, vp, C.c_int)


class RefError(RuntimeError):
    pass


def _ck(status):
    if status < 0:
        raise RefError(f"reference error {status}: {lib().sqfref_last_error().decode()}")
    return status


class OracleCorpus:
    """A corpus with the product Corpus's fields (src_len, tgt_len, src_ids,
    tgt_ids, npairs), generated without the product library."""

    def __init__(self, sl, tl, si, ti):
        self.src_len, self.tgt_len, self.src_ids, self.tgt_ids = sl, tl, si, ti
        self.npairs = len(sl)


def synthetic_corpus(npairs, src_vocab, tgt_vocab, zipf_s=1.1, seed=1, stream=4242):
    """SURVEY §8(d) generator on the reference's RngStream (ref_capi.cpp); equal
    to paper_1904_01038_b200.synthetic_corpus (tests/test_boundary.py)."""
    sl, tl = np.zeros(npairs, np.int32), np.zeros(npairs, np.int32)
    st, tt = C.c_int64(), C.c_int64()
    _ck(lib().sqfref_synthetic_corpus(npairs, src_vocab, tgt_vocab, zipf_s, seed, stream, _ptr(sl), _ptr(tl), None,
                                      None, C.byref(st), C.byref(tt)))
    si, ti = np.zeros(max(st.value, 1), np.int32), np.zeros(max(tt.value, 1), np.int32)
    _ck(lib().sqfref_synthetic_corpus(npairs, src_vocab, tgt_vocab, zipf_s, seed, stream, _ptr(sl), _ptr(tl),
                                      _ptr(si), _ptr(ti), C.byref(st), C.byref(tt)))
    return OracleCorpus(sl, tl, si[:st.value], ti[:tt.value])


class RefCorpus:
    """Owns a reference-side copy of a corpus (paper_1904_01038_b200.Corpus-like)."""

    def __init__(self, corpus):
        self.c = corpus
        self.h = lib().sqfref_corpus_create(corpus.npairs, _ptr(corpus.src_len), _ptr(corpus.tgt_len),
                                            _ptr(corpus.src_ids), _ptr(corpus.tgt_ids))

    def __del__(self):
        if getattr(self, "h", None):
            lib().sqfref_corpus_free(self.h)
            self.h = None


# ---------------------------------------------------------------- numerics
def quantize_fp16(x: float) -> float:
    return float(lib().sqfref_quantize_fp16(x))


def quantize_array(a: np.ndarray) -> np.ndarray:
    out = np.ascontiguousarray(a, np.float32).copy()
    lib().sqfref_quantize_many(_ptr(out), out.size)
    return out


def rng_u64(seed, stream, counter, n):
    out = np.zeros(n, np.uint64)
    lib().sqfref_rng_u64(seed, stream, counter, n, _ptr(out))
    return out


def rng_double(seed, stream, counter, n):
    out = np.zeros(n, np.float64)
    lib().sqfref_rng_double(seed, stream, counter, n, _ptr(out))
    return out


def rng_normal(seed, stream, counter, n):
    out = np.zeros(n, np.float64)
    lib().sqfref_rng_normal(seed, stream, counter, n, _ptr(out))
    return out


def rng_below(seed, stream, counter, bound, n):
    out = np.zeros(n, np.uint64)
    lib().sqfref_rng_below(seed, stream, counter, bound, n, _ptr(out))
    return out


def positional_row(pos, d):
    out = np.zeros(d, np.float32)
    lib().sqfref_positional_row(pos, d, _ptr(out))
    return out


# ---------------------------------------------------------------- data
def make_batches(corpus, max_tokens, max_sentences=0, seed=1):
    rc = RefCorpus(corpus)
    n = C.c_int32()
    sizes = np.zeros(max(1, corpus.npairs), np.int32)
    members = np.zeros(max(1, corpus.npairs), np.int32)
    _ck(lib().sqfref_make_batches(rc.h, max_tokens, max_sentences, seed, C.byref(n), _ptr(sizes), _ptr(members)))
    out, k = [], 0
    for b in range(n.value):
        out.append(members[k:k + sizes[b]].tolist())
        k += sizes[b]
    return out


def shuffle_epoch(nbatches, seed, epoch):
    o = np.zeros(max(1, nbatches), np.int32)
    _ck(lib().sqfref_shuffle_epoch(nbatches, seed, epoch, _ptr(o)))
    return o[:nbatches].tolist()


def make_minibatch(corpus, members):
    rc = RefCorpus(corpus)
    m = np.asarray(members, np.int32)
    maxw = int(max(corpus.src_len.max(), corpus.tgt_len.max()))
    cap = max(1, len(m) * maxw)
    dims = np.zeros(3, np.int32)
    src, tin, tout = (np.zeros(cap, np.int32) for _ in range(3))
    sl, tl = np.zeros(max(1, len(m)), np.int32), np.zeros(max(1, len(m)), np.int32)
    nt = C.c_int64()
    _ck(lib().sqfref_make_minibatch(rc.h, _ptr(m), len(m), _ptr(dims), _ptr(src), _ptr(tin), _ptr(tout), _ptr(sl),
                                    _ptr(tl), C.byref(nt)))
    r, s, t = (int(x) for x in dims)
    return {"rows": r, "src_width": s, "tgt_width": t, "source": src[:r * s].reshape(r, s),
            "target_in": tin[:r * t].reshape(r, t), "target_out": tout[:r * t].reshape(r, t),
            "src_lens": sl[:r].copy(), "tgt_lens": tl[:r].copy(), "ntokens": nt.value}


def bucket_gradients(sizes, threshold):
    s = np.asarray(sizes, np.int64)
    n = C.c_int32()
    st, en = np.zeros(len(s) + 1, np.int64), np.zeros(len(s) + 1, np.int64)
    _ck(lib().sqfref_bucket_gradients(_ptr(s), len(s), threshold, C.byref(n), _ptr(st), _ptr(en)))
    return list(zip(st[:n.value].tolist(), en[:n.value].tolist()))


def inverse_sqrt(base, warmup, init, step):
    o = C.c_double()
    _ck(lib().sqfref_inverse_sqrt(base, warmup, init, step, C.byref(o)))
    return o.value


def cosine_restart(base, eta_min, period, t_mult, step):
    o = C.c_double()
    _ck(lib().sqfref_cosine_restart(base, eta_min, period, t_mult, step, C.byref(o)))
    return o.value


def adam(params, grads, m, v, t, lr, b1=0.9, b2=0.98, eps=1e-8):
    p = np.ascontiguousarray(params, np.float32).copy()
    g = np.ascontiguousarray(grads, np.float32)
    mm = np.ascontiguousarray(m, np.float32).copy()
    vv = np.ascontiguousarray(v, np.float32).copy()
    _ck(lib().sqfref_adam(_ptr(p), _ptr(g), p.size, _ptr(mm), _ptr(vv), t, lr, b1, b2, eps))
    return p, mm, vv


def scaler_run(init, window, mn, mx, overflow):
    ov = np.asarray(overflow, np.uint8)
    sc = np.zeros(max(1, len(ov)), np.float64)
    d = C.c_int32()
    _ck(lib().sqfref_scaler_run(init, window, mn, mx, _ptr(ov), len(ov), _ptr(sc), C.byref(d)))
    return sc[:len(ov)].tolist(), d.value


# ---------------------------------------------------------------- tape ops
def xent(logits, gold, eps, fp16=False, seed=1.0, pad=1):
    lg = np.ascontiguousarray(logits, np.float32)
    r, v = lg.shape
    gold = np.ascontiguousarray(gold, np.int32)
    active = (gold != pad).astype(np.uint8)
    loss, nll = np.zeros(r, np.float32), np.zeros(r, np.float32)
    corr = np.zeros(r, np.uint8)
    dl = np.zeros((r, v), np.float32)
    _ck(lib().sqfref_xent(_ptr(lg), r, v, _ptr(gold), _ptr(active), eps, int(fp16), seed, _ptr(loss), _ptr(nll),
                          _ptr(corr), _ptr(dl)))
    return loss, nll, corr, dl


def layer_norm(x, gamma, beta, dy=None, fp16=False):
    x = np.ascontiguousarray(x, np.float32)
    r, d = x.shape
    y = np.zeros_like(x)
    dx, dg, db = np.zeros_like(x), np.zeros(d, np.float32), np.zeros(d, np.float32)
    dyp = _ptr(np.ascontiguousarray(dy, np.float32)) if dy is not None else None
    dyk = np.ascontiguousarray(dy, np.float32) if dy is not None else None
    _ck(lib().sqfref_layer_norm(_ptr(x), r, d, _ptr(np.ascontiguousarray(gamma, np.float32)),
                                _ptr(np.ascontiguousarray(beta, np.float32)), int(fp16),
                                _ptr(dyk) if dyk is not None else None, _ptr(y), _ptr(dx), _ptr(dg), _ptr(db)))
    del dyp
    return y, dx, dg, db


def attention(q, k, v, heads, key_base, key_len, dout=None, fp16=False):
    q, k, v = (np.ascontiguousarray(a, np.float32) for a in (q, k, v))
    rq, d = q.shape
    rk = k.shape[0]
    out = np.zeros_like(q)
    dq, dk, dv = np.zeros_like(q), np.zeros_like(k), np.zeros_like(v)
    kb = np.ascontiguousarray(key_base, np.int32)
    kl = np.ascontiguousarray(key_len, np.int32)
    do = np.ascontiguousarray(dout, np.float32) if dout is not None else None
    _ck(lib().sqfref_attention(_ptr(q), rq, _ptr(k), _ptr(v), rk, d, heads, _ptr(kb), _ptr(kl), int(fp16),
                               _ptr(do) if do is not None else None, _ptr(out), _ptr(dq), _ptr(dk), _ptr(dv)))
    return out, dq, dk, dv


def linear(x, w, b=None, dy=None, fp16=False):
    x = np.ascontiguousarray(x, np.float32)
    w = np.ascontiguousarray(w, np.float32)
    r, k = x.shape
    o = w.shape[0]
    y, dx, dw = np.zeros((r, o), np.float32), np.zeros_like(x), np.zeros_like(w)
    db = np.zeros(o, np.float32)
    bb = np.ascontiguousarray(b, np.float32) if b is not None else None
    dd = np.ascontiguousarray(dy, np.float32) if dy is not None else None
    _ck(lib().sqfref_linear(_ptr(x), r, k, _ptr(w), _ptr(bb) if bb is not None else None, o, int(fp16),
                            _ptr(dd) if dd is not None else None, _ptr(y), _ptr(dx), _ptr(dw), _ptr(db)))
    return y, dx, dw, db


# ---------------------------------------------------------------- trainer
def _kv(overrides):
    keys = [str(k) for k in overrides]
    vals = [str(v).lower() if isinstance(v, bool) else str(v) for v in overrides.values()]
    ka = (cp * max(1, len(keys)))(*[k.encode() for k in keys])
    va = (cp * max(1, len(vals)))(*[v.encode() for v in vals])
    return ka, va, len(keys)


def simulate_timeline(workers, accum, mode, compute, buckets):
    """The reference's simulate_timeline + format_report (simulator.cpp) on a
    scenario given as values; returns the report text."""
    modes = {"serial_sync": 0, "overlap": 1, "overlap_accum": 2}
    c = np.ascontiguousarray(np.asarray(compute, np.float64).reshape(workers, accum))
    b = np.ascontiguousarray(np.asarray(buckets, np.float64))
    buf = C.create_string_buffer(1 << 16)
    _ck(lib().sqfref_simulate_timeline(workers, accum, modes[mode], _ptr(c), _ptr(b), len(b), buf, 1 << 16))
    return buf.value.decode()


def checkpoint_read(path):
    """The reference's read_checkpoint (checkpoint.cpp:226-320): (version, params, opt)."""
    L = lib()
    v, npar, nopt = C.c_int32(), C.c_int64(), C.c_int64()
    p = str(path).encode()
    _ck(L.sqfref_checkpoint_read(p, C.byref(v), C.byref(npar), None, C.byref(nopt), None))
    params = np.zeros(npar.value, np.float32)
    opt = np.zeros(max(1, nopt.value), np.float32)
    _ck(L.sqfref_checkpoint_read(p, C.byref(v), C.byref(npar), _ptr(params), C.byref(nopt), _ptr(opt)))
    return int(v.value), params, opt[:nopt.value]


def checkpoint_meta(path, key):
    buf = C.create_string_buffer(4096)
    _ck(lib().sqfref_checkpoint_meta(str(path).encode(), key.encode(), buf, 4096))
    return buf.value.decode()


class RefTrainer:
    """The reference's own Trainer over an in-memory corpus (trainer.hpp:84-85)."""

    def __init__(self, arch, overrides, corpus, src_vocab, tgt_vocab):
        self.corpus = RefCorpus(corpus)
        k, v, n = _kv(overrides)
        self.h = lib().sqfref_trainer_create(arch.encode(), k, v, n, self.corpus.h, src_vocab, tgt_vocab)
        if not self.h:
            raise RefError(lib().sqfref_last_error().decode())
        self.workers = int(overrides.get("workers", 1))
        self.accum = int(overrides.get("accum", 1))

    def __del__(self):
        if getattr(self, "h", None):
            lib().sqfref_trainer_free(self.h)
            self.h = None

    def train_one(self):
        st = StatsC()
        r = _ck(lib().sqfref_trainer_train_one(self.h, C.byref(st)))
        return None if r == 1 else st.as_dict()

    def train_step(self, sub):
        counts = np.array([len(m) for row in sub for m in row], np.int32)
        members = np.array([x for row in sub for m in row for x in m] or [0], np.int32)
        st = StatsC()
        _ck(lib().sqfref_trainer_train_step(self.h, self.corpus.h, _ptr(members), _ptr(counts), len(sub),
                                            len(sub[0]), C.byref(st)))
        return st.as_dict()

    def generate(self, sources, mode="beam", stream_ids=None, no_cache=False, beam=4, max_len=0,
                 diverse_groups=1, topk=1, lenpen=0.6, diverse_strength=0.5, temperature=1.0, seed=1):
        """The reference's beam_search / diverse_beam_search / top_k_sample
        (generate.hpp:46-90) on this trainer's model (fp32)."""
        src, lens = _pad_rows(sources)
        ids = None if stream_ids is None else np.ascontiguousarray(stream_ids, np.uint64)
        h = C.c_void_p()
        _ck(lib().sqfref_generate(self.h, {"beam": 0, "diverse": 1, "sample": 2}[mode], _ptr(src), _ptr(lens),
                                  len(lens), src.shape[1], beam, max_len, diverse_groups, topk, lenpen,
                                  diverse_strength, temperature, seed, None if ids is None else _ptr(ids),
                                  int(no_cache), C.byref(h)))
        try:
            return [[_read_hyp(lib().sqfref_gen_hyp, h, s, k) for k in range(lib().sqfref_gen_count(h, s))]
                    for s in range(len(lens))]
        finally:
            lib().sqfref_gen_free(h)

    def set_injector(self, steps):
        a = np.asarray(list(steps) or [0], np.int64)
        _ck(lib().sqfref_trainer_set_injector(self.h, _ptr(a), len(list(steps))))

    @property
    def num_params(self):
        return int(lib().sqfref_trainer_num_params(self.h))

    def params(self):
        out = np.zeros(self.num_params, np.float32)
        _ck(lib().sqfref_trainer_params(self.h, _ptr(out)))
        return out

    def set_params(self, p):
        p = np.ascontiguousarray(p, np.float32)
        _ck(lib().sqfref_trainer_set_params(self.h, _ptr(p)))

    def manifest(self):
        out, buf = [], C.create_string_buffer(256)
        for i in range(lib().sqfref_trainer_manifest_size(self.h)):
            off, num = C.c_int64(), C.c_int64()
            _ck(lib().sqfref_trainer_manifest_entry(self.h, i, buf, 256, C.byref(off), C.byref(num)))
            out.append((buf.value.decode(), off.value, num.value))
        return out

    def adam_state(self):
        m, v = np.zeros(self.num_params, np.float32), np.zeros(self.num_params, np.float32)
        t = C.c_int64()
        _ck(lib().sqfref_trainer_adam_state(self.h, _ptr(m), _ptr(v), C.byref(t)))
        return m, v, t.value

    def scaler(self):
        s, g = C.c_double(), C.c_int64()
        _ck(lib().sqfref_trainer_scaler(self.h, C.byref(s), C.byref(g)))
        return s.value, g.value

    def progress(self):
        s, e, c, n = C.c_int64(), C.c_int32(), C.c_int32(), C.c_int32()
        _ck(lib().sqfref_trainer_progress(self.h, C.byref(s), C.byref(e), C.byref(c), C.byref(n)))
        return {"step": s.value, "epoch": e.value, "cursor": c.value, "batches_per_epoch": n.value}

    def subbatch_grad(self, members, seed=1.0):
        """Gradient of one sub-batch on the (shadow of the) master (trainer.cpp:223-240)."""
        m = np.asarray(members, np.int32)
        g = np.zeros(self.num_params, np.float32)
        st = StatsC()
        _ck(lib().sqfref_trainer_subbatch_grad(self.h, self.corpus.h, _ptr(m), len(m), seed, _ptr(g), C.byref(st)))
        return g, st.as_dict()

    def save(self, path):
        """The reference's save_checkpoint (checkpoint.cpp:187-224)."""
        _ck(lib().sqfref_trainer_save(self.h, str(path).encode()))

    def evaluate(self, corpus):
        rc = RefCorpus(corpus)
        loss, nll, nt, nc = C.c_double(), C.c_double(), C.c_int64(), C.c_int64()
        _ck(lib().sqfref_trainer_evaluate(self.h, rc.h, C.byref(loss), C.byref(nll), C.byref(nt), C.byref(nc)))
        return {"loss": loss.value, "nll": nll.value, "ntokens": nt.value, "ncorrect": nc.value}


def sample_from_topk(logits, k, temperature, u):
    x = np.ascontiguousarray(logits, np.float32)
    out = C.c_int32()
    _ck(lib().sqfref_sample_from_topk(_ptr(x), len(x), k, temperature, u, C.byref(out)))
    return out.value


def batch_for_inference(lengths, max_tokens):
    lens = np.ascontiguousarray(lengths, np.int32)
    n = len(lens)
    sizes, members = np.zeros(max(n, 1), np.int32), np.zeros(max(n, 1), np.int32)
    ng = C.c_int32()
    _ck(lib().sqfref_batch_for_inference(_ptr(lens), n, max_tokens, C.byref(ng), _ptr(sizes), _ptr(members)))
    out, at = [], 0
    for i in range(ng.value):
        out.append(members[at:at + sizes[i]].tolist())
        at += sizes[i]
    return out


def _pad_rows(sources):
    lens = np.array([len(r) for r in sources], np.int32)
    src = np.full((len(lens), max(1, int(lens.max()) if len(lens) else 1)), 1, np.int32)
    for i, r in enumerate(sources):
        src[i, :len(r)] = r
    return src, lens


def _read_hyp(fn, h, s, k, cap=4096):
    tok, sc = np.zeros(cap, np.int32), np.zeros(cap, np.float32)
    n, cum, score, fs, fin = C.c_int32(), C.c_double(), C.c_double(), C.c_int32(), C.c_int32()
    _ck(fn(h, s, k, _ptr(tok), _ptr(sc), cap, C.byref(n), C.byref(cum), C.byref(score), C.byref(fs), C.byref(fin)))
    return {"tokens": tok[:n.value].tolist(), "step_scores": sc[:n.value].tolist(), "cum_logprob": cum.value,
            "score": score.value, "finish_step": fs.value, "finished": bool(fin.value)}
