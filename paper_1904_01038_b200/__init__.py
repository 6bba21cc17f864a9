"""B200-native mixed-precision data-parallel Transformer training step.

Python face of the C-ABI library (include/sqf_trainer.h, include/sqf_kernels.h).
It mirrors the seqforge reference's Trainer surface (trainer.hpp:80-125): same
config keys, registry names, StepStats, train_one / train_step / evaluate,
overflow injector, scaler, progress. All compute runs in the native library's
sm_100a kernels; nothing here computes.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import _lib as L

__all__ = ["Corpus", "Trainer", "synthetic_corpus", "make_batches", "shuffle_epoch", "make_minibatch",
           "split_counts", "bucket_gradients", "model_init", "scaler_run", "schedule_lr", "quantize_fp16",
           "nccl_unique_id", "NativeError", "BOS", "PAD", "EOS", "UNK"]

BOS, PAD, EOS, UNK = 0, 1, 2, 3
NativeError = L.NativeError


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


@dataclass
class Corpus:
    """Eos-terminated id sequences, concatenated (SequencePair list, data.hpp:50-54)."""
    src_len: np.ndarray
    tgt_len: np.ndarray
    src_ids: np.ndarray
    tgt_ids: np.ndarray

    @property
    def npairs(self) -> int:
        return int(self.src_len.shape[0])

    @classmethod
    def from_pairs(cls, pairs):
        sl = np.array([len(s) for s, _ in pairs], np.int32)
        tl = np.array([len(t) for _, t in pairs], np.int32)
        si = np.array([x for s, _ in pairs for x in s], np.int32)
        ti = np.array([x for _, t in pairs for x in t], np.int32)
        return cls(sl, tl, si, ti)

    def pair(self, i: int):
        so = int(self.src_len[:i].sum())
        to = int(self.tgt_len[:i].sum())
        return (self.src_ids[so:so + self.src_len[i]].tolist(), self.tgt_ids[to:to + self.tgt_len[i]].tolist())

    def handle(self):
        return L.sqf_corpus_create(self.npairs, _ptr(self.src_len), _ptr(self.tgt_len), _ptr(self.src_ids),
                                   _ptr(self.tgt_ids))


def synthetic_corpus(npairs: int, src_vocab: int, tgt_vocab: int, zipf_s: float = 1.1, seed: int = 1) -> Corpus:
    """SURVEY §8(d) generator: lengths clamp(round(exp(3.1+0.6z)),1,200), ids Zipf(s) over [4, V)."""
    sl = np.zeros(npairs, np.int32)
    tl = np.zeros(npairs, np.int32)
    st, tt = C.c_int64(), C.c_int64()
    L.check(L.sqf_synthetic_corpus(npairs, src_vocab, tgt_vocab, zipf_s, seed, _ptr(sl), _ptr(tl), None, None,
                                   C.byref(st), C.byref(tt)))
    si = np.zeros(st.value, np.int32)
    ti = np.zeros(tt.value, np.int32)
    L.check(L.sqf_synthetic_corpus(npairs, src_vocab, tgt_vocab, zipf_s, seed, _ptr(sl), _ptr(tl), _ptr(si), _ptr(ti),
                                   C.byref(st), C.byref(tt)))
    return Corpus(sl, tl, si, ti)


def make_batches(corpus: Corpus, max_tokens: int, max_sentences: int = 0, seed: int = 1):
    h = corpus.handle()
    try:
        n = C.c_int32()
        sizes = np.zeros(max(1, corpus.npairs), np.int32)
        members = np.zeros(max(1, corpus.npairs), np.int32)
        L.check(L.sqf_make_batches(h, max_tokens, max_sentences, seed, C.byref(n), _ptr(sizes), _ptr(members)))
        out, k = [], 0
        for b in range(n.value):
            out.append(members[k:k + sizes[b]].tolist())
            k += sizes[b]
        return out
    finally:
        L.sqf_corpus_free(h)


def shuffle_epoch(nbatches: int, seed: int, epoch: int):
    order = np.zeros(max(1, nbatches), np.int32)
    L.check(L.sqf_shuffle_epoch(nbatches, seed, epoch, _ptr(order)))
    return order[:nbatches].tolist()


def make_minibatch(corpus: Corpus, members):
    h = corpus.handle()
    try:
        m = np.asarray(members, np.int32)
        maxw = int(max(corpus.src_len.max(), corpus.tgt_len.max())) if corpus.npairs else 1
        cap = max(1, len(m) * maxw)
        dims = np.zeros(3, np.int32)
        src, tin, tout = (np.zeros(cap, np.int32) for _ in range(3))
        sl, tl = np.zeros(max(1, len(m)), np.int32), np.zeros(max(1, len(m)), np.int32)
        nt = C.c_int64()
        L.check(L.sqf_make_minibatch(h, _ptr(m), len(m), _ptr(dims), _ptr(src), _ptr(tin), _ptr(tout), _ptr(sl),
                                     _ptr(tl), C.byref(nt)))
        r, s, t = (int(x) for x in dims)
        return {"rows": r, "src_width": s, "tgt_width": t, "source": src[:r * s].reshape(r, s),
                "target_in": tin[:r * t].reshape(r, t), "target_out": tout[:r * t].reshape(r, t),
                "src_lens": sl[:r].copy(), "tgt_lens": tl[:r].copy(), "ntokens": nt.value}
    finally:
        L.sqf_corpus_free(h)


def split_counts(rows: int, workers: int, accum: int):
    c = np.zeros(workers * accum, np.int32)
    L.check(L.sqf_split_counts(rows, workers, accum, _ptr(c)))
    return c.tolist()


def bucket_gradients(sizes, threshold: int):
    s = np.asarray(sizes, np.int64)
    n = C.c_int32()
    st = np.zeros(len(s) + 1, np.int64)
    en = np.zeros(len(s) + 1, np.int64)
    L.check(L.sqf_bucket_gradients(_ptr(s), len(s), threshold, C.byref(n), _ptr(st), _ptr(en)))
    return list(zip(st[:n.value].tolist(), en[:n.value].tolist()))


def _kv(overrides):
    keys = [str(k) for k in overrides]
    vals = [str(v).lower() if isinstance(v, bool) else str(v) for v in overrides.values()]
    return L.cstrs(keys), L.cstrs(vals), len(keys)


def model_init(arch: str, overrides: dict):
    """Initial canonical-order parameters of the model (host, model.cpp:135-150)."""
    k, v, n = _kv(overrides)
    num = C.c_int64()
    ms = C.c_int()
    L.check(L.sqf_model_init(arch.encode(), k, v, n, None, 0, C.byref(num), C.byref(ms)))
    out = np.zeros(num.value, np.float32)
    L.check(L.sqf_model_init(arch.encode(), k, v, n, _ptr(out), num.value, C.byref(num), C.byref(ms)))
    return out


def scaler_run(init, window, mn, mx, overflow):
    ov = np.asarray(overflow, np.uint8)
    sc = np.zeros(max(1, len(ov)), np.float64)
    d = C.c_int32()
    L.check(L.sqf_scaler_run(init, window, mn, mx, _ptr(ov), len(ov), _ptr(sc), C.byref(d)))
    return sc[:len(ov)].tolist(), d.value


def schedule_lr(name, step, lr=5e-4, warmup=400, warmup_init_lr=0.0, eta_min=0.0, period=1000, t_mult=1.0):
    out = C.c_double()
    L.check(L.sqf_schedule_lr(name.encode(), lr, warmup, warmup_init_lr, eta_min, period, t_mult, step,
                              C.byref(out)))
    return out.value


def quantize_fp16(x: float) -> float:
    return float(L.sqf_quantize_fp16(x))


def load_task(arch: str, overrides: dict):
    """The task the config names, made through the registry (e.g. task=translation
    with train_src/train_tgt files): (src_vocab, tgt_vocab, [(source ids, target ids)])."""
    k, v, n = _kv(overrides)
    h = L.sqf_task_create(arch.encode(), k, v, n)
    if not h:
        raise L.NativeError(L.sqf_last_status(), L.sqf_last_error().decode())
    try:
        sv, tv, npairs, ns, nt = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int64(), C.c_int64()
        L.check(L.sqf_task_info(h, C.byref(sv), C.byref(tv), C.byref(npairs), C.byref(ns), C.byref(nt)))
        sl = np.zeros(max(1, npairs.value), np.int32)
        tl = np.zeros(max(1, npairs.value), np.int32)
        si = np.zeros(max(1, ns.value), np.int32)
        ti = np.zeros(max(1, nt.value), np.int32)
        L.check(L.sqf_task_pairs(h, _ptr(sl), _ptr(tl), _ptr(si), _ptr(ti)))
        pairs, a, b = [], 0, 0
        for i in range(npairs.value):
            pairs.append((si[a:a + sl[i]].tolist(), ti[b:b + tl[i]].tolist()))
            a += sl[i]
            b += tl[i]
        return sv.value, tv.value, pairs
    finally:
        L.sqf_task_free(h)


def simulate_timeline(scenario: str) -> dict:
    """Timeline model of a data-parallel step (simulator.cpp): scenario text in,
    {"makespan", "idle": [...], "exposed_comm", "total_compute"} out."""
    buf = C.create_string_buffer(1 << 16)
    L.check(L.sqf_simulate_timeline(scenario.encode(), buf, 1 << 16))
    out = {"idle": []}
    for line in buf.value.decode().splitlines():
        f = line.split()
        if f[0] == "idle":
            out["idle"].append(float(f[2]))
        else:
            out[f[0]] = float(f[1])
    out["text"] = buf.value.decode()
    return out


def read_checkpoint(path):
    """Raw parse of an SQFG checkpoint: (version, meta dict, params, opt)."""
    v, npar, nopt, mb = C.c_int32(), C.c_int64(), C.c_int64(), C.c_int64()
    p = os.fspath(path).encode()
    L.check(L.sqf_checkpoint_info(p, C.byref(v), C.byref(npar), C.byref(nopt), C.byref(mb)))
    params = np.zeros(npar.value, np.float32)
    opt = np.zeros(max(1, nopt.value), np.float32)
    meta = C.create_string_buffer(mb.value)
    L.check(L.sqf_checkpoint_read(p, _ptr(params), _ptr(opt), meta, mb.value))
    kv = dict(line.split(" = ", 1) for line in meta.value.decode().splitlines() if line)
    return int(v.value), kv, params, opt[:nopt.value]


def nccl_unique_id() -> bytes:
    buf = (C.c_char * 128)()
    L.check(L.sqf_nccl_unique_id(buf))
    return bytes(buf)


@dataclass
class EvalStats:
    loss: float
    nll: float
    ntokens: int
    ncorrect: int


_COLL_NP = {L.COLL_F32: np.float32, L.COLL_F16: np.float16, L.COLL_BF16: np.uint16, L.COLL_F64: np.float64}


def _host_allreduce_trampoline(fn):
    def cb(buf, count, dtype, _user):
        try:
            arr = np.ctypeslib.as_array(C.cast(buf, C.POINTER(C.c_uint8)), shape=(count * np.dtype(
                _COLL_NP[dtype]).itemsize,)).view(_COLL_NP[dtype])
            fn(arr, dtype)
            return 0
        except Exception:  # noqa: BLE001 -- reported as a status through the C ABI
            import traceback
            traceback.print_exc()
            return 1
    return cb


class Trainer:
    """Drop-in for the reference's Trainer (trainer.hpp:80-125) on B200.

    ``arch`` + ``overrides`` resolve like Registry::resolve_architecture; pass a
    ``corpus`` for an in-memory task (the reference's task-injecting ctor) or set
    ``task=synthetic`` in the overrides. ``rank``/``world``/``nccl_id`` place this
    process in the data-parallel group (one process per GPU).
    """

    def __init__(self, arch: str, overrides: dict | None = None, corpus: Corpus | None = None,
                 src_vocab: int = 0, tgt_vocab: int = 0, rank: int = 0, world: int = 1,
                 nccl_id: bytes | None = None, host_allreduce=None):
        overrides = dict(overrides or {})
        self.overrides = overrides
        k, v, n = _kv(overrides)
        self.corpus = corpus
        if corpus is not None:
            task = (_ptr(corpus.src_len), _ptr(corpus.tgt_len), _ptr(corpus.src_ids), _ptr(corpus.tgt_ids),
                    corpus.npairs, src_vocab, tgt_vocab)
        else:
            task = (None, None, None, None, 0, 0, 0)
        if host_allreduce is not None:
            # host_allreduce(array) sums a numpy view of the buffer in place
            # over all ranks (e.g. torch.distributed gloo); tests/tooling only
            self._coll_cb = L.HOST_ALLREDUCE_FN(_host_allreduce_trampoline(host_allreduce))
            h = L.sqf_trainer_create_host_collective(arch.encode(), k, v, n, *task, rank, world, self._coll_cb, None)
        else:
            idbuf = (C.c_char * 128).from_buffer_copy(nccl_id) if nccl_id else None
            h = L.sqf_trainer_create(arch.encode(), k, v, n, *task, rank, world, idbuf)
        if not h:
            raise L.NativeError(L.sqf_last_status(), (L.sqf_last_error() or b"").decode())
        self._h = h
        self.workers = int(overrides.get("workers", 1))
        self.accum = int(overrides.get("accum", 1))

    def close(self):
        if getattr(self, "_h", None):
            L.sqf_trainer_free(self._h)
            self._h = None

    def __del__(self):
        self.close()

    @property
    def collective(self) -> str:
        return L.sqf_trainer_collective(self._h).decode()

    # ---- the hot path
    def train_one(self):
        st = L.StepStats()
        r = L.check(L.sqf_trainer_train_one(self._h, C.byref(st)))
        return None if r == 1 else st.as_dict()

    def train_step(self, sub):
        """sub[w][a] = list of corpus indices (reference train_step(sub[W][A]))."""
        counts = np.array([len(m) for row in sub for m in row], np.int32)
        members = np.array([x for row in sub for m in row for x in m] or [0], np.int32)
        st = L.StepStats()
        L.check(L.sqf_trainer_train_step(self._h, _ptr(members), _ptr(counts), C.byref(st)))
        return st.as_dict()

    def evaluate(self, corpus_idx) -> EvalStats:
        idx = np.asarray(corpus_idx, np.int32)
        loss, nll, nt, nc = C.c_double(), C.c_double(), C.c_int64(), C.c_int64()
        L.check(L.sqf_trainer_evaluate(self._h, _ptr(idx), len(idx), C.byref(loss), C.byref(nll), C.byref(nt),
                                       C.byref(nc)))
        return EvalStats(loss.value, nll.value, nt.value, nc.value)

    # ---- generation (reference generate.hpp:46-90; decoder on the device)
    def gen_config(self) -> dict:
        """gen_config_from(the resolved config) (generate.cpp:15-26)."""
        g = L.GenConfigC()
        L.check(L.sqf_gen_config_default(self._h, C.byref(g)))
        return {f: getattr(g, f) for f, _ in L.GenConfigC._fields_}

    def generate(self, sources, mode: str = "beam", stream_ids=None, **cfg) -> list:
        """beam_search / diverse_beam_search / top_k_sample over source id rows
        (eos-terminated lists; [] = empty row). Returns one list of Hypothesis per
        sentence (one element for mode="sample")."""
        modes = {"beam": 0, "diverse": 1, "sample": 2}
        if mode not in modes:
            raise ValueError(f"unknown generation mode {mode!r}")
        g = L.GenConfigC(**{**self.gen_config(), **cfg})
        src, lens = _pad_rows(sources)
        ids = None if stream_ids is None else np.ascontiguousarray(stream_ids, np.uint64)
        h = C.c_void_p()
        L.check(L.sqf_generate(self._h, modes[mode], _ptr(src), _ptr(lens), len(lens), src.shape[1], C.byref(g),
                               None if ids is None else _ptr(ids), C.byref(h)))
        try:
            return [[_read_hyp(L.sqf_gen_hyp, h, s, k) for k in range(L.sqf_gen_count(h, s))]
                    for s in range(len(lens))]
        finally:
            L.sqf_gen_free(h)

    # ---- state
    @property
    def num_params(self) -> int:
        return int(L.sqf_trainer_num_params(self._h))

    def params(self) -> np.ndarray:
        out = np.zeros(self.num_params, np.float32)
        L.check(L.sqf_trainer_params(self._h, _ptr(out)))
        return out

    def set_params(self, p: np.ndarray):
        p = np.ascontiguousarray(p, np.float32)
        L.check(L.sqf_trainer_set_params(self._h, _ptr(p)))

    def last_grads(self) -> np.ndarray:
        out = np.zeros(self.num_params, np.float32)
        L.check(L.sqf_trainer_last_grads(self._h, _ptr(out)))
        return out

    def manifest(self):
        out = []
        buf = C.create_string_buffer(256)
        for i in range(L.sqf_trainer_manifest_size(self._h)):
            off, num, doff = C.c_int64(), C.c_int64(), C.c_int64()
            L.check(L.sqf_trainer_manifest_entry(self._h, i, buf, 256, C.byref(off), C.byref(num), C.byref(doff)))
            out.append((buf.value.decode(), off.value, num.value, doff.value))
        return out

    def adam_state(self):
        m = np.zeros(self.num_params, np.float32)
        v = np.zeros(self.num_params, np.float32)
        t = C.c_int64()
        L.check(L.sqf_trainer_adam_state(self._h, _ptr(m), _ptr(v), C.byref(t)))
        return m, v, t.value

    def scaler(self):
        s, g = C.c_double(), C.c_int64()
        L.check(L.sqf_trainer_scaler(self._h, C.byref(s), C.byref(g)))
        return s.value, g.value

    def progress(self):
        s, e, c, n = C.c_int64(), C.c_int32(), C.c_int32(), C.c_int32()
        L.check(L.sqf_trainer_progress(self._h, C.byref(s), C.byref(e), C.byref(c), C.byref(n)))
        return {"step": s.value, "epoch": e.value, "cursor": c.value, "batches_per_epoch": n.value}

    def set_overflow_injector(self, steps):
        a = np.asarray(list(steps) or [0], np.int64)
        L.check(L.sqf_trainer_set_injector(self._h, _ptr(a), len(list(steps))))

    def restore(self, step, epoch, cursor, scale=0.0, successes=0):
        L.check(L.sqf_trainer_restore(self._h, step, epoch, cursor, scale, successes))

    @property
    def kernel_launches(self) -> int:
        return int(L.sqf_trainer_kernel_launches(self._h))

    @property
    def last_step_ms(self) -> float:
        return float(L.sqf_trainer_last_step_ms(self._h))

    def flush_ms(self) -> float:
        """Wait (on the trainer stream) for the last step's optimizer update,
        which overlaps the next step; device ms from the step's end to there."""
        v = float(L.sqf_trainer_flush_ms(self._h))
        if v < 0:
            raise L.NativeError(L.sqf_last_status(), L.sqf_last_error().decode())
        return v

    @property
    def last_io_bytes(self):
        """(host->device, device->host) bytes moved by the last step."""
        d2h = C.c_int64()
        h2d = L.sqf_trainer_last_io_bytes(self._h, C.byref(d2h))
        return int(h2d), int(d2h.value)

    def save(self, path: str):
        """Checkpoint (SQFG v2, the reference's container) of the full training state."""
        L.check(L.sqf_trainer_save(self._h, os.fspath(path).encode()))

    def load(self, path: str) -> int:
        """Restore a checkpoint (ours or the reference's) into this trainer; returns the file version."""
        v = C.c_int32()
        L.check(L.sqf_trainer_load(self._h, os.fspath(path).encode(), C.byref(v)))
        return int(v.value)

    def overlap_log(self):
        """(bucket issue order, number issued while backward was running) of the last step."""
        cap = 1 << 16
        buf = (C.c_int32 * cap)()
        early = C.c_int32()
        n = L.sqf_trainer_overlap_log(self._h, buf, cap, C.byref(early))
        return list(buf[:n]), int(early.value)

    @property
    def stream(self) -> int:
        return int(L.sqf_trainer_stream(self._h) or 0)

    def set_profile(self, on=True):
        """True/1: serialised per-launch timing; 2: timeline of the concurrent schedule."""
        L.check(L.sqf_trainer_set_profile(self._h, int(on)))

    def timeline(self):
        """Timeline mode: the last step's launches as rows (stream, class, t0_ms, t1_ms);
        stream 0 = main, 1 = side (parameter gradients, optimizer), 2 = comm."""
        n = L.sqf_trainer_timeline(self._h, None, 0)
        out = np.zeros((max(n, 1), 4), np.float32)
        L.sqf_trainer_timeline(self._h, out.ctypes.data, n)
        return out[:n]

    def profile(self):
        """Per kernel class: {name: (ms, flops, bytes, launches)} accumulated since set_profile."""
        out = {}
        for c in range(64):
            ms, fl, by, n = C.c_double(), C.c_double(), C.c_double(), C.c_int64()
            name = L.sqf_trainer_profile(self._h, c, C.byref(ms), C.byref(fl), C.byref(by), C.byref(n))
            if not name:
                break
            out[name.decode()] = (ms.value, fl.value, by.value, n.value)
        return out


# ---- generation helpers (reference generate.hpp)
@dataclass
class Hypothesis:
    tokens: list
    step_scores: list
    cum_logprob: float
    score: float
    finish_step: int
    finished: bool


def _pad_rows(sources):
    lens = np.array([len(r) for r in sources], np.int32)
    width = max(1, int(lens.max()) if len(lens) else 1)
    src = np.full((len(lens), width), 1, np.int32)  # pad id 1
    for i, r in enumerate(sources):
        src[i, :len(r)] = r
    return src, lens


def _read_hyp(fn, h, s, k, cap=4096):
    tok = np.zeros(cap, np.int32)
    sc = np.zeros(cap, np.float32)
    n, cum, score, fs, fin = C.c_int32(), C.c_double(), C.c_double(), C.c_int32(), C.c_int32()
    st = fn(h, s, k, _ptr(tok), _ptr(sc), cap, C.byref(n), C.byref(cum), C.byref(score), C.byref(fs), C.byref(fin))
    if st != 0:
        raise RuntimeError(f"generation: reading hypothesis failed ({st})")
    return Hypothesis(tok[:n.value].tolist(), sc[:n.value].tolist(), cum.value, score.value, fs.value,
                      bool(fin.value))


def score_hypothesis(cum_logprob: float, length: int, alpha: float) -> float:
    out = C.c_double()
    L.check(L.sqf_score_hypothesis(cum_logprob, length, alpha, C.byref(out)))
    return out.value


def sample_from_topk(logits, k: int, temperature: float, u: float) -> int:
    x = np.ascontiguousarray(logits, np.float32)
    out = C.c_int32()
    L.check(L.sqf_sample_from_topk(_ptr(x), len(x), k, temperature, u, C.byref(out)))
    return out.value


def batch_for_inference(lengths, max_tokens: int) -> list:
    lens = np.ascontiguousarray(lengths, np.int32)
    n = len(lens)
    sizes = np.zeros(max(n, 1), np.int32)
    members = np.zeros(max(n, 1), np.int32)
    ng = C.c_int32()
    L.check(L.sqf_batch_for_inference(_ptr(lens), n, max_tokens, C.byref(ng), _ptr(sizes), _ptr(members)))
    out, at = [], 0
    for i in range(ng.value):
        out.append(members[at:at + sizes[i]].tolist())
        at += sizes[i]
    return out
