"""TEST INFRASTRUCTURE ONLY — a numpy restatement of the reference's hot-path
algorithms (seqforge, /root/reference/proj), each function citing the file:line
it follows. It is pinned against the compiled reference (oracle/_ref) by
tests/test_restatement.py and serves as an independent, readable statement of
the semantics the B200 kernels implement. Never imported by the product.
"""
from __future__ import annotations

import math

import numpy as np

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


# ------------------------------------------------------------------ rng.cpp
def fmix64(k: int) -> int:
    """MurmurHash3 finaliser (rng.cpp:10-17)."""
    k &= 0xFFFFFFFFFFFFFFFF
    k ^= k >> 33
    k = (k * 0xFF51AFD7ED558CCD) & 0xFFFFFFFFFFFFFFFF
    k ^= k >> 33
    k = (k * 0xC4CEB9FE1A85EC53) & 0xFFFFFFFFFFFFFFFF
    k ^= k >> 33
    return k


class RngStream:
    """(seed, stream, counter) -> u64 (rng.cpp:21-51, rng.hpp:22-28)."""

    def __init__(self, seed: int, stream: int, counter: int = 0):
        self.seed, self.stream, self.counter = seed, stream, counter

    def next_u64(self) -> int:
        h = fmix64((self.seed + 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF)
        h = fmix64(h ^ self.stream)
        h = fmix64(h ^ self.counter)
        self.counter += 1
        return h

    def next_double(self) -> float:
        return (self.next_u64() >> 11) * 2.0 ** -53

    def next_below(self, n: int) -> int:
        return 0 if n <= 1 else (self.next_u64() * n) >> 64

    def shuffle(self, v: list) -> None:
        for i in range(len(v), 1, -1):
            j = self.next_below(i)
            v[i - 1], v[j] = v[j], v[i - 1]


# ------------------------------------------------------------------ fp16.cpp
def quantize_fp16(x):
    """Round to the binary16 grid, RNE, overflow to inf (fp16.cpp:22-76)."""
    with np.errstate(over="ignore"):
        return np.asarray(x, np.float32).astype(np.float16).astype(np.float32)


# ------------------------------------------------------------------ data.cpp
def make_batches(pairs, max_tokens: int, max_sentences: int = 0):
    """Sort by (tgt len, src len, index), greedy pack under rows*max(S,T) (data.cpp:115-161)."""
    if max_tokens < 1:
        raise ValueError("max_tokens must be >= 1")
    order = sorted(range(len(pairs)), key=lambda i: (len(pairs[i][1]), len(pairs[i][0]), i))
    out, cur, width = [], [], 0
    for i in order:
        w = max(len(pairs[i][0]), len(pairs[i][1]))
        n = len(cur) + 1
        fits = n * max(width, w) <= max_tokens and (max_sentences <= 0 or n <= max_sentences)
        if cur and not fits:
            out.append(cur)
            cur, width = [], 0
        cur.append(i)
        width = max(width, w)
    if cur:
        out.append(cur)
    return out


def shuffle_epoch(nbatches: int, seed: int, epoch: int):
    """Fisher-Yates over batch indices with RngStream(seed, epoch) (data.cpp:163-170)."""
    if epoch < 1:
        raise ValueError("epoch must be >= 1")
    order = list(range(nbatches))
    RngStream(seed, epoch).shuffle(order)
    return order


def make_minibatch(pairs, members, pad=1, bos=0):
    """Padded id matrices: source, target_in = bos + tgt[:-1], target_out = tgt (data.cpp:172-219)."""
    rows = [pairs[m] for m in members]
    S = max(len(s) for s, _ in rows)
    T = max(len(t) for _, t in rows)
    src = np.full((len(rows), S), pad, np.int32)
    tin = np.full((len(rows), T), pad, np.int32)
    tout = np.full((len(rows), T), pad, np.int32)
    for r, (s, t) in enumerate(rows):
        src[r, :len(s)] = s
        tin[r, 0] = bos
        tin[r, 1:len(t)] = t[:-1]
        tout[r, :len(t)] = t
    return {"source": src, "target_in": tin, "target_out": tout,
            "src_lens": np.array([len(s) for s, _ in rows], np.int32),
            "tgt_lens": np.array([len(t) for _, t in rows], np.int32),
            "ntokens": int(sum(len(t) for _, t in rows))}


def split_counts(rows: int, workers: int, accum: int):
    """Row-wise split into W*A contiguous groups (trainer.cpp:186-202)."""
    g = workers * accum
    return [rows // g + (1 if i < rows % g else 0) for i in range(g)]


def bucket_gradients(sizes, threshold: int):
    """Buckets cut walking parameters in reverse canonical order (trainer.cpp:50-73)."""
    offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    out, acc, hi = [], 0, len(sizes)
    for i in range(len(sizes) - 1, -1, -1):
        acc += sizes[i]
        if acc >= threshold:
            out.append((int(offs[i]), int(offs[hi])))
            hi, acc = i, 0
    if hi > 0:
        out.append((0, int(offs[hi])))
    return out


# ------------------------------------------------------------------ trainer.cpp / optim.cpp
def scaler_run(init, window, mn, mx, overflow):
    """LossScaler policy (trainer.cpp:21-48): returns scales after each update and the diverging index."""
    scale, good, out = float(init), 0, []
    for i, ov in enumerate(overflow):
        if ov:
            good = 0
            scale *= 0.5
            if scale < mn:
                return out + [0.0] * (len(overflow) - len(out)), i
        else:
            good += 1
            if good >= window:
                good, scale = 0, min(2.0 * scale, mx)
        out.append(scale)
    return out, -1


def inverse_sqrt(base: float, warmup: int, init: float, step: int) -> float:
    """optim.cpp:97-113."""
    if step < 1:
        raise ValueError("step must be >= 1")
    if step <= warmup:
        return init + (base - init) * step / warmup
    return base * math.sqrt((warmup if warmup > 0 else 1) / step)


def adam(p, g, m, v, t: int, lr: float, b1=0.9, b2=0.98, eps=1e-8):
    """One Adam update in double math with fp32 storage (optim.cpp:48-66); t = steps already taken."""
    t += 1
    bc1, bc2 = 1.0 - b1 ** t, 1.0 - b2 ** t
    gd = np.asarray(g, np.float32).astype(np.float64)
    m32 = (b1 * np.asarray(m, np.float32).astype(np.float64) + (1.0 - b1) * gd).astype(np.float32)
    v32 = (b2 * np.asarray(v, np.float32).astype(np.float64) + (1.0 - b2) * gd * gd).astype(np.float32)
    upd = lr * (m32.astype(np.float64) / bc1) / (np.sqrt(v32.astype(np.float64) / bc2) + eps)
    return (np.asarray(p, np.float32).astype(np.float64) - upd).astype(np.float32), m32, v32


# ------------------------------------------------------------------ tape.cpp ops (float64 statements)
def xent(logits, gold, eps: float, seed: float = 1.0, pad: int = 1):
    """Label-smoothed CE per row + dlogits (tape.cpp:259-290, 481-502; criterions.cpp:10-36)."""
    lg = np.asarray(logits, np.float64)
    R, V = lg.shape
    loss, nll, corr = np.zeros(R), np.zeros(R), np.zeros(R, np.int64)
    dl = np.zeros_like(lg)
    for r in range(R):
        if gold[r] == pad:
            continue
        m = lg[r].max()
        lse = m + math.log(np.exp(lg[r] - m).sum())
        nll[r] = lse - lg[r, gold[r]]
        corr[r] = int(np.argmax(lg[r]) == gold[r])  # first max wins
        loss[r] = nll[r] if eps == 0 else (1 - eps) * nll[r] + eps / V * (lse - lg[r]).sum()
        tgt = np.full(V, eps / V)
        tgt[gold[r]] += 1 - eps
        dl[r] = seed * (np.exp(lg[r] - lse) - tgt)
    return loss, nll, corr, dl


def layer_norm(x, gamma, beta, dy, eps=1e-5):
    """Two-pass LN fwd + bwd (kernels.cpp:30-45, tape.cpp:383-418)."""
    x = np.asarray(x, np.float64)
    mean = x.mean(1, keepdims=True)
    var = ((x - mean) ** 2).mean(1, keepdims=True)
    rstd = 1.0 / np.sqrt(var + eps)
    xh = (x - mean) * rstd
    y = xh * gamma + beta
    dxh = dy * gamma
    dx = rstd * (dxh - dxh.mean(1, keepdims=True) - xh * (dxh * xh).mean(1, keepdims=True))
    return y, dx, (dy * xh).sum(0), np.asarray(dy, np.float64).sum(0)


def attention(q, k, v, heads, key_base, key_len, dout):
    """Multi-head attention over per-row key spans, fwd + bwd (tape.cpp:229-258, 426-480)."""
    q, k, v, dout = (np.asarray(a, np.float64) for a in (q, k, v, dout))
    R, d = q.shape
    dh = d // heads
    sc = 1.0 / math.sqrt(dh)
    out, dq, dk, dv = np.zeros_like(q), np.zeros_like(q), np.zeros_like(k), np.zeros_like(v)
    for r in range(R):
        kb, kl = key_base[r], key_len[r]
        if kl == 0:
            continue
        for h in range(heads):
            cs = slice(h * dh, (h + 1) * dh)
            K, Vv = k[kb:kb + kl, cs], v[kb:kb + kl, cs]
            s = sc * (K @ q[r, cs])
            p = np.exp(s - s.max())
            p /= p.sum()
            out[r, cs] = p @ Vv
            dp = Vv @ dout[r, cs]
            ds = p * (dp - (p * dp).sum())
            dq[r, cs] = sc * (ds @ K)
            dk[kb:kb + kl, cs] += sc * np.outer(ds, q[r, cs])
            dv[kb:kb + kl, cs] += np.outer(p, dout[r, cs])
    return out, dq, dk, dv
