"""Timeline of one C4 training step on the concurrent schedule (main stream,
side stream, overlapped optimizer): per-launch [t0, t1] from CUDA events, then
per stream the busy time by kernel class and the idle gaps. Events between
launches break programmatic-dependent-launch overlap, so the step is a little
slower than in bench.py; this is for attribution, not a benchmark."""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

CLS = ["gemm_fwd", "gemm_dgrad", "gemm_wgrad", "attn_fwd", "attn_bwd", "layernorm", "xent", "embed", "bias_grad",
       "optim"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--accum", type=int, default=0)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    import torch
    torch.cuda.set_device(0)
    import paper_1904_01038_b200 as sqf
    cfg = dict(bench.CONFIGS[a.config])
    if a.accum:
        cfg["accum"] = a.accum
    V = cfg["vocab"]
    corpus = sqf.synthetic_corpus(20000, V, V, 1.1, 1)
    ov = {"max_tokens": cfg["max_tokens"], "accum": cfg["accum"], "dispatch": "deal",
          "fp16": cfg["prec"] == "fp16", "seed": 1, "max_epochs": 1000, "fp16_init_scale": 1.0,
          "fp16_min_scale": 2.0 ** -14}
    tr = sqf.Trainer(cfg["arch"], ov, corpus=corpus, src_vocab=V, tgt_vocab=V)
    for _ in range(a.warmup):
        tr.train_one()
    plain = []
    for _ in range(2):
        tr.train_one()
        plain.append(tr.last_step_ms)
    tr.set_profile(2)
    s = tr.train_one()
    tl = tr.timeline()
    step_ms = tr.last_step_ms
    tr.set_profile(0)
    print(f"step ms without events {np.mean(plain):.2f}; with timeline events {step_ms:.2f}; tokens {s['ntokens']}")
    def union(iv):
        tot, cur = 0.0, None
        for t0, t1 in sorted(iv):
            if cur is None or t0 > cur[1]:
                if cur:
                    tot += cur[1] - cur[0]
                cur = [t0, t1]
            else:
                cur[1] = max(cur[1], t1)
        return tot + (cur[1] - cur[0] if cur else 0.0)
    allv = [(float(r[2]), float(r[3])) for r in tl]
    if allv:
        span = max(t1 for _, t1 in allv) - min(t0 for t0, _ in allv)
        print(f"any stream busy {union(allv):.2f} ms of span {span:.2f} ms")
    for st, name in ((0, "main"), (1, "side"), (2, "comm"), (3, "forward-ahead")):
        rows = tl[tl[:, 0] == st]
        if not len(rows):
            continue
        busy = {}
        for r in rows:
            busy[CLS[int(r[1])]] = busy.get(CLS[int(r[1])], 0.0) + float(r[3] - r[2])
        iv = sorted((float(r[2]), float(r[3])) for r in rows)
        union, cur = 0.0, None
        for t0, t1 in iv:
            if cur is None or t0 > cur[1]:
                if cur:
                    union += cur[1] - cur[0]
                cur = [t0, t1]
            else:
                cur[1] = max(cur[1], t1)
        if cur:
            union += cur[1] - cur[0]
        span = iv[-1][1] - iv[0][0]
        print(f"{name}: {len(rows)} launches, busy {union:.2f} ms of span {span:.2f} ms "
              f"(idle {span - union:.2f})")
        for k, v in sorted(busy.items(), key=lambda x: -x[1]):
            print(f"   {k:12s} {v:8.2f} ms")
    if a.out:
        np.savetxt(a.out, tl, fmt="%.4f", delimiter=",", header="stream,class,t0_ms,t1_ms")


if __name__ == "__main__":
    main()
