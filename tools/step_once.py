"""Run W warm-up steps + 1 step of a bench config through the public API (for ncu
launch lists / kernel captures). Not a benchmark: timings under a profiler are
not reported anywhere."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--accum", type=int, default=0)
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
    s = tr.train_one()
    print("step", s, "launches", tr.kernel_launches)


if __name__ == "__main__":
    main()
