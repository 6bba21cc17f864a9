"""Regenerate tests/golden/oracle_golden.json from the reference itself
(oracle/_ref/libseqforge_ref.so, built from /root/reference by oracle/Makefile).
Run in the build container: python tests/golden/make_golden.py"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import ref  # noqa: E402
from paper_1904_01038_b200 import synthetic_corpus  # noqa: E402


def main():
    ref.build()
    out = {
        "rng_u64_1_4242": [int(x) for x in ref.rng_u64(1, 4242, 0, 8)],
        "shuffle_37_1_3": ref.shuffle_epoch(37, 1, 3),
        "batches_200_512": ref.make_batches(synthetic_corpus(200, 1000, 1000, 1.1, 1), 512, 0, 1),
        "xent": [],
    }
    rng = np.random.default_rng(7)
    for fp16, eps, seed in [(False, 0.1, 1.0), (True, 0.1, 128.0), (False, 0.0, 1.0)]:
        lg = (rng.standard_normal((3, 11)) * 2).astype(np.float32)
        if fp16:
            lg = ref.quantize_array(lg)
        gold = [4, 1, 7]
        loss, nll, corr, dl = ref.xent(lg, gold, eps, fp16, seed)
        out["xent"].append({"logits": lg.tolist(), "gold": gold, "eps": eps, "fp16": fp16, "seed": seed,
                            "loss": loss.tolist(), "dlogits": dl.tolist()})
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "oracle_golden.json")
    with open(path, "w") as f:
        json.dump(out, f)
    print("wrote", path)


if __name__ == "__main__":
    main()
