"""Generation throughput: beam search over a batch of
synthetic source sentences with the B200 decoder, incremental (K/V caches on
the device) vs cache-free, next to the reference's generate.cpp on the host
(a bounded sample). Prints one JSON line. Random-init weights (the speed does
not depend on them; hypotheses run to the length cap more often than with a
trained model, which is the conservative case)."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--arch", default="transformer_base_defaults")
    ap.add_argument("--vocab", type=int, default=1000)
    ap.add_argument("--sentences", type=int, default=32)
    ap.add_argument("--beam", type=int, default=4)
    ap.add_argument("--max-len", type=int, default=0)
    ap.add_argument("--ref-sentences", type=int, default=4)
    ap.add_argument("--precision", choices=["fp32", "fp16", "bf16"], default="fp32")
    args = ap.parse_args()
    import paper_1904_01038_b200 as sqf
    c = sqf.synthetic_corpus(max(args.sentences, 64), args.vocab, args.vocab, 1.1, 1)
    ov = {"max_tokens": 1024, "seed": 1}
    tov = dict(ov, **({args.precision: True} if args.precision != "fp32" else {}))
    tr = sqf.Trainer(args.arch, tov, corpus=c, src_vocab=args.vocab, tgt_vocab=args.vocab)
    src = [list(c.pair(i)[0]) for i in range(args.sentences)]
    out = {"workload": f"{args.arch} beam {args.beam}, {args.sentences} sentences, V={args.vocab}, {args.precision} weights"}
    tr.generate(src[:2], "beam", beam=args.beam, max_len=args.max_len)  # warm-up
    for name, nc, reps in (("incremental", False, 5), ("recompute", True, 1)):
        times = []
        for _ in range(reps):
            t0 = time.perf_counter()
            res = tr.generate(src, "beam", beam=args.beam, max_len=args.max_len, no_cache=nc)
            times.append(time.perf_counter() - t0)
        dt = sorted(times)[len(times) // 2]  # median
        toks = sum(len(hs[0].tokens) for hs in res)
        out[name] = {"s": dt, "runs_s": times, "best_hyp_tokens": toks, "sentences_per_s": len(src) / dt,
                     "tokens_per_s": toks / dt}
    try:
        if args.ref_sentences < 1:
            raise RuntimeError("skipped (--ref-sentences 0)")
        from oracle import ref
        r = ref.RefTrainer(args.arch, ov, c, args.vocab, args.vocab)
        r.set_params(tr.params())
        t0 = time.perf_counter()
        rr = r.generate(src[:args.ref_sentences], "beam", beam=args.beam, max_len=args.max_len)
        dt = time.perf_counter() - t0
        out["reference_cpu_1core"] = {"s": dt, "sentences": args.ref_sentences,
                                      "sentences_per_s": args.ref_sentences / dt}
        mine = tr.generate(src[:args.ref_sentences], "beam", beam=args.beam, max_len=args.max_len)
        out["same_best_tokens_as_reference"] = all(m[0].tokens == q[0]["tokens"] for m, q in zip(mine, rr))
    except Exception as e:  # the oracle is optional here
        out["reference_cpu_1core"] = f"unavailable: {e}"
    print(json.dumps(out))


if __name__ == "__main__":
    main()
