#!/usr/bin/env python
"""Benchmark: training target tokens/sec of the B200 mixed-precision
data-parallel Transformer step (BASELINE.json metric), one process per GPU.

  python bench.py [--gpus N --steps K --warmup W --config C4|C3|C2|C1 --impl ours|reference]

Default workload (N=1): BASELINE.json configs[3] (C4) — transformer_vaswani_wmt_en_de_big,
fp16, max_tokens 3584 per GPU, update_freq (accum) 16, "deal" dispatch (each GPU packs its
own length-bucketed batches, fairseq semantics), synthetic WMT-shaped corpus.
A step = one optimizer update = accum sub-batches of forward+backward + overflow check + Adam.

Prints ONE JSON line (rank 0). `value` = whole-job target tokens / max-over-ranks device
time of the K steps (CUDA events recorded inside the native trainer on its own stream);
`e2e` = the same tokens over CUDA events on the trainer stream bracketing the K public
`Trainer.train_one()` calls (host batch packing, pinned H2D of ids, D2H of StepStats
included). `roofline` comes from a profiling pass after the timed region (all launches serialised on the
trainer stream, CUDA events around every launch) for the dominant kernel class (tcgen05 GEMM).
`cpu_baseline` times the reference itself (oracle/_ref, the seqforge C++ library built
from its own sources) on a bounded sample of the same workload on the host cores.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# algorithmic training FLOPs per target token (fwd + dgrad + wgrad GEMMs)
CONFIGS = {
    "C4": dict(arch="transformer_vaswani_wmt_en_de_big", vocab=32768, max_tokens=3584, accum=16, prec="fp16",
               flops_per_tok=1258.29e6, desc="transformer_vaswani_wmt_en_de_big fp16, max_tokens 3584/GPU, "
                                              "update_freq 16"),
    "C3": dict(arch="transformer_wmt_en_de", vocab=32768, max_tokens=4096, accum=1, prec="fp16",
               flops_per_tok=364.90e6, desc="transformer_wmt_en_de base fp16, max_tokens 4096/GPU"),
    "C2": dict(arch="transformer_iwslt_de_en", vocab=10000, max_tokens=4096, accum=1, prec="fp16",
               flops_per_tok=219.46e6, desc="transformer_iwslt_de_en fp16, max_tokens 4096"),
    "C1": dict(arch="transformer_base_defaults", vocab=1000, max_tokens=1024, accum=1, prec="fp32",
               flops_per_tok=1.367e6, desc="tiny (2+2, d=64) fp32, max_tokens 1024"),
}


def peaks():
    p = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "source": "fallback"}
    try:
        m = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        p.update({k: m[k] for k in ("hbm_gbs", "bf16_tflops", "bf16_tflops_sustained") if k in m})
        p["source"] = "measured"
    except Exception:
        pass
    return p


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    def __init__(self, gpu_index=0):
        self.gpu = gpu_index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                f = [x.strip() for x in out.split(",")]
                self.samples.append(f)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        sm = sorted(float(s[0]) for s in self.samples if s and s[0].replace(".", "").isdigit())
        mx = [float(s[1]) for s in self.samples if len(s) > 1 and s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("gloo", rank=rank, world_size=world)
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def allmax(x, world):
    if world <= 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def allsum(x, world):
    if world <= 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


# ---------------------------------------------------------------- CPU reference arm
def reference_sample(cfg, threads, max_tokens, steps, warmup):
    """The reference's own Trainer (oracle/_ref, built from /root/reference's sources) on
    the host cores: `threads` independent trainers (the reference is single-threaded),
    each running train_one on its own batch stream of the same synthetic workload."""
    os.environ["SEQFORGE_LOG"] = "quiet"  # the reference warns per oversized singleton
    from oracle import ref
    V = cfg["vocab"]
    # the same corpus as the GPU arm, drawn through the reference's own RngStream
    # (the product library is never loaded on this arm)
    corpus = ref.synthetic_corpus(4000, V, V, 1.1, 1)
    ov = {"max_tokens": max_tokens, "fp16": cfg["prec"] == "fp16", "seed": 1, "max_epochs": 1000}
    trainers = [None] * threads

    def make(i):
        o = dict(ov)
        o["seed"] = i + 1  # distinct epoch shuffles -> distinct batches per worker
        trainers[i] = ref.RefTrainer(cfg["arch"], o, corpus, V, V)

    ts = [threading.Thread(target=make, args=(i,)) for i in range(threads)]
    [t.start() for t in ts]
    [t.join() for t in ts]
    results = []

    def one_round():
        toks = [0] * threads

        def run(i):
            s = trainers[i].train_one()
            toks[i] = s["ntokens"] if s else 0
        t0 = time.perf_counter()
        th = [threading.Thread(target=run, args=(i,)) for i in range(threads)]
        [t.start() for t in th]
        [t.join() for t in th]
        return sum(toks), time.perf_counter() - t0

    for _ in range(warmup):
        one_round()
    for _ in range(steps):
        results.append(one_round())
    tok = sum(r[0] for r in results)
    sec = sum(r[1] for r in results)
    return tok / sec, tok, sec


def ref_threads():
    n = os.cpu_count() or 1
    return max(1, min(n, int(os.environ.get("SQF_REF_THREADS", "8"))))


def host_cpu():
    """(CPU model, logical CPUs) of the box the reference arm runs on."""
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return model, os.cpu_count() or 1


def run_reference_arm(args, cfg):
    rank, world, _ = dist_setup()
    if rank != 0:
        return
    thr = ref_threads()
    mt = args.ref_max_tokens
    value, tok, sec = reference_sample(cfg, thr, mt, args.steps, args.warmup)
    sample = (f"{args.steps} rounds x {thr} threads x 1 train_one step of {cfg['arch']} "
              f"({cfg['prec']} emulated by the reference) at max_tokens={mt}: {tok} target tokens in {sec:.1f} s")
    line = {"metric": METRIC, "value": value, "unit": "tgt_tokens/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * sec / max(1, args.steps), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": cfg["prec"], "data": "synthetic",
            "impl": "reference",
            "config": {"workload": cfg["desc"] + f" (CPU sample at max_tokens {mt})", "arch": cfg["arch"]},
            "cpu_baseline": {"value": value, "unit": "tgt_tokens/s", "cores": thr, "kind": "reference",
                             "sample": sample, "cpu_model": host_cpu()[0], "nproc": host_cpu()[1]},
            "e2e": {"value": value, "unit": "tgt_tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


METRIC = "train tgt tokens/sec, Transformer-big fp16, 1/2/4/8 B200 vs host CPU ref"


# ---------------------------------------------------------------- B200 arm
def run_ours(args, cfg):
    import torch
    rank, world, local = dist_setup()
    torch.cuda.set_device(local)
    import paper_1904_01038_b200 as sqf

    nccl_id = None
    if world > 1:
        import torch.distributed as dist
        obj = [sqf.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    V = cfg["vocab"]
    total_batches = world * cfg["accum"] * (args.warmup + args.steps + 2)
    npairs = max(4000, int(total_batches * cfg["max_tokens"] / 28 * 1.1))
    npairs = min(npairs, 400000)
    corpus = sqf.synthetic_corpus(npairs, V, V, 1.1, 1)
    ov = {"max_tokens": cfg["max_tokens"], "accum": cfg["accum"], "workers": world, "dispatch": "deal",
          "fp16": cfg["prec"] == "fp16", "bf16": cfg["prec"] == "bf16", "seed": 1, "max_epochs": 1000,
          "warmup": 4000, "lr": 5e-4, "bucket_threshold": 1 << 23, "overlap_allreduce": not args.no_overlap}
    # The reference's scaler defaults (128 / window 256 / floor 2^-5,
    # registry.cpp:205-208) unless overridden: gradients are un-normalised token
    # sums until after the all-reduce (trainer.cpp:264-265), so at ~51k tokens
    # per update the warm-up skips a few steps while the scale settles.
    if args.fp16_init_scale:
        ov["fp16_init_scale"] = args.fp16_init_scale
        ov["fp16_min_scale"] = 2.0 ** -14
    tr = sqf.Trainer(cfg["arch"], ov, corpus=corpus, src_vocab=V, tgt_vocab=V, rank=rank, world=world,
                     nccl_id=nccl_id)
    # warm-up: at least W steps, and until the dynamic loss scale has settled
    # (a clean, non-skipped update) so every timed step carries a full update
    done, clean = 0, False
    while done < args.warmup or (not clean and done < args.warmup + 30):
        s = tr.train_one()
        clean = not s["skipped"]
        done += 1
    ext = torch.cuda.ExternalStream(tr.stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(world)
    torch.cuda.synchronize()
    tokens = skipped = launches = 0
    dev_ms = 0.0
    h2d = 0
    with ClockSampler(local) as clk:
        e0.record(ext)
        for _ in range(args.steps):
            s = tr.train_one()
            tokens += s["ntokens"]
            skipped += int(s["skipped"])
            dev_ms += tr.last_step_ms
            h2d += tr.last_io_bytes[0]
            launches += tr.kernel_launches
        # the last step's optimizer update overlaps what would be the next
        # step: close the timed region behind it
        dev_ms += tr.flush_ms()
        e1.record(ext)
        torch.cuda.synchronize()
    barrier(world)
    e2e_ms = e0.elapsed_time(e1)
    dev_ms_max = allmax(dev_ms, world)
    e2e_ms_max = allmax(e2e_ms, world)
    # packed id matrices + embedding-backward segments uploaded per step (this rank)
    h2d = int(h2d / max(1, args.steps))

    # profiling pass (not timed): CUDA events around every launch on the trainer stream
    tr.set_profile(True)
    ps = tr.train_one()
    prof = tr.profile()
    tr.set_profile(False)
    if rank != 0:
        return
    pk = peaks()
    gemm = [prof[k] for k in ("gemm_fwd", "gemm_dgrad", "gemm_wgrad")]
    g_ms = sum(x[0] for x in gemm)
    g_fl = sum(x[1] for x in gemm)
    g_n = sum(x[3] for x in gemm)
    g_by = sum(x[2] for x in gemm)
    tot_ms = sum(x[0] for x in prof.values())
    achieved = g_fl / (g_ms * 1e-3) / 1e12 if g_ms > 0 else 0.0
    peak = pk["bf16_tflops_sustained"]
    value = tokens / (dev_ms_max * 1e-3)
    e2e = tokens / (e2e_ms_max * 1e-3)
    mfu = value / world * cfg["flops_per_tok"] / 1e12 / pk["bf16_tflops"]
    traffic = None
    try:  # DRAM bytes per GEMM launch from the committed ncu --set full capture
        traffic = json.load(open(os.path.join(ROOT, "profiles", "roofline_traffic.json")))["dram_bytes_per_launch"]
    except Exception:
        pass
    line = {
        "metric": METRIC, "value": value, "unit": "tgt_tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dev_ms_max / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": cfg["prec"], "data": "synthetic",
        "config": {"workload": cfg["desc"], "arch": cfg["arch"], "max_tokens_per_gpu": cfg["max_tokens"],
                   "update_freq": cfg["accum"], "dispatch": "deal", "global_batch_tokens": tokens // args.steps,
                   "parallelism": f"dp{world}", "l2": "inputs > L2 (weights+grads+Adam state+activations, GBs)",
                   "skipped_steps": skipped, "loss_scale": tr.scaler()[0] if cfg["prec"] == "fp16" else None,
                   "warmup_steps_run": done,
                   "sub_batch_grouping": ("off" if cfg["prec"] == "fp32" or os.environ.get("SQF_PAIR_SUBBATCH") == "0"
                                          else "an update's 16 packed sub-batches run up to %s per pass as unpadded parts "
                                               "(same batches and tokens; embedding/attention per part; "
                                               "SQF_PAIR_GROUP / SQF_PAIR_PARTS)" % os.environ.get("SQF_PAIR_GROUP", "6")),
                   "allreduce": ("bucketed NCCL, overlapped with the last backward" if not args.no_overlap
                                 else "bucketed NCCL after backward") if world > 1 else "none (1 GPU)"},
        "e2e": {"value": e2e, "unit": "tgt_tokens/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 36},
        "gpu_launches": launches,
        "roofline": {"bound": "tensor", "kernel": "tcgen05 GEMM (fwd/dgrad/wgrad, fused epilogues)",
                     "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak if peak else None,
                     "peak_source": f"{pk['source']} bf16_tflops_sustained (kernel timed inside the step)",
                     "traffic": traffic, "traffic_unit": "DRAM bytes per GEMM launch (ncu --set full capture)",
                     "algorithmic_bytes_per_launch": g_by / g_n if g_n else None, "gemm_share_of_step": g_ms / tot_ms if tot_ms else None,
                     "gemm_launches_per_step": g_n},
        "model_flops_util": mfu,
        "profile_ms_per_step": {k: round(v[0], 3) for k, v in prof.items()},
        "clocks": clk.summary(),
    }
    if world == 1:
        line["predicted_scaling"] = predict_scaling(tr, sqf, dev_ms_max / args.steps, cfg["accum"])
    if world == 1 and not args.no_cpu_baseline:
        try:
            thr = ref_threads()
            v, tok, sec = reference_sample(cfg, thr, args.ref_max_tokens, 1, 0)
            line["cpu_baseline"] = {
                "value": v, "unit": "tgt_tokens/s", "cores": thr, "kind": "reference",
                "cpu_model": host_cpu()[0], "nproc": host_cpu()[1],
                "sample": f"{thr} threads x 1 train_one of {cfg['arch']} at max_tokens={args.ref_max_tokens} "
                          f"({tok} target tokens, {sec:.1f} s) with the reference built from its sources"}
        except Exception as ex:  # the GPU number stands on its own
            line["cpu_baseline"] = {"value": None, "unit": "tgt_tokens/s", "cores": 0, "kind": "reference",
                                    "sample": f"unavailable: {ex}"}
    print(json.dumps(line), flush=True)


def predict_scaling(tr, sqf, step_ms, accum, bus_gbs=400.0):
    """Model, not a measurement: the reference's timeline simulator
    (simulate_timeline, overlap_accum policy) fed with this run's measured
    sub-batch time and each gradient bucket's ring all-reduce time at an
    assumed NCCL bus bandwidth over NVLink 5 (bus_gbs, per direction).
    Returns the predicted weak-scaling efficiency at 2/4/8 GPUs."""
    sizes = [e[2] for e in sorted(tr.manifest(), key=lambda e: e[3])]
    buckets = sqf.bucket_gradients(sizes, 1 << 23)
    esize = 2
    sub_ms = step_ms / accum
    out = {"model": "simulate_timeline overlap_accum, ring all-reduce at %.0f GB/s bus bandwidth (assumed)" % bus_gbs,
           "sub_batch_ms": round(sub_ms, 3)}
    for n in (2, 4, 8):
        comm = [max(1e-6, 2.0 * (n - 1) / n * (b - a) * esize / (bus_gbs * 1e9) * 1e3) for a, b in buckets]
        rows = "\n".join(f"compute {w} " + " ".join([repr(sub_ms)] * accum) for w in range(n))
        text = f"workers {n}\naccum {accum}\nmode overlap_accum\n{rows}\nbuckets " + " ".join(map(repr, comm)) + "\n"
        r = sqf.simulate_timeline(text)
        out[f"efficiency_{n}gpu"] = round(sub_ms * accum / r["makespan"], 4)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C4", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-max-tokens", type=int, default=24)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-overlap", action="store_true", help="all-reduce after backward (C5 'overlap off')")
    ap.add_argument("--max-tokens", type=int, default=0, help="per-GPU token budget override (C5 sweep)")
    ap.add_argument("--accum", type=int, default=0, help="update_freq override")
    ap.add_argument("--fp16-init-scale", type=float, default=0.0,
                    help="start the loss scale here (and lower its floor to 2^-14) instead of the reference defaults")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    if args.max_tokens:
        cfg["max_tokens"] = args.max_tokens
        cfg["desc"] += f" (max_tokens override {args.max_tokens})"
    if args.accum:
        cfg["accum"] = args.accum
        cfg["desc"] += f" (update_freq override {args.accum})"
    if args.impl == "reference":
        run_reference_arm(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
