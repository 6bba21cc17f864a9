"""Per-kernel-class summary of an ncu metrics capture of one training step
(ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,
sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --csv):
launches, summed duration, DRAM bytes and achieved DRAM GB/s per class.
ncu serialises launches and flushes caches between them, so durations are
cold-cache upper bounds; the class SHARE of the step is what to compare."""
import collections
import csv
import re
import sys

UNITS = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "%": 1.0}


def kclass(name):
    n = name.split("(")[0]
    m = re.search(r"gemm_tc2?<(\d+), (\w+), (\w+)", n)
    if m:
        a_mn, b_mn = m.group(2) in ("1", "true"), m.group(3) in ("1", "true")
        return "gemm_wgrad" if a_mn else ("gemm_dgrad" if b_mn else "gemm_fwd")
    for pat, cls in (("ln_gb_", "layernorm_params"), ("ln_fwd", "layernorm_fwd"), ("ln_dx", "layernorm_dx"),
                     ("fwd_k", "attention_fwd"), ("bwd_", "attention_bwd"), ("xent", "xent"),
                     ("adam", "optimizer"), ("nonfinite", "overflow_check"), ("embed", "embedding"),
                     ("colred", "column_sums"), ("convert", "cast"), ("dropout", "dropout")):
        if pat in n:
            return cls
    return "other:" + n.replace("void ", "")[:40]


def main(path):
    per = collections.defaultdict(dict)
    names = {}
    for r in csv.DictReader(l for l in open(path) if l.startswith('"')):
        i = r["ID"]
        names[i] = r["Kernel Name"]
        try:
            per[i][r["Metric Name"]] = float(r["Metric Value"].replace(",", "")) * UNITS.get(r["Metric Unit"], 1.0)
        except ValueError:
            pass
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    for i, m in per.items():
        a = agg[kclass(names[i])]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        a[3] += m.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", 0.0) * m.get(
            "gpu__time_duration.sum", 0.0)
    tot = sum(a[1] for a in agg.values())
    print(f"{'class':22s} {'launches':>8s} {'us':>10s} {'share':>6s} {'DRAM MB':>9s} {'GB/s':>7s} {'tensor%':>7s}")
    for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        gbs = a[2] / (a[1] * 1e3) if a[1] else 0.0
        tp = a[3] / a[1] if a[1] else 0.0
        print(f"{k:22s} {a[0]:8d} {a[1]:10.1f} {100 * a[1] / tot:5.1f}% {a[2] / 1e6:9.1f} {gbs:7.0f} {tp:7.1f}")
    print(f"{'total':22s} {sum(a[0] for a in agg.values()):8d} {tot:10.1f}")


if __name__ == "__main__":
    main(sys.argv[1])
