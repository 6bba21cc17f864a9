"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel."""
import collections
import csv
import sys


def main(path):
    agg = collections.defaultdict(lambda: [0, 0.0])
    hdr = None
    for r in csv.reader(open(path)):
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        u = d["Metric Unit"]
        v = v / 1e3 if u in ("ns", "nsecond") else v * 1e3 if u in ("ms", "msecond") else v
        name = d["Kernel Name"].split("(")[0].replace("void ", "")
        tmpl = d["Kernel Name"].split("(")[0]
        agg[tmpl][0] += 1
        agg[tmpl][1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"total {tot:.1f} us over {sum(v[0] for v in agg.values())} launches")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{v[1]:10.1f} us {v[0]:5d} launches {100 * v[1] / tot:5.1f}%  {k[:90]}")


if __name__ == "__main__":
    main(sys.argv[1])
