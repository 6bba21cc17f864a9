#!/bin/bash
# ncu --set full of single GEMM shapes in isolation (tools/gemm_one.py), with the
# L2 / tensor-pipe / stall summary. Usage: bash tools/gemm_ncu.sh TAG "shape:tile:pair ..."
TAG=${1:-gemm_ncu}; O=gpurun_out/$TAG; mkdir -p $O
for spec in ${2:-"big8k:256:1 fwd_ffn1:256:1 fwd_out:256:1"}; do
  IFS=: read name tile pair <<< "$spec"
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 3 -c 1 -o $O/${name}_$tile_$pair \
    python tools/gemm_one.py $name $tile $pair > $O/${name}.log 2>&1
  ncu -i $O/${name}_$tile_$pair.ncu-rep --page raw --csv > $O/${name}.raw.csv 2>/dev/null
  rm -f $O/${name}_$tile_$pair.ncu-rep
  python - "$O/${name}.raw.csv" "$name" <<'PY'
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h, r = rows[0], rows[2]
def g(k):
    return r[h.index(k)] if k in h else "?"
keys = ["gpu__time_duration.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "lts__t_sectors.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum.per_second",
        "l1tex__m_xbar2l1tex_read_bytes.sum.per_second", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpc__cycles_elapsed.max", "sm__cycles_active.avg"]
print(sys.argv[2], " ".join(f"{k.split('.')[0].replace('__','.')}[{k.split('.',1)[1][:18]}]={g(k)}" for k in keys))
st = []
for i, k in enumerate(h):
    if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"):
        try:
            st.append((float(r[i].replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError:
            pass
t = sum(v for v, _ in st) or 1
print("   stalls:", " ".join(f"{k}={v/t:.2f}" for v, k in sorted(st, reverse=True)[:6]))
PY
done
