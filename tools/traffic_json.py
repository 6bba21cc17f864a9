"""profiles/roofline_traffic.json from an `ncu --set full` GEMM capture
(raw CSV): mean DRAM bytes (read + write) per captured gemm_tc2 launch."""
import csv
import json
import sys


def main(raw_csv, out, source):
    rows = list(csv.reader(open(raw_csv)))
    head = rows[0]
    idx = {h: i for i, h in enumerate(head)}
    vals = []
    for r in rows[2:]:
        if "gemm_tc2" not in r[idx["Kernel Name"]]:
            continue
        unit_r, unit_w = rows[1][idx["dram__bytes_read.sum"]], rows[1][idx["dram__bytes_write.sum"]]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd = float(r[idx["dram__bytes_read.sum"]].replace(",", "")) * scale.get(unit_r, 1)
        wr = float(r[idx["dram__bytes_write.sum"]].replace(",", "")) * scale.get(unit_w, 1)
        vals.append(rd + wr)
    json.dump({"kernel": "tcgen05 CTA-pair GEMM (gemm_tc2, TMA-store epilogue)",
               "dram_bytes_per_launch": sum(vals) / len(vals), "launches": len(vals), "source": source},
              open(out, "w"), indent=1)
    print(len(vals), sum(vals) / len(vals))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3])
