"""One line per captured launch from an `ncu --page raw --csv` export: duration,
DRAM bytes and throughput, achieved occupancy, tensor-pipe and issue activity."""
import csv
import sys

COLS = {
    "dur_us": "gpu__time_duration.sum",
    "dram_rd": "dram__bytes_read.sum",
    "dram_wr": "dram__bytes_write.sum",
    "occ_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "mem_pct": "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "l2_pct": "lts__t_sectors.avg.pct_of_peak_sustained_elapsed",
    "issue_pct": "sm__inst_issued.avg.pct_of_peak_sustained_active",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "regs": "launch__registers_per_thread",
}
UNIT = {"gpu__time_duration.sum": 1e-3}  # ns -> us


def main(path):
    rows = list(csv.reader(open(path)))
    if len(rows) < 3:
        return
    head, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(head)}
    for r in rows[2:]:
        out = [r[idx["Kernel Name"]][:48]] if "Kernel Name" in idx else []
        vals = {}
        for k, m in COLS.items():
            if m in idx:
                v = r[idx[m]].replace(",", "")
                try:
                    x = float(v)
                except ValueError:
                    continue
                u = units[idx[m]]
                if m == "gpu__time_duration.sum":
                    x = x * {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(u, 1.0)
                if m.startswith("dram__bytes"):
                    x = x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1.0)
                vals[k] = x
        if "dram_rd" in vals and "dram_wr" in vals and vals.get("dur_us"):
            vals["dram_GBs"] = (vals["dram_rd"] + vals["dram_wr"]) / (vals["dur_us"] * 1e3)
        out += [f"{k}={v:.4g}" for k, v in vals.items()]
        print(" ".join(out))


if __name__ == "__main__":
    main(sys.argv[1])
