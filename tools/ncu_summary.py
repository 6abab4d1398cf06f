"""Summarise an ncu report (--page raw) into a small JSON for profiles/:
python tools/ncu_summary.py <report.ncu-rep> [workload]"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__inst_executed_pipe_fp64.sum", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__inst_executed.sum.per_cycle_active", "launch__grid_size", "launch__block_size",
        "launch__cluster_size", "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg.per_second"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
         "second": 1, "Kbyte/second": 1e3}


def main():
    rep = sys.argv[1]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for row in rows[2:]:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        item = {"kernel": d.get("Kernel Name", "")[:120]}
        for k in KEYS:
            if k in d and d[k] != "":
                v = d[k].replace(",", "")
                try:
                    val = float(v)
                except ValueError:
                    val = v
                item[k] = [val, u.get(k, "")]
        rd, wr = item.get("dram__bytes_read.sum"), item.get("dram__bytes_write.sum")
        if rd and wr:
            item["dram_bytes_per_launch"] = rd[0] * SCALE.get(rd[1], 1) + wr[0] * SCALE.get(wr[1], 1)
        out.append(item)
    res = {"report": rep, "workload": sys.argv[2] if len(sys.argv) > 2 else None, "kernels": out}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
