"""Summarise an ncu report (raw page) into the metrics the roofline needs (development tool)."""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "lts__t_bytes.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg.per_second",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed"]


def summary(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {"kernel": vals[hdr.index("Kernel Name")]}
    for k in KEYS:
        if k in hdr:
            d[k] = (vals[hdr.index(k)], units[hdr.index(k)])
    stalls = {}
    for i, h in enumerate(hdr):
        if h.startswith("smsp__average_warp_latency_issue_stalled_") or (h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")):
            try:
                v = float(vals[i].replace(",", ""))
            except ValueError:
                continue
            if v > 0:
                stalls[h.split("stalled_")[1]] = v
    d["stalls_top"] = sorted(stalls.items(), key=lambda kv: -kv[1])[:12]
    return d


if __name__ == "__main__":
    for rep in sys.argv[1:]:
        print(json.dumps(summary(rep), indent=1))
