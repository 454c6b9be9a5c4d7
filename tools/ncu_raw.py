"""Print selected raw metrics of an ncu report (development tool).

    python tools/ncu_raw.py gpurun_out/prof.ncu-rep [more metric names]
"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "launch__grid_size", "launch__cluster_dim_x", "sm__cycles_elapsed.avg.per_second",
        "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum",
        "launch__registers_per_thread", "smsp__warps_active.avg.per_cycle_active"]


def main():
    rep = sys.argv[1]
    keys = KEYS + sys.argv[2:]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for v in rows[2:]:
        print("--", v[hdr.index("Kernel Name")][:70] if "Kernel Name" in hdr else "")
        for k in keys:
            if k in hdr:
                i = hdr.index(k)
                print(f"  {k:62s} {v[i]:>18s} {units[i]}")


if __name__ == "__main__":
    main()
