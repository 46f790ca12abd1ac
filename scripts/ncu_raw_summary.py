"""Print the key per-kernel metrics of an `ncu --page raw --csv` export (one row per profiled launch)."""
import csv
import io
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__grid_size"]
t = open(sys.argv[1]).read()
t = t[t.find('"ID"'):]
rows = list(csv.reader(io.StringIO(t)))
h, units = rows[0], rows[1]
for r in rows[2:]:
    print(r[h.index("Kernel Name")][:70])
    for w in WANT:
        if w in h:
            print(f"    {w} = {r[h.index(w)]} {units[h.index(w)]}")
