"""Print the key metrics of one ncu report (--page raw) as an aligned text summary for profiles/.
usage: python tools/ncu_summary.py REPORT.ncu-rep "title line" > profiles/<name>.txt"""
import csv
import io
import subprocess
import sys

KEYS = ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "launch__occupancy_limit", "lts__t_sector_hit_rate.pct", "sm__pipe_tensor_cycles_active.avg.pct",
        "sm__pipe_tensor_subpipe", "sm__pipe_fp64_cycles_active.avg.pct", "sm__inst_executed_pipe_xu.avg.pct",
        "sm__throughput.avg.pct", "sm__warps_active.avg.pct", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__average_warps_issue_stalled", "dram__bytes.sum.per_second")

rep, title = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
for r in rows[2:]:
    d = dict(zip(hdr, r))
    u = dict(zip(hdr, units))
    print(f"# {d.get('Kernel Name', '?')[:110]}  ({title})")
    for k in hdr:
        if any(k.startswith(x) for x in KEYS) and d[k] not in ("", "n/a"):
            if "stalled" in k and not k.endswith("_per_issue_active.ratio"):
                continue
            print(f"{k:<90} {d[k]} {u.get(k, '')}")
