"""Copy the evidence of an evidence job (tools/jobs/r2_evidence.sh: files gpurun_out/<prefix>*) into
profiles/ as summaries named <tag>_*.
usage: python tools/refresh_profiles.py [prefix (default e_)] [tag (default r2)]"""
import csv
import sys
import json
import os
import shutil
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G, P = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")
PRE = sys.argv[1] if len(sys.argv) > 1 else "e_"
TAG = sys.argv[2] if len(sys.argv) > 2 else "r2"
SCALE = {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return rows[0], rows[1], dict(zip(rows[0], rows[2]))


def summary(rep, dst, keys):
    h, units, d = raw(rep)
    with open(dst, "w") as f:
        f.write("# " + d["Kernel Name"][:100] + "  (headline, ncu --set full --clock-control none, one launch)\n")
        for k in h:
            if any(k.startswith(s) for s in keys) and ".min" not in k and ".max" not in k:
                f.write(f"{k:80s} {d[k]} {units[h.index(k)]}\n")
    return h, units, d


keys = ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "sm__throughput.avg.pct", "gpu__compute_memory_throughput.avg.pct", "sm__pipe_fp64_cycles_active.avg.pct",
        "sm__pipe_tensor_cycles_active.avg.pct", "launch__registers_per_thread", "launch__grid_size",
        "sm__warps_active.avg.pct")
h, units, d = summary(os.path.join(G, f"{PRE}select.ncu-rep"), os.path.join(P, f"{TAG}_ncu_select_summary.txt"), keys)
rd, wr = float(d["dram__bytes_read.sum"]), float(d["dram__bytes_write.sum"])
ur, uw = units[h.index("dram__bytes_read.sum")], units[h.index("dram__bytes_write.sum")]
json.dump({"config": "headline", "kernel": "rpc_select_blocked_kernel<bf16,128> (block = 16)",
           "dram_bytes_per_launch": int(rd * SCALE[ur] + wr * SCALE[uw]),
           "source": f"profiles/{TAG}_ncu_select_summary.txt (dram__bytes_read.sum {rd} {ur} + dram__bytes_write.sum {wr} {uw})"},
          open(os.path.join(P, "select_traffic_headline_b16.json"), "w"), indent=1)
for k in ("attend", "weights"):
    if os.path.exists(os.path.join(G, f"{PRE}{k}.ncu-rep")):
        summary(os.path.join(G, f"{PRE}{k}.ncu-rep"), os.path.join(P, f"{TAG}_ncu_{k}_summary.txt"), keys)

rows = list(csv.reader(open(os.path.join(G, f"{PRE}launches.csv"))))
hh, out = None, []
for r in rows:
    if r and r[0] == "ID":
        hh = r
        continue
    if hh and len(r) == len(hh):
        dd = dict(zip(hh, r))
        if dd["Metric Name"] == "gpu__time_duration.sum":
            nm = dd["Kernel Name"].split("(")[0].replace("void ", "").replace("unnamed>::", "").replace("wc::<", "")
            out.append((nm, float(dd["Metric Value"].replace(",", "")) / 1000.0))
start = [i for i, (n, v) in enumerate(out) if "prologue_pass1" in n][1]
seq = []
for n, v in out[start:]:
    seq.append((n, v))
    if "attend_tc_kernel" in n or "attend_ws_kernel" in n:
        break
tot = sum(v for n, v in seq)
bench = json.loads(open(os.path.join(G, f"{PRE}bench.json")).read().strip().splitlines()[-1])
st = bench["stages_ms"]
lines = ["# ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv -- python bench.py --steps 2 --warmup 1"
         " --no-cpu-baseline --no-e2e --no-exact --no-variants",
         "# headline (n = m = 65536, d = 128, r = 256, bf16, blocked selection b = 16): one wildcat_forward, per-launch",
         "# device time; cold-cache and serialised under ncu, so compare SHARES, not absolutes"]
lines += [f"{v:10.1f} us  {100 * v / tot:5.1f} %  {n}" for n, v in seq]
lines.append(f"{tot:10.1f} us  total; selection share {sum(v for n, v in seq if 'select' in n) / tot:.3f} "
             f"(bench stage events: {st['select']:.3f} / {bench['ms_per_step']:.3f} = {st['select'] / bench['ms_per_step']:.3f})")
open(os.path.join(P, f"{TAG}_launches_headline_summary.txt"), "w").write("\n".join(lines) + "\n")
shutil.copy(os.path.join(G, f"{PRE}launches.csv"), os.path.join(P, f"{TAG}_launches_headline.csv"))
shutil.copy(os.path.join(G, f"{PRE}trace.txt"), os.path.join(P, f"{TAG}_blocked_trace_headline.txt"))
for a, b in ((f"{PRE}bench.json", f"{TAG}_bench_headline.json"), (f"{PRE}ref.json", f"{TAG}_bench_reference.json")):
    open(os.path.join(P, b), "w").write(open(os.path.join(G, a)).read().strip().splitlines()[-1] + "\n")
print("\n".join(lines))
