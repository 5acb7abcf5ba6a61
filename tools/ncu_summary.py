"""Summarize an ncu report: key metrics per kernel + hottest SASS lines (run here, no GPU)."""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
keys = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "l1tex__t_sector_hit_rate.pct",
        "launch__registers_per_thread", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"]
stall = [k for k in hdr if re.match(r"smsp__average_warps_issue_stalled_.*_per_issue_active.ratio", k)]
for r in rows[2:]:
    print("==", r[hdr.index("Kernel Name")][:90])
    for k in keys:
        if k in hdr:
            print(f"   {k:70s} {r[hdr.index(k)]:>16s} {units[hdr.index(k)]}")
    st = sorted(((float(r[hdr.index(k)] or 0), k) for k in stall), reverse=True)[:6]
    print("   stalls:", ", ".join(f"{k.split('stalled_')[1].split('_per')[0]}={v:.2f}" for v, k in st))
if len(sys.argv) > 2:
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    kern, data, h = None, {}, None
    for r in csv.reader(io.StringIO(src)):
        if r and r[0] == "Kernel Name":
            kern = r[1]; data[kern] = []; continue
        if r and r[0] == "Address":
            h = r; continue
        if kern: data[kern].append(r)
    for k, v in data.items():
        ie, s, ss = h.index("Instructions Executed"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
        tot = sum(int(x[ie]) for x in v); tots = sum(int(x[ss]) for x in v)
        print("##", k[:80], "inst", tot)
        for x in v:
            if int(x[ie]) > tot * float(sys.argv[2]):
                print(f"{int(x[ie]) / tot * 100:5.2f}% {int(x[ss]) / max(tots, 1) * 100:5.1f}%  {x[s]}")
