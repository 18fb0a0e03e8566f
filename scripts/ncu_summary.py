"""Summarise one ncu report: headline metrics, stall reasons, top SASS lines by samples."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
d = dict(zip(r[0], r[2]))
keys = ["Kernel Name", "gpu__time_duration.sum", "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "local_load_requests" ]
for k in keys:
    if k in d:
        print(f"{k:70s} {d[k]}")
st = []
for k, v in d.items():
    if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
        try:
            st.append((float(v.replace(",", "")), k[len("smsp__pcsamp_warps_issue_stalled_"):]))
        except ValueError:
            pass
tot = sum(v for v, _ in st)
print("stalls:", ", ".join(f"{k} {100*v/tot:.1f}%" for v, k in sorted(st, reverse=True)[:10]))
if len(sys.argv) > 2:
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    h = rows[1]
    ix = {k: i for i, k in enumerate(h)}
    data = rows[2:]
    S = "Warp Stall Sampling (All Samples)"
    scols = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
    data.sort(key=lambda x: -int(x[ix[S]] or 0))
    for x in data[: int(sys.argv[2])]:
        top = sorted(((int(x[ix[k]] or 0), k) for k in scols), reverse=True)[:2]
        print(f"{int(x[ix[S]] or 0):6d} {x[ix['Source']][:58]:58s} {top}")
