"""Per-CUDA-source-line instruction and stall-sample shares from an ncu report
(`--page source --print-source cuda,sass`). Usage: ncu_lines.py REPORT [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur = None
rows = []
for r in csv.reader(io.StringIO(txt)):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
    elif r[0] == "Line No":
        ix = {k: i for i, k in enumerate(r) if k not in ("Source",)}
        ix["Source"] = 1
    elif r[0].isdigit() and cur:
        rows.append((cur, int(r[0]), r))
IE, S = "Instructions Executed", "Warp Stall Sampling (All Samples)"
def num(v):
    try:
        return int(v)
    except ValueError:  # '-' or a mis-split source line with quotes
        return 0
ti = sum(num(r[ix[IE]]) for _, _, r in rows) or 1
ts = sum(num(r[ix[S]]) for _, _, r in rows) or 1
print(f"total warp instructions {ti}, stall samples {ts}")
agg = sorted(rows, key=lambda x: -num(x[2][ix[S]]))
for f, l, r in agg[:n]:
    print(f"{f:16s}{l:5d} {100*num(r[ix[IE]])/ti:5.1f}%i {100*num(r[ix[S]])/ts:5.1f}%s  {r[1].strip()[:70]}")
