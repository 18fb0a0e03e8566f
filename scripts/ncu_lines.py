"""Per-source-line instruction / stall attribution for one kernel of an ncu report.
usage: ncu_lines.py REPORT KERNEL_REGEX [top]"""
import csv, re, subprocess, sys, os, glob
rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{kre}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
# the CSV may hold several kernels: keep the first section
secs = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
end = secs[1] if len(secs) > 1 else len(rows)
name = rows[0][1]; h = rows[1]; data = [r for r in rows[2:end] if len(r) == len(h) and r[0] != "Address"]
i_ex = h.index('Instructions Executed'); i_s = h.index('Warp Stall Sampling (All Samples)')
base = int(data[0][0], 16)
met = {int(r[0], 16) - base: (int(r[i_ex] or 0), int(r[i_s] or 0)) for r in data}
mangled = None
so = os.environ.get("CF_SO", "/root/repo/paper_1005_3158_b200/libcastfem_b200.so")
subprocess.run("rm -rf /tmp/cubx && mkdir /tmp/cubx && cd /tmp/cubx && cuobjdump -xelf all " + so + " >/dev/null",
               shell=True)
cub = [f for f in glob.glob("/tmp/cubx/*.cubin") if "cf_api" in f][0]
dis = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout.split("\n")
# find function by demangled-ish name match on template args
tmpl = re.search(r"tile_kernel<(.*)>\(", name) or re.search(r"update_kernel<(.*)>\(", name)
key = "tile_kernel" if "tile_kernel" in name else "update_kernel"
args = [a.strip() for a in tmpl.group(1).split(",")] if tmpl else []
enc = "I" + "".join("Lb1E" if a in ("(bool)1", "true") else "Lb0E" if a in ("(bool)0", "false") else "Li" + a.replace("(int)", "") + "E" for a in args) + "E"
start = [i for i, l in enumerate(dis) if l.startswith("//--------------------- .text.") and key in l and enc in l][0]
cur = None; o2l = {}
for l in dis[start + 1:]:
    if l.startswith("//---------------------"): break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m: cur = (m.group(1).split('/')[-1], int(m.group(2))); continue
    m = re.search(r'/\*([0-9a-f]{4,})\*/', l)
    if m and cur: o2l[int(m.group(1), 16)] = cur
from collections import defaultdict
agg = defaultdict(lambda: [0, 0])
for off, (ex, st) in met.items():
    k = o2l.get(off, ('?', 0)); agg[k][0] += ex; agg[k][1] += st
tot = sum(v[0] for v in agg.values()); tst = sum(v[1] for v in agg.values())
print(name[:80], "instr", tot, "stall samples", tst)
srcs = {}
for fn in set(k[0] for k in agg):
    p = f"/root/repo/paper_1005_3158_b200/csrc/{fn}"
    srcs[fn] = open(p).read().split("\n") if os.path.exists(p) else []
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    fn, ln = k
    text = srcs[fn][ln - 1].strip()[:75] if srcs.get(fn) and 0 < ln <= len(srcs[fn]) else ""
    print(f"{fn}:{ln:4d} stall {100*v[1]/tst:5.1f}% instr {100*v[0]/tot:5.1f}%  {text}")
