"""SASS instruction mix of the built product library per kernel (cuobjdump -sass): the evidence
that the tile kernel streams with TMA bulk copies (UBLKCP + SYNCS mbarrier ops), reduces with no
shared-memory fp64 atomics (ATOMS), uses fp64 RED only in the atomic-mode variants (REDG), and
has no tensor-core work (no HMMA / UTCMMA / tcgen05) -- an fp64 non-contraction path.
    python scripts/sass_summary.py > profiles/r02_sass_mix.md"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.path.join(ROOT, "paper_1005_3158_b200", "libcastfem_b200.so")
CLASSES = {
    "UBLKCP": r"UBLKCP", "SYNCS": r"SYNCS", "LDGSTS (cp.async)": r"LDGSTS", "ATOMS": r"\bATOMS",
    "REDG / RED (global atomics)": r"\bRED(G)?\b|\bREDG\b", "ATOMG": r"\bATOMG", "DFMA": r"\bDFMA",
    "DADD": r"\bDADD", "DMUL": r"\bDMUL", "MUFU (rcp/rsq seeds)": r"\bMUFU", "LDS": r"\bLDS", "STS": r"\bSTS",
    "LDG": r"\bLDG", "STG": r"\bSTG", "BAR": r"\bBAR\b|\bBAR\.", "tensor (HMMA/UTCMMA/UTC*)": r"HMMA|UTCMMA|UTCHMMA|UTCQMMA",
}


def main():
    out = subprocess.run(["cuobjdump", "-sass", SO], capture_output=True, text=True, check=True).stdout
    kernels = collections.OrderedDict()
    cur = None
    for line in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            kernels[cur] = []
            continue
        if cur and re.match(r"\s*/\*[0-9a-f]{4,}\*/", line):
            kernels[cur].append(line)
    arch = re.findall(r"arch = (sm_\w+)", out)
    print("# SASS instruction mix (static counts) — libcastfem_b200.so\n")
    print(f"`cuobjdump -sass paper_1005_3158_b200/libcastfem_b200.so`; arch: {sorted(set(arch))}; "
          f"{len(kernels)} kernels (template variants).\n")
    names = list(CLASSES)
    print("| kernel (demangled prefix) | instr | " + " | ".join(names) + " |")
    print("|---|---|" + "---|" * len(names))
    totals = collections.Counter()
    for k, lines in kernels.items():
        dem = subprocess.run(["c++filt", k], capture_output=True, text=True).stdout.strip()
        short = dem.replace("(anonymous namespace)::", "").split("(")[0].replace("cfb::", "")[:70]
        counts = [sum(1 for ln in lines if re.search(CLASSES[c], ln)) for c in names]
        for c, v in zip(names, counts):
            totals[c] += v
        if "tile_kernel" in dem or "update_kernel" in dem or len(lines) > 0 and any(counts[:6]):
            if "tile_kernel" in dem and "128" not in dem:
                continue
            print(f"| `{short}` | {len(lines)} | " + " | ".join(str(v) for v in counts) + " |")
    print("\nTotals over all kernels: " + ", ".join(f"{c} {totals[c]}" for c in names))


if __name__ == "__main__":
    sys.exit(main())
