"""Instruction mass of one kernel grouped by execution count (which loop level a
line belongs to), with the dominant opcodes of each group.
usage: ncu_buckets.py rep kernel-regex [top]"""
import csv, subprocess, sys
from collections import Counter, defaultdict
rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 12
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{kre}"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hi]
iS, iSm, iE = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
mass, lines, ops, smp = Counter(), Counter(), defaultdict(Counter), Counter()
tot = 0
for r in rows[hi + 1:]:
    if not r or r[0] == "Address" or "Kernel" in r[0]:
        break
    try:
        e, sm = int(r[iE] or 0), int(r[iSm] or 0)
    except ValueError:
        continue
    src = r[iS].strip()
    op = src.split()[0] if not src.startswith("@") else src.split()[1]
    b = round(e, -3)
    mass[b] += e; lines[b] += 1; ops[b][op.split(".")[0]] += 1; smp[b] += sm; tot += e
print(f"total {tot:,}")
for b, m in mass.most_common(top):
    print(f"exec~{b:>12,}  lines {lines[b]:4d}  mass {m:>13,} ({m / tot:5.1%})  samples {smp[b]:6,}  "
          + " ".join(f"{k}:{v}" for k, v in ops[b].most_common(8)))
