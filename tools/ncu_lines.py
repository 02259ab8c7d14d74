"""Dump SASS lines (exec count, stall samples, text) of one kernel of an .ncu-rep.
usage: ncu_lines.py rep kernel-regex [min_exec] [lo-hi]"""
import csv, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]
mn = int(sys.argv[3]) if len(sys.argv) > 3 else 0
rng = tuple(int(v) for v in sys.argv[4].split("-")) if len(sys.argv) > 4 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{kre}"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hi]
iS, iSm, iE = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
body = []
for r in rows[hi + 1:]:
    if not r or r[0] == "Address" or "Kernel" in r[0]:
        break
    try:
        body.append((r[iS].strip(), int(r[iSm] or 0), int(r[iE] or 0)))
    except ValueError:
        pass
tot = sum(b[2] for b in body)
print(f"total instructions {tot:,}  samples {sum(b[1] for b in body):,}")
for k, (s, sm, e) in enumerate(body):
    if e >= mn and (rng is None or rng[0] <= k <= rng[1]):
        print(f"{k:5d} {e:>10,} {sm:>6,}  {s[:90]}")
