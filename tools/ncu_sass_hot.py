"""Per-instruction hot spots of the first kernel in an .ncu-rep (SASS page):
executed warp instructions and stall samples, in program order, with the
address ranges that dominate.  usage: ncu_sass_hot.py rep [kernel-substring] [top]"""
import csv, subprocess, sys
rep = sys.argv[1]
sub = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
args = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
if sub:
    args += ["-k", f"regex:{sub}"]
out = subprocess.run(args, capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hdr_i]
iA, iS, iSm, iE = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
body = []
for r in rows[hdr_i + 1:]:
    if not r or r[0] == "Address" or r[0].startswith("Kernel"):
        break
    try:
        body.append((r[iA], r[iS].strip(), int(r[iSm] or 0), int(r[iE] or 0)))
    except ValueError:
        pass
tot_e = sum(b[3] for b in body); tot_s = sum(b[2] for b in body)
print(f"instructions {tot_e:,}  samples {tot_s:,}  sass lines {len(body)}")
for k, (a, src, sm, ex) in enumerate(body):
    if ex * 200 > tot_e or sm * 100 > tot_s:
        print(f"{k:5d} {ex:>12,} {sm:>7,}  {src[:90]}")
