"""DRAM traffic per launch of the bench kernels from an ncu --set full report:
    python tools/ncu_traffic.py rep out.json workload-label [name=regex ...]
writes {"workload": ..., name: {"kernel", "dram_read_bytes", "dram_write_bytes", "ms", "traffic_bytes"}}
(first matching launch of each regex) -- bench.py reads it for roofline.traffic."""
import csv, json, re, subprocess, sys
rep, out, label = sys.argv[1], sys.argv[2], sys.argv[3]
pairs = [a.split("=", 1) for a in sys.argv[4:]]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, units = rows[0], rows[1]
def val(r, k):
    v = float(r[h.index(k)].replace(",", ""))
    u = units[h.index(k)]
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "usecond": 1e-3,
                "ms": 1, "msecond": 1, "nsecond": 1e-6}.get(u, 1)
res = {"source": f"ncu --set full --clock-control none ({rep.split('/')[-1]}), first launch of each kernel",
       "workload": label}
for name, rx in pairs:
    for r in rows[2:]:
        if re.search(rx, r[h.index("Kernel Name")]):
            rd, wr = val(r, "dram__bytes_read.sum"), val(r, "dram__bytes_write.sum")
            res[name] = {"kernel": r[h.index("Kernel Name")], "dram_read_bytes": rd, "dram_write_bytes": wr,
                         "ms": val(r, "gpu__time_duration.sum"), "traffic_bytes": rd + wr}
            break
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
