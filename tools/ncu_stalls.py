"""Warp-state sampling shares of one ncu report (sum of the SASS page's stall_* columns).
   python tools/ncu_stalls.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[h]
cols = [i for i, c in enumerate(hdr) if c.startswith("stall_") and "Not Issued" not in c]
tot = {hdr[i]: 0.0 for i in cols}
for r in rows[h + 1:]:
    if len(r) != len(hdr):
        continue
    for i in cols:
        try:
            tot[hdr[i]] += float(r[i])
        except ValueError:
            pass
s = sum(tot.values()) or 1.0
print("warp-state sampling (share of all samples):")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    if v:
        print(f"  {100 * v / s:6.2f}%  {k[6:]}")
