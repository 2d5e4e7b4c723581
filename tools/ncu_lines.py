"""Warp-stall samples of an ncu report aggregated by CUDA source line (needs -lineinfo and
--import-source).   python tools/ncu_lines.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
agg, src, path = {}, {}, ""
rows = csv.reader(io.StringIO(out))
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr[:2], r[:2]))
    try:
        s = float(r[4] or 0)
    except ValueError:
        continue
    key = (path, d["Line No"])
    agg[key] = agg.get(key, 0.0) + s
    src.setdefault(key, r[1])
tot = sum(agg.values()) or 1.0
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{100 * v / tot:6.2f}%  {k[0]}:{k[1]}  {src[k].strip()[:100]}")
