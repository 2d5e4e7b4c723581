"""Per-instruction stall samples of an ncu report (SASS source page), grouped into regions between
barrier-like instructions, plus the top instructions.  python tools/ncu_sass_regions.py rep [top]"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
i = next(k for k, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[i]
data = [dict(zip(hdr, r)) for r in rows[i + 1:] if len(r) == len(hdr)]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
tot = sum(float(d["Warp Stall Sampling (All Samples)"] or 0) for d in data) or 1
ex = sum(float(d["Instructions Executed"] or 0) for d in data) or 1
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
print(f"total samples {tot:.0f}, warp instructions {ex:.0f}")
# regions: split at BAR.SYNC / SYNCS.PHASECHK (waits) / EXIT
reg, cur = [], {"start": 0, "samp": 0.0, "ex": 0.0, "first": ""}
for k, d in enumerate(data):
    s = d["Source"].strip()
    cur["samp"] += float(d["Warp Stall Sampling (All Samples)"] or 0)
    cur["ex"] += float(d["Instructions Executed"] or 0)
    if not cur["first"]:
        cur["first"] = s
    if "BAR.SYNC" in s or "EXIT" in s:
        cur["end"] = k
        cur["last"] = s
        reg.append(cur)
        cur = {"start": k + 1, "samp": 0.0, "ex": 0.0, "first": ""}
cur["end"] = len(data) - 1
cur["last"] = ""
reg.append(cur)
print("regions split at BAR.SYNC/EXIT (index range, % samples, % instructions):")
for r in reg:
    print(f"  [{r['start']:5d},{r['end']:5d}]  {100 * r['samp'] / tot:6.2f}%  {100 * r['ex'] / ex:6.2f}%  {r['first'][:40]} .. {r['last'][:40]}")
print("top instructions by samples:")
for k, d in sorted(enumerate(data), key=lambda kd: -float(kd[1]["Warp Stall Sampling (All Samples)"] or 0))[:top]:
    st = sorted(((float(d[c] or 0), c[6:]) for c in stall_cols), reverse=True)[:2]
    print(f"  {k:5d} {100 * float(d['Warp Stall Sampling (All Samples)'] or 0) / tot:5.2f}%  ex {d['Instructions Executed']:>9s}  "
          f"{d['Source'].strip()[:60]:60s} {st[0][1]}:{st[0][0]:.0f} {st[1][1]}:{st[1][0]:.0f}")
