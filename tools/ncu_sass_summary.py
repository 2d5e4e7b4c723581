"""Summarise an ncu report's SASS source page: stall samples and executed instructions by
opcode and the hottest instructions.   python tools/ncu_sass_summary.py report.ncu-rep [kernel-regex]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hdr_i]
data = [dict(zip(hdr, r)) for r in rows[hdr_i + 1:] if len(r) == len(hdr)]


def num(v):
    try:
        return float(v)
    except ValueError:
        return 0.0


tot_s = sum(num(d["Warp Stall Sampling (All Samples)"]) for d in data)
tot_i = sum(num(d["Instructions Executed"]) for d in data)
by_op = collections.defaultdict(lambda: [0.0, 0.0])
for d in data:
    op = d["Source"].split()[0] if d["Source"].split() else "?"
    if op.startswith("@"):
        op = d["Source"].split()[1]
    op = op.split(".")[0]
    by_op[op][0] += num(d["Warp Stall Sampling (All Samples)"])
    by_op[op][1] += num(d["Instructions Executed"])
print(f"total stall samples {tot_s:.0f}  executed warp instructions {tot_i:.0f}")
print("opcode            samples%   instr%")
for op, (s, i) in sorted(by_op.items(), key=lambda kv: -kv[1][0])[:25]:
    print(f"{op:16s} {100 * s / tot_s:8.2f} {100 * i / tot_i:8.2f}")
print("\nhottest instructions (samples)")
for d in sorted(data, key=lambda d: -num(d["Warp Stall Sampling (All Samples)"]))[:30]:
    print(f'{num(d["Warp Stall Sampling (All Samples)"]):8.0f} {num(d["Instructions Executed"]):12.0f}  {d["Address"][-5:]}  {d["Source"][:90]}')
