"""Executed SASS instructions of one kernel grouped by opcode (ncu source page):
python tools/sass_ops.py report.ncu-rep [top] [kernel-regex]"""
import collections, csv, io, subprocess, sys
rep = sys.argv[1]
flt = ["--kernel-name", "regex:" + sys.argv[3]] if len(sys.argv) > 3 else []
raw = subprocess.run(["ncu", "-i", rep, *flt, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = None
agg = collections.Counter()
tot = 0
for r in rows:
    if r and r[0] == "Address":
        hdr = {k: i for i, k in enumerate(r)}
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    src = r[hdr["Source"]].strip()
    try:
        n = float(r[hdr["Instructions Executed"]] or 0)
    except ValueError:
        continue
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    agg[op] += n
    tot += n
for op, n in agg.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 30):
    print(f"{op:12s} {n:14.0f} {100*n/tot:5.1f}%")
print("total", tot)
