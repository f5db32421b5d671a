"""Executed instructions and stall samples per CUDA source line of one kernel
in an ncu report (source page, cuda,sass view).

    python tools/ncu_lines.py report.ncu-rep [top]
"""
import collections, csv, io, subprocess, sys
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
agg = collections.Counter()
stall = collections.Counter()
src_of = {}
fname = None
hdr = None
cur_line = None
for r in csv.reader(io.StringIO(raw)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = {k: i for i, k in enumerate(r)}
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0]:
        cur_line = (fname, int(r[0]))
        src_of[cur_line] = r[1].strip()[:100]
    try:
        n = float(r[hdr["Instructions Executed"]] or 0)
        sm = float(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)
    except (ValueError, KeyError):
        continue
    agg[cur_line] += n
    stall[cur_line] += sm
tot = sum(agg.values())
tots = sum(stall.values())
print(f"total executed {tot:.0f}, stall samples {tots:.0f}")
for k, n in agg.most_common(top):
    print(f"{n:11.0f} {100*n/tot:5.1f}%  st {100*stall[k]/max(tots,1):5.1f}%  {k[0]}:{k[1]:<5} {src_of.get(k, '')}")
