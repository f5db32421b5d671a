"""Per-source-line instruction counts / stall samples for one kernel.

usage: python tools/sass_lines.py <report.ncu-rep> <lib-or-object> <mangled-kernel-substring> [top] [demangled-substring]
Joins ncu's SASS page (executed instructions, stall samples per SASS
address) with nvdisasm -g line info of the same cubin.
"""
import csv, io, os, re, subprocess, sys, tempfile, collections

rep, obj, kern = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        blocks.append(cur)
    elif cur is not None:
        cur["rows"].append(r)
# the report block: 4th argument (a substring of the demangled name), else the first
pick = sys.argv[5] if len(sys.argv) > 5 else None
blk = next(b for b in blocks if (pick is None or pick in b["name"]))
hdr = blk["rows"][0]
idx = {k: i for i, k in enumerate(hdr)}
data = blk["rows"][1:]
base = int(data[0][idx["Address"]], 16)
# line info from nvdisasm
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, capture_output=True)
cubins = [os.path.join(tmp, f) for f in os.listdir(tmp) if f.endswith(".cubin")]
start = None
for cb in cubins:
    sass = subprocess.run(["nvdisasm", "-g", "-c", cb], capture_output=True, text=True).stdout
    lines = sass.split("\n")
    for i, l in enumerate(lines):
        if l.startswith("//----") and kern in l:
            start = i
            break
    if start is not None:
        break
off2line = {}
curline = "?"
for l in lines[start + 1:]:
    if l.startswith("//----"):
        break
    m = re.search(r'line (\d+)', l)
    if "//## File" in l and m:
        curline = int(m.group(1))
    m2 = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if m2:
        off2line[int(m2.group(1), 16)] = curline
agg = collections.defaultdict(lambda: [0.0, 0.0])
for r in data:
    off = int(r[idx["Address"]], 16) - base
    ln = off2line.get(off, "?")
    agg[ln][0] += float(r[idx["Instructions Executed"]] or 0)
    agg[ln][1] += float(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
ti = sum(v[0] for v in agg.values())
ts = sum(v[1] for v in agg.values())
print(f"kernel {blk['name'][:80]}  instr {ti:.3e}  samples {ts:.0f}")
src = {}
srcpath = "/root/repo/paper_1804_09152_b200/csrc/ft_step.cu"
if os.path.exists(srcpath):
    src = {i + 1: t for i, t in enumerate(open(srcpath).read().split("\n"))}
for ln, (ie, ss) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{str(ln):>5} instr {100*ie/ti:5.1f}%  stall {100*ss/max(ts,1):5.1f}%  {src.get(ln, '').strip()[:90]}")
