"""Per-source-line executed instructions and stall samples of each kernel in
an ncu report: python tools/ncu_src.py report.ncu-rep [kernel-substring] [top]"""
import collections, csv, io, subprocess, sys
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
want = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
agg = collections.defaultdict(collections.Counter)
stall = collections.defaultdict(collections.Counter)
src = {}
fn = fname = hdr = cur = None
for r in csv.reader(io.StringIO(raw)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        fn = r[1]
        continue
    if r[0] == "Line No":
        hdr = {k: i for i, k in enumerate(r)}
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0]:
        cur = (fname, int(r[0]))
        src[cur] = r[1].strip()[:95]
    try:
        n = float(r[hdr["Instructions Executed"]] or 0)
        sm = float(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)
    except (ValueError, KeyError):
        continue
    agg[fn][cur] += n
    stall[fn][cur] += sm
for fn in agg:
    if want not in fn:
        continue
    tot = sum(agg[fn].values())
    ts = sum(stall[fn].values()) or 1
    print(f"===== {fn}  instructions {tot:.0f}")
    for k, n in agg[fn].most_common(top):
        print(f"{n:11.0f} {100 * n / tot:5.1f}%  st {100 * stall[fn][k] / ts:5.1f}%  {k[0]}:{k[1]:<5} {src.get(k, '')}")
