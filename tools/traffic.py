"""profiles/step_kernel_traffic.json from an ncu DRAM capture of the step's
column kernels (the `traffic` figure bench.py reports beside the roofline):

    ncu --profile-from-start off --cache-control none --clock-control none \\
        --metrics dram__bytes_read.sum,dram__bytes_write.sum \\
        -k regex:"prep_kernel|band_kernel|wide3_kernel|wide4_kernel|wide_kernel|finalize_kernel" \\
        --csv --log-file traffic.csv python tools/prof_window.py --steps 8
    python tools/traffic.py traffic.csv 8 > profiles/step_kernel_traffic.json

The engine hash is bench.py's (the step sources), so bench.py uses the file
only for the build it was measured on."""
import collections, csv, hashlib, json, os, sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
h = hashlib.sha256()
for f in ("ft_step.cu", "ft_arith.cuh", "ft_common.cuh"):
    h.update(open(os.path.join(REPO, "paper_1804_09152_b200", "csrc", f), "rb").read())
steps = int(sys.argv[2])
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
tot = collections.Counter()
per_kernel = collections.defaultdict(collections.Counter)
for r in rows:
    if r and r[0] == "ID":
        hdr = {k: i for i, k in enumerate(r)}
        continue
    if not hdr or len(r) < len(hdr):
        continue
    name, unit, val = r[hdr["Kernel Name"]].split("(")[0], r[hdr["Metric Unit"]], float(r[hdr["Metric Value"]])
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    m = r[hdr["Metric Name"]]
    tot[m] += val * scale
    per_kernel[name][m] += val * scale / steps
rd, wr = tot["dram__bytes_read.sum"] / steps, tot["dram__bytes_write.sum"] / steps
print(json.dumps({
    "engine_hash": h.hexdigest()[:16], "precision": "exact", "n_vertices": 10000000, "seeds": 4096,
    "dram_bytes_per_step": rd + wr, "dram_read_bytes": rd, "dram_write_bytes": wr,
    "per_kernel": {k: {"read": v["dram__bytes_read.sum"], "write": v["dram__bytes_write.sum"]}
                   for k, v in per_kernel.items()},
    "kernels": "one step's kernels: prep, band, wide3, wide4, wide, finalize (with the deep pass)",
    "window": f"C3 steps 83..{82 + steps} (tools/prof_window.py)",
    "note": "ncu --cache-control none: L2 carries over between kernels as in the pipeline; per step, "
            "averaged over the window"}, indent=1))
