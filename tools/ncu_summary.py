"""Key metrics of every kernel in an ncu report (details page)."""
import csv, io, subprocess, sys
keys = ('Duration', 'DRAM Throughput', 'Memory Throughput', 'Executed Ipc Active', 'Achieved Occupancy',
        'Registers Per Thread', 'L1/TEX Hit Rate', 'L2 Hit Rate', 'Warp Cycles Per Issued Instruction',
        'Executed Instructions', 'Theoretical Occupancy', 'Compute (SM) Throughput', 'Issue Slots Busy',
        'Avg. Active Threads Per Warp', 'Block Limit Shared Mem', 'Block Limit Registers')
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h = r[0]
cur = None
for row in r[1:]:
    d = dict(zip(h, row))
    if d.get("Kernel Name") != cur:
        cur = d.get("Kernel Name")
        print("==", cur[:100])
    if d.get("Metric Name") in keys:
        print(f"   {d['Metric Name']:40s} {d['Metric Value']} {d.get('Metric Unit','')}")
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h = r[0]
for v in r[2:]:
    st = {k: x for k, x in zip(h, v) if 'pcsamp_warps_issue_stalled' in k and not k.endswith('not_issued')}
    tot = sum(float(x) for x in st.values() if x.replace('.', '').isdigit())
    print("   stalls:", ", ".join(f"{k.split('stalled_')[1]} {100*float(x)/tot:.0f}%" for k, x in sorted(st.items(), key=lambda kv: -float(kv[1] or 0))[:8] if tot))
    for k, x in zip(h, v):
        if k in ('dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_bytes.sum', 'l1tex__t_bytes.sum'):
            print(f"   {k} {x}")
