"""Summarise an ncu report: key metrics, stall reasons, top stalled SASS lines, per-region sample shares."""
import csv, subprocess, sys
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(raw))
d = dict(zip(rows[0], rows[2]))
keys = ['gpu__time_duration.sum', 'launch__registers_per_thread', 'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active', 'sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active', 'smsp__inst_executed.sum', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'dram__bytes_read.sum', 'dram__bytes_write.sum']
for k in keys:
    print(f"{k:70s} {d.get(k)}")
for h, v in zip(rows[0], rows[2]):
    if h.startswith('smsp__pcsamp_warps_issue_stalled') and not h.endswith('not_issued'):
        try:
            if int(v.replace(',', '')) > 20000:
                print(f"  {h[33:]:40s} {v}")
        except ValueError:
            pass
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(src))
hdr = rows[1]; data = rows[2:]
isrc, istall, iexec = hdr.index('Source'), hdr.index('Warp Stall Sampling (All Samples)'), hdr.index('Instructions Executed')
tot = sum(int(r[istall]) for r in data if r[istall].isdigit())
print("total samples", tot)
for r in sorted([r for r in data if r[istall].isdigit()], key=lambda r: -int(r[istall]))[:int(sys.argv[2]) if len(sys.argv) > 2 else 12]:
    print(r[istall].rjust(8), r[iexec].rjust(12), r[isrc][:90])
