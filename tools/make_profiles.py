"""Summarise a gpurun bench/profile run (tools/run_bench_profile.sh TAG=...) into profiles/ (tracked)."""
import collections, csv, json, shutil, subprocess, sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag, out = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else sys.argv[1]
G = os.path.join(ROOT, "gpurun_out"); P = os.path.join(ROOT, "profiles")
shutil.copy(os.path.join(G, f"bench_{tag}.json"), os.path.join(P, f"bench_{out}.json"))
rows = list(csv.reader(open(os.path.join(G, f"launches_{tag}.csv"))))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
hdr = rows[hi]; data = rows[hi + 1:]
kn, mv, mn = hdr.index('Kernel Name'), hdr.index('Metric Value'), hdr.index('Metric Name')
agg = collections.defaultdict(lambda: [0, 0.0])
for r in data:
    if len(r) > mv and r[mn] == 'gpu__time_duration.sum':
        agg[r[kn].split('(')[0]][0] += 1
        agg[r[kn].split('(')[0]][1] += float(r[mv].replace(',', ''))
tot = sum(v[1] for v in agg.values())
lines = ["ncu --metrics gpu__time_duration.sum --clock-control none --csv (cold-cache, serialised launches) of",
         "`python bench.py --steps 1 --warmup 1 --skip-cpu --skip-e2e --iters 3` on one B200 (" + out + ").",
         "Shares of GPU time per kernel (all launches of the command, including prepare and the roofline probe):", "",
         f"{'kernel':72s} {'launches':>8s} {'total ms':>12s} {'share':>8s}"]
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    lines.append(f"{k[:72]:72s} {n:8d} {t/1e6:12.3f} {100*t/tot:7.2f}%")
open(os.path.join(P, f"{out}_launches.txt"), "w").write("\n".join(lines) + "\n")
shutil.copy(os.path.join(G, f"launches_{tag}.csv"), os.path.join(P, f"{out}_launches.csv"))
rep = os.path.join(G, f"prof_estep_{tag}.ncu-rep")
if not os.path.exists(rep):   # launch list only (the E-step kernel's full capture is an earlier round's)
    print("\n".join(lines[:14]))
    sys.exit(0)
raw = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout.splitlines()))
d = dict(zip(raw[0], raw[2])); u = dict(zip(raw[0], raw[1]))
launches = [dict(zip(raw[0], r)) for r in raw[2:] if len(r) == len(raw[0])]   # every captured launch
keys = ['Kernel Name', 'gpu__time_duration.sum', 'launch__grid_size', 'launch__block_size', 'launch__registers_per_thread',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active', 'sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed',
        'sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active', 'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active', 'sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active',
        'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'smsp__inst_executed.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'sm__cycles_elapsed.avg.per_second']
txt = [f"{k:70s} {d.get(k, '?'):>24s} {u.get(k, '')}" for k in keys]
for h, v in zip(raw[0], raw[2]):
    if h.startswith('smsp__pcsamp_warps_issue_stalled') and not h.endswith('not_issued'):
        try:
            if int(v.replace(',', '')) > 10000:
                txt.append(f"  stall {h[33:]:40s} {v}")
        except ValueError:
            pass
open(os.path.join(P, f"{out}_estep_ncu_summary.txt"), "w").write(
    "ncu --set full --clock-control none --import-source on -k regex:" + os.environ.get("KREGEX", "estep_tc_kernel") + " -s 1 -c 1 on\n"
    "`python bench.py --steps 1 --warmup 1 --skip-cpu --skip-e2e --iters 3` (scale config, M=N=524288), one B200.\n\n"
    + "\n".join(txt) + "\n")
shutil.copy(rep, os.path.join(P, f"{out}_estep_full.ncu-rep"))
mult = {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9}
# one lsgcpd_estep call = one tensor-core launch per half of the targets (two on scale): the captured launches
# (consecutive halves) are summed
per = []
for x in launches:
    try:
        v = float(x['dram__bytes_read.sum'].replace(',', '')) * mult[u['dram__bytes_read.sum']] + \
            float(x['dram__bytes_write.sum'].replace(',', '')) * mult[u['dram__bytes_write.sum']]
    except ValueError:
        continue
    if v == v:   # ncu leaves some replays without DRAM counters (-nan)
        per.append(v)
HALVES = 2   # tensor-core launches per lsgcpd_estep call on scale (Sched::halves)
tr = sum(per) / len(per) * HALVES
json.dump({"workload": "scale", "n_gpus": 1, "kernel": d['Kernel Name'], "dram_bytes_per_launch": tr,
           "launches_per_estep": HALVES,
           "source": f"profiles/{out}_estep_ncu_summary.txt (dram__bytes_read.sum + dram__bytes_write.sum per "
                     f"tensor-core launch, mean of {len(per)} captured, x {HALVES} launches per lsgcpd_estep call)"},
          open(os.path.join(P, "estep_dram_bytes.json"), "w"), indent=1)
print("\n".join(lines[:12])); print("\n".join(txt))
