"""Summarise tools/microbench/run_pipes.sh output into profiles/microbench_peaks.json: the best FFMA2 lane-op
rate and MUFU.EX2 rate per second over the runs, the in-kernel clock estimate and the sampled SM clocks.
python tools/microbench/pipes_summary.py gpurun_out/TAG [profiles/microbench_peaks.json]"""
import json
import re
import statistics
import sys

d = sys.argv[1]
out = sys.argv[2] if len(sys.argv) > 2 else "profiles/microbench_peaks.json"
best, mhz = {}, {}
for ln in open(f"{d}/pipes.txt"):
    m = re.match(r"(\w+)\s+blocks=(\d+).*?([\d.e+]+) ops/s.*=> (\d+) MHz", ln)
    if m:
        name, rate, f = m.group(1), float(m.group(3)), float(m.group(4))
        if rate > best.get(name, 0):
            best[name], mhz[name] = rate, f
clk = []
for ln in open(f"{d}/pipes_clocks.csv"):
    p = [x.strip() for x in ln.split(",")]
    try:
        clk.append(float(p[0]))
    except (ValueError, IndexError):
        pass
res = {"ffma2_lane_ops_per_s": best.get("ffma2"), "ffma_lane_ops_per_s": best.get("ffma"),
       "ex2_per_s": best.get("ex2"),
       "in_kernel_mhz_lower_bound": {k: mhz[k] for k in ("ffma2", "ex2") if k in mhz},
       "sampled_sm_mhz": {"median": statistics.median(clk) if clk else None, "max": max(clk) if clk else None,
                          "samples": len(clk)},
       "note": "in_kernel_mhz_lower_bound = mean block clock64 span / launch wall time (blocks do not span the whole "
               "launch, so it is a lower bound); sampled_sm_mhz is the nvidia-smi clock during the runs",
       "how": "tools/microbench/run_pipes.sh: best of 15 runs x {2,4} blocks/SM of 256 threads, 8 independent chains; "
              "ex2 kernel = 1 MUFU.EX2 + 1 FMUL per element (MUFU-bound)"}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
