#!/bin/bash
# Run a measurement command with the GPU clock sampled under load: nvidia-smi every 100 ms in the background,
# then append to the command's output a summary of the samples taken while the GPU was busy (utilization >= 50 %):
# median / min SM clock, max SM clock, throttle reasons seen.  Usage: tools/with_clocks.sh OUT.txt cmd args...
out=$1; shift
tmp=$(mktemp)
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,utilization.gpu,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv,noheader,nounits -lms 100 > $tmp 2>/dev/null &
smi=$!
"$@" > $out 2>&1
rc=$?
kill $smi 2>/dev/null; wait $smi 2>/dev/null
python3 - "$tmp" >> $out <<'PY'
import statistics, sys
rows = []
for ln in open(sys.argv[1]):
    p = [x.strip() for x in ln.split(",")]
    try:
        rows.append((float(p[0]), float(p[1]), float(p[2]), p[3:7]))
    except (ValueError, IndexError):
        pass
busy = [r for r in rows if r[2] >= 50]
label = ">= 50 %"
if not busy:   # short tools (e.g. prepare: ms-long kernels between host syncs) rarely fill a 100-ms window
    busy, label = [r for r in rows if r[2] > 0], "> 0 %"
names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
reasons = sorted({n for r in busy for n, v in zip(names, r[3]) if v.lower() == "active"})
if busy:
    sm = [r[0] for r in busy]
    print(f"# clocks under load: SM median {statistics.median(sm):.0f} MHz (min {min(sm):.0f}), max {max(r[1] for r in busy):.0f} MHz, "
          f"{len(busy)} of {len(rows)} 100-ms samples at {label} utilization; throttle reasons: {reasons or 'none'}")
else:
    print(f"# clocks under load: no sample at >= 50 % utilization ({len(rows)} samples)")
PY
rm -f $tmp
exit $rc
