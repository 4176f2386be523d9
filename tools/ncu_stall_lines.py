"""Per-SASS-line stall breakdown of an ncu report (source page): the top lines by samples with their dominant stall
reasons, and the stall totals split by instruction execution count class (e.g. the pair loop vs the helper warps).
python tools/ncu_stall_lines.py <report.ncu-rep> [top N]"""
import csv
import subprocess
import sys
from collections import Counter, defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout.splitlines()
rows = list(csv.reader(out))
hdr, data = rows[1], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]


def num(r, h):
    v = r[ix[h]].replace(",", "")
    return int(v) if v.isdigit() else 0


lines = [r for r in data if num(r, "Warp Stall Sampling (All Samples)") > 0]
tot = sum(num(r, "Warp Stall Sampling (All Samples)") for r in lines)
print(f"total samples {tot}")
for r in sorted(lines, key=lambda r: -num(r, "Warp Stall Sampling (All Samples)"))[:top]:
    s = num(r, "Warp Stall Sampling (All Samples)")
    rs = sorted(((num(r, h), h[6:]) for h in reasons), reverse=True)[:3]
    print(f"{s:8d} {num(r, 'Instructions Executed'):11d}  {r[ix['Source']][:60]:60s} " +
          " ".join(f"{n}:{v}" for v, n in rs if v))
by_exec = defaultdict(Counter)
for r in lines:
    e = num(r, "Instructions Executed")
    for h in reasons:
        by_exec[e][h[6:]] += num(r, h)
print("\nstall totals by execution-count class (top classes):")
for e, c in sorted(by_exec.items(), key=lambda kv: -sum(kv[1].values()))[:8]:
    t = sum(c.values())
    print(f"  exec {e:11d}: {t:8d} ({t / tot:5.1%})  " + " ".join(f"{k}:{v / t:.0%}" for k, v in c.most_common(5)))
