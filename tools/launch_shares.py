"""Share of GPU time per kernel from an ncu launch list (--metrics gpu__time_duration.sum --csv).
python tools/launch_shares.py LAUNCHES.csv [...]"""
import collections
import csv
import sys


def shares(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    h = rows[0]
    ik, im, iv = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    iu = h.index("Metric Unit")
    tot = collections.Counter()
    cnt = collections.Counter()
    for r in rows[1:]:
        if r[im] != "gpu__time_duration.sum":
            continue
        v = float(r[iv].replace(",", ""))
        v *= {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(r[iu], 1.0)
        name = r[ik].split("(")[0].split("<")[0].replace("void ", "").replace("lsg::", "")
        tot[name] += v
        cnt[name] += 1
    T = sum(tot.values())
    print(f"== {path}: {sum(cnt.values())} launches, {T:.1f} us of kernel time")
    for k, v in tot.most_common():
        print(f"  {k:34s} {cnt[k]:5d} launches {v:12.1f} us  {100 * v / T:6.2f} %")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        shares(p)
