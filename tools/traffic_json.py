"""Sum DRAM bytes per lsgcpd_estep call from ncu metric CSVs (tools/runs: one per world size G) into
profiles/estep_dram_bytes.json {"workload", "by_n_gpus": {G: bytes}}.  python tools/traffic_json.py DIR WORKLOAD"""
import csv
import glob
import json
import os
import re
import sys

d, wl = sys.argv[1], sys.argv[2]
out = {"workload": wl, "by_n_gpus": {}, "per_kernel": {},
       "how": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum on the second lsgcpd_estep call of a rank's "
              "source shard (tools/estep_shard_once.py CONFIG G; every kernel of the call summed), one B200"}
for f in sorted(glob.glob(os.path.join(d, "dram_G*.csv"))):
    G = re.search(r"dram_G(\d+)", f).group(1)
    rows = [r for r in csv.reader(open(f)) if len(r) > 10]
    h = rows[0]
    ik, im, iu, iv = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
    tot, per = 0.0, {}
    for r in rows[1:]:
        v = float(r[iv].replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(r[iu], 1)
        tot += v
        k = r[ik].split("(")[0].replace("void ", "")
        per[k] = per.get(k, 0.0) + v
    out["by_n_gpus"][G] = tot
    out["per_kernel"][G] = per
json.dump(out, open("profiles/estep_dram_bytes.json", "w"), indent=1)
print(json.dumps(out, indent=1))
