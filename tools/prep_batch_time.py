"""lsgcpd_prepare_batch wall time, repeated (host launch cost vs device time), for B problems of n points.
python tools/prep_batch_time.py [B] [n] [reps]"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_15039_b200 as lsg  # noqa: E402
import synth  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 550
n = int(sys.argv[2]) if len(sys.argv) > 2 else 3500
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
wls = synth.make_batch(B, n)
clouds = [torch.from_numpy(w.target).cuda() for w in wls]
lsg.prepare_batch(clouds, wls[0].knn_k)
torch.cuda.synchronize()
for r in range(reps):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    t0 = time.perf_counter()
    e0.record()
    tg = lsg.prepare_batch(clouds, wls[0].knn_k)
    e1.record()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    print(f"prepare_batch B={B} n={n}: wall {(t1 - t0) * 1e3:8.1f} ms  device span {e0.elapsed_time(e1):8.1f} ms",
          flush=True)
    del tg
