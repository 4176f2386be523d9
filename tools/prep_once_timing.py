"""lsgcpd_prepare_target wall time, call by call (diagnostic: first-call and allocator effects).
python tools/prep_once_timing.py [config] [calls]"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_15039_b200 as lsg  # noqa: E402
import synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "object"
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 8
wl = synth.make(name)
Y = torch.from_numpy(wl.target).cuda()
for i in range(calls):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tg = lsg.prepare_target(Y, wl.knn_k)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    X = torch.from_numpy(wl.source).cuda()
    run = lsg.EstepRunner(tg, X)
    for _ in range(20):
        run(wl.R_expected, wl.t_expected, 1e-3, wl.w)
    torch.cuda.synchronize()
    print(f"{name} call {i}: prepare_target {(t1 - t0) * 1e3:8.2f} ms", flush=True)
