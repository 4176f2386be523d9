"""Time lsgcpd_estep (CUDA events on its stream) on a config at the σ² of a short registration's end and at σ²₀;
prints pairs/s per residual mode.  With LSGCPD_LIB=<diag .so> it times a diagnostic build.
python tools/estep_time.py [config] [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_15039_b200 as lsg  # noqa: E402
import synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "scale"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
wl = synth.make(name)
tgt = lsg.prepare_target(torch.from_numpy(wl.target).cuda(), wl.knn_k)
X = torch.from_numpy(wl.source).cuda()
run = lsg.EstepRunner(tgt, X)
tag = os.path.basename(os.environ.get("LSGCPD_LIB", "product"))
for s2 in (0.02, 0.14):
    run(wl.R_expected, wl.t_expected, s2, wl.w)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        run(wl.R_expected, wl.t_expected, s2, wl.w)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"{tag:24s} {name} sigma2 {s2:.3g}: {ms:9.3f} ms/E step  {wl.M * wl.N / ms * 1e3:.4e} pairs/s", flush=True)
