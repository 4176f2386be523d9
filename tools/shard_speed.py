"""Per-rank work of the sharded scale registration: lsgcpd_register on the source shard rank 0 of G ranks
would own (contiguous N/G points, full target), timed on one GPU.  With the per-iteration all-reduce of 75
doubles (~10-30 µs over NVLink, not included) this bounds the strong-scaling efficiency T1 / (G · T_G)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_2103_15039_b200 as lsg
from paper_2103_15039_b200.dist import shard_range
wl = synth.make(os.environ.get("CFG", "scale"))
tgt = lsg.prepare_target(torch.from_numpy(wl.target).cuda(), wl.knn_k)
res = {}
for G in (1, 2, 4, 8):
    lo, hi = shard_range(wl.N, 0, G)
    X = torch.from_numpy(np.ascontiguousarray(wl.source[lo:hi])).cuda()
    reg = lsg.Registrar(tgt, X, wl.iters)
    reg(w=wl.w); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(2):
        reg(w=wl.w)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 2
    res[G] = ms
    eff = res[1] / (G * ms)
    print(f"G={G}: shard N={hi - lo}: {ms:9.1f} ms per registration ({wl.iters} iters)  "
          f"{wl.M * (hi - lo) * wl.iters / ms * 1e3:.3e} pairs/s per rank  efficiency bound {eff:.3f}", flush=True)
