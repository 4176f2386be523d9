"""One prepare + a short registration of a config (for ncu captures of the secondary kernels: kNN / surface
fit, em_tail / moments, Newton).  python tools/secondary_once.py CONFIG [ITERS]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_2103_15039_b200 as lsg
cfg = sys.argv[1]
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
wl = synth.make(cfg)
tgt = lsg.prepare_target(torch.from_numpy(wl.target).cuda(), wl.knn_k)
X = torch.from_numpy(wl.source).cuda()
out = lsg.Registrar(tgt, X, iters)(w=wl.w)
torch.cuda.synchronize()
print(cfg, wl.M, wl.N, iters, out["iters"], float(out["sigma2"]))
