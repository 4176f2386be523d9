"""Five EM iterations of the tiny and object registrations (a short program to capture with ncu)."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch, synth
import paper_2103_15039_b200 as lsg
for cfg in ("tiny", "object"):
    wl = synth.make(cfg)
    tgt = lsg.prepare_target(torch.from_numpy(wl.target).cuda(), wl.knn_k)
    X = torch.from_numpy(wl.source).cuda()
    reg = lsg.Registrar(tgt, X, 5)
    out = reg(w=wl.w)
torch.cuda.synchronize()
