"""Registration time per iteration vs newton_max (tiny/object): the single-warp FP64 Newton kernel's share."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_2103_15039_b200 as lsg
for cfg in ("tiny", "object"):
    wl = synth.make(cfg)
    tgt = lsg.prepare_target(torch.from_numpy(wl.target).cuda(), wl.knn_k)
    X = torch.from_numpy(wl.source).cuda()
    reg = lsg.Registrar(tgt, X, wl.iters)
    for nm in (0, 1, 3, 10):
        reg(w=wl.w, newton_max=nm); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(5):
            reg(w=wl.w, newton_max=nm)
        e1.record(); torch.cuda.synchronize()
        print(f"{cfg} newton_max={nm:2d}: {e0.elapsed_time(e1) / 5 / wl.iters * 1e3:7.1f} us/iter", flush=True)
