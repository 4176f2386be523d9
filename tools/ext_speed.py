"""Model extensions measured like the base path: registration time per EM iteration
with the uniform w, with w from the outlier ratio η (Eq. 7), with per-point confidences (Eq. 8, w_n) and with
the affine group, on the object and rgbd configs.  Graphs warmed up; events around whole calls."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_2103_15039_b200 as lsg

for cfg in ("object", "rgbd"):
    wl = synth.make(cfg)
    tgt = lsg.prepare_target(torch.from_numpy(wl.target).cuda(), wl.knn_k)
    X = torch.from_numpy(wl.source).cuda()
    conf = lsg.depth_confidence(X) if cfg == "rgbd" else torch.rand(wl.N, device="cuda", generator=torch.Generator("cuda").manual_seed(5))
    reg = lsg.Registrar(tgt, X, wl.iters)
    variants = (("uniform w", dict(w=wl.w)), ("eta=0.1 (Eq. 7)", dict(eta=0.1)),
                ("w_n from phi (Eq. 8)", dict(w=wl.w, src_conf=conf)), ("affine group", dict(w=wl.w, group="affine")))
    for name, kw in variants:
        reg(**kw); torch.cuda.synchronize()
        reps = 5 if cfg == "object" else 2
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(reps):
            out = reg(**kw)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        print(f"{cfg:6s} {name:22s}: {ms:8.2f} ms per registration, {ms / wl.iters * 1e3:8.1f} us/iteration, "
              f"status {out['status']}, iters {out['iters']}", flush=True)
