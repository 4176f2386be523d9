"""Fixed cost of one lsgcpd_register call (setup, σ²₀, graph capture + instantiate, result copies) vs per-iteration
cost: time per call for max_iters = 1, 2, 10, 50 on small problems."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_2103_15039_b200 as lsg
for cfg in ("tiny", "object"):
    wl = synth.make(cfg)
    tgt = lsg.prepare_target(torch.from_numpy(wl.target).cuda(), wl.knn_k)
    X = torch.from_numpy(wl.source).cuda()
    for it in (1, 2, 10, 50):
        reg = lsg.Registrar(tgt, X, it)
        reg(w=wl.w); torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(20):
            reg(w=wl.w)
        torch.cuda.synchronize()
        print(f"{cfg:6s} max_iters={it:3d}: {(time.perf_counter() - t0) / 20 * 1e6:9.1f} us per call", flush=True)
