"""Registration wall time per config through lsgcpd_register (CUDA graph), vs E-step time × iterations."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
import paper_2103_15039_b200 as lsg
for cfg in os.environ.get("CFGS", "tiny,object,rgbd,lidar").split(","):
    wl = synth.make(cfg)
    tgt = lsg.prepare_target(torch.from_numpy(wl.target).cuda(), wl.knn_k)
    X = torch.from_numpy(wl.source).cuda()
    reg = lsg.Registrar(tgt, X, wl.iters)
    out = reg(w=wl.w)
    torch.cuda.synchronize()
    reps = 20 if wl.M < 20000 else 2
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        out = reg(w=wl.w)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    run = lsg.EstepRunner(tgt, X)
    run(out["R"], out["t"], out["sigma2"], wl.w); torch.cuda.synchronize()
    e0.record()
    for _ in range(reps * 4):
        run(out["R"], out["t"], out["sigma2"], wl.w)
    e1.record(); torch.cuda.synchronize()
    es = e0.elapsed_time(e1) / (reps * 4)
    Yd = torch.from_numpy(wl.target).cuda()
    tps = []
    for _ in range(3):   # the fastest of three calls: a single call can include a caching-allocator cudaMalloc
        torch.cuda.synchronize(); t0 = time.perf_counter()
        tg2 = lsg.prepare_target(Yd, wl.knn_k)
        torch.cuda.synchronize(); tps.append((time.perf_counter() - t0) * 1e3)
    tp = min(tps)
    print(f"{cfg:7s} M={wl.M} N={wl.N} iters={wl.iters}: register {ms:9.3f} ms  ({ms/wl.iters*1e3:8.1f} us/iter)  "
          f"E step {es*1e3:8.1f} us  -> E-step share {es*wl.iters/ms:5.1%}  prepare {tp:7.2f} ms  "
          f"pairs/s {wl.M*wl.N*wl.iters/ms*1e3:.3e}", flush=True)
