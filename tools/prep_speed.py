"""Time lsgcpd_prepare_target per BASELINE config."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_2103_15039_b200 as lsg
for cfg in os.environ.get("CFGS", "object,rgbd,lidar,scale").split(","):
    wl = synth.make(cfg)
    Y = torch.from_numpy(wl.target).cuda()
    lsg.prepare_target(Y, wl.knn_k); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        lsg.prepare_target(Y, wl.knn_k)
    torch.cuda.synchronize()
    print(f"{os.environ.get('TAG','')} {cfg:7s} M={wl.M}: prepare {(time.perf_counter() - t0) / 3 * 1e3:8.2f} ms", flush=True)
