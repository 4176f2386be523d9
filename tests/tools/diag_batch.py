import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import oracle, synth
from oracle import se3
import paper_2103_15039_b200 as lsg
def dev(a): return torch.from_numpy(np.ascontiguousarray(a)).cuda()
wls = synth.make_batch(4, int(os.environ.get("NPTS", "600")), seed=11)
preps = []
for w in wls:
    tgt, ann = lsg.prepare_target(dev(w.target), w.knn_k, annotations=True)
    preps.append((tgt, {"Y": w.target.astype(np.float64), "normals": ann["normals"].cpu().numpy().astype(np.float64),
                        "alpha": ann["alpha"].cpu().numpy().astype(np.float64)}))
rng = np.random.default_rng(4)
confs = [rng.uniform(0.3, 1.0, w.N).astype(np.float32) for w in wls]
kw = dict(eta=0.1, sigma2_init=float(os.environ.get("S2I", "1e-3")))
ITERS = int(os.environ.get("ITERS", "20"))
res = {}
for mode in ("1", "0"):
    lsg.set_option("tc", int(mode))
    res["batch_tc" + mode] = lsg.register_batch([p[0] for p in preps], [dev(w.source) for w in wls], ITERS,
                                                src_confs=[dev(c) for c in confs], **kw)
for b in range(4):
    tgt, t64 = preps[b]
    ora = oracle.register(t64, wls[b].source, 0.0, ITERS, tgt.volume, tgt.extent, sigma2_0=kw["sigma2_init"] or None, eta=0.1,
                          phi_x=confs[b].astype(np.float64))
    line = f"b={b}"
    for k, out in res.items():
        line += f"  {k}: {se3.rotation_angle(out['R'][b].T @ ora['R']):.2e}"
    for mode in ("1", "0"):
        lsg.set_option("tc", int(mode))
        s = lsg.register(tgt, dev(wls[b].source), ITERS, src_conf=dev(confs[b]), **kw)
        line += f"  single_tc{mode}: {se3.rotation_angle(s['R'].T @ ora['R']):.2e}"
    print(line, flush=True)
