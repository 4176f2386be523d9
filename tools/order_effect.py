"""E-step time on a config with the source as given vs Z-ordered (lsgcpd_estep; far rule on).  Diagnostic."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_15039_b200 as lsg  # noqa: E402
import synth  # noqa: E402
from tools.far_rule_probe import morton_order  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "scale"
wl = synth.make(name)
tgt = lsg.prepare_target(torch.from_numpy(wl.target).cuda(), wl.knn_k)
for rep in range(2):
    for order in ("given", "morton"):
        S = wl.source if order == "given" else wl.source[morton_order(wl.source)]
        run = lsg.EstepRunner(tgt, torch.from_numpy(np.ascontiguousarray(S)).cuda())
        for s2 in (0.02,):
            run(wl.R_expected, wl.t_expected, s2, wl.w)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            for _ in range(5):
                run(wl.R_expected, wl.t_expected, s2, wl.w)
            e1.record()
            torch.cuda.synchronize()
            print(f"{name} source {order:6s}: {e0.elapsed_time(e1) / 5:9.3f} ms per E step", flush=True)
