"""Potential of the far-point rule for the batched registrations (NEXT-3) with Morton-ordered sources: batch
time with the sources as generated and Z-ordered per problem, far rule off and on.  Diagnostic."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_15039_b200 as lsg  # noqa: E402
import synth  # noqa: E402
from tools.far_rule_probe import morton_order  # noqa: E402

B, n = 550, 3500
wls = synth.make_batch(B, n)
tgts = lsg.prepare_batch([torch.from_numpy(w.target).cuda() for w in wls], wls[0].knn_k)
for order in ("given", "morton"):
    srcs = [torch.from_numpy(np.ascontiguousarray(w.source if order == "given" else w.source[morton_order(w.source)])).cuda()
            for w in wls]
    for fr in (0, 1):
        with lsg.options(far_rule=fr):
            reg = lsg.BatchRegistrar(tgts, srcs, wls[0].iters)
            reg(w=0.1)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            for _ in range(3):
                reg(w=0.1)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 3
        print(f"batch sources {order:6s} far_rule={fr}: {ms:8.1f} ms  {B / ms * 1e3:7.1f} registrations/s", flush=True)
