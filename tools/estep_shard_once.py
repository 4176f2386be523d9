"""One warm-up and one measured lsgcpd_estep of a source shard (N/G points) of a config against the whole
target, for ncu DRAM-byte captures of the per-rank E step at world size G.
python tools/estep_shard_once.py CONFIG G"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_15039_b200 as lsg  # noqa: E402
import synth  # noqa: E402
from paper_2103_15039_b200.dist import shard_range  # noqa: E402

name, G = sys.argv[1], int(sys.argv[2])
wl = synth.make(name)
lo, hi = shard_range(wl.N, 0, G)
tgt = lsg.prepare_target(torch.from_numpy(wl.target).cuda(), wl.knn_k)
X = torch.from_numpy(wl.source[lo:hi].copy()).cuda()
run = lsg.EstepRunner(tgt, X)
for _ in range(2):
    run(wl.R_expected, wl.t_expected, 0.02, wl.w)
torch.cuda.synchronize()
print(name, G, hi - lo)
