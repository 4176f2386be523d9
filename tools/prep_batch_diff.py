"""Where lsgcpd_prepare_batch and lsgcpd_prepare_target differ (diagnostic): per target, the differing bytes per
section (header, body, tensor-core section, slots).  python tools/prep_batch_diff.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_15039_b200 as lsg  # noqa: E402
import synth  # noqa: E402

clouds = [w.target for w in synth.make_batch(3, 900, seed=5, ragged=True)]
rng = np.random.default_rng(2)
clouds.append(np.concatenate([rng.normal(0, 0.02, (800, 3)), rng.uniform(-20, 20, (60, 3))]).astype(np.float32))
clouds.append(synth.make("tiny").target)
dev = [torch.from_numpy(c).cuda() for c in clouds]
batch = lsg.prepare_batch(dev, 10)
for i, (c, tb) in enumerate(zip(dev, batch)):
    ts = lsg.prepare_target(c, 10)
    a, b = tb.buf.cpu().numpy(), ts.buf.cpu().numpy()
    M = tb.M
    M_pad = (M + 255) // 256 * 256
    hdr, body = 256, 256 + M_pad * 64
    tc = body + (M_pad // 64) * 10240
    for name, lo, hi in (("header", 0, hdr), ("body", hdr, body), ("tc", body, tc), ("slots", tc, len(a))):
        d = np.nonzero(a[lo:hi] != b[lo:hi])[0]
        print(f"target {i} M={M} {name:6s}: {len(d)} bytes differ" + (f", first at +{d[0]}" if len(d) else ""))
    # the permutation and the per-target fields
    sa = a[tc:].view(np.int32)[:M]
    sb = b[tc:].view(np.int32)[:M]
    print(f"   slots equal: {np.array_equal(sa, sb)}")
