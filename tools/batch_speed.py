"""Throughput of batched small registrations (NEXT-3) vs one lsgcpd_register call per problem."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
import paper_2103_15039_b200 as lsg
B = int(os.environ.get("B", "550")); n = int(os.environ.get("NPTS", "3500")); iters = int(os.environ.get("ITERS", "50"))
wls = synth.make_batch(B, n)
clouds = [torch.from_numpy(w.target).cuda() for w in wls]
# each variant timed after a warm-up of itself, the previous variant's targets freed first (allocator state)
tgts = [lsg.prepare_target(c, w.knn_k) for c, w in zip(clouds, wls)]
del tgts
torch.cuda.synchronize(); t0 = time.perf_counter()
tgts = [lsg.prepare_target(c, w.knn_k) for c, w in zip(clouds, wls)]
torch.cuda.synchronize(); t_each = time.perf_counter() - t0
del tgts
tgts = lsg.prepare_batch(clouds, wls[0].knn_k)
del tgts
torch.cuda.synchronize(); t1 = time.perf_counter()
tgts = lsg.prepare_batch(clouds, wls[0].knn_k)
torch.cuda.synchronize(); t2 = time.perf_counter()
print(f"prepare {B} targets: {t_each * 1e3:.1f} ms one call each, {(t2 - t1) * 1e3:.1f} ms in one lsgcpd_prepare_batch",
      flush=True)
srcs = [torch.from_numpy(w.source).cuda() for w in wls]
reg = lsg.BatchRegistrar(tgts, srcs, iters)
reg(w=0.1); torch.cuda.synchronize()
t0 = time.perf_counter(); out = reg(w=0.1); torch.cuda.synchronize(); dt = time.perf_counter() - t0
pairs = sum(w.M * w.N for w in wls) * iters
ang = [np.degrees(np.arccos(np.clip((np.trace(out["R"][b].T @ w.R_expected) - 1) / 2, -1, 1))) for b, w in enumerate(wls)]
print(f"batch B={B} n={n} iters={iters}: {dt*1e3:.1f} ms  {B/dt:.1f} registrations/s  {pairs/dt:.3e} pair-evals/s  "
      f"median rot err {np.median(ang):.3f} deg, {np.mean(np.array(ang) < 1.0)*100:.0f}% < 1 deg", flush=True)
K = min(B, int(os.environ.get("SEQ", "40")))
regs = [lsg.Registrar(tgts[b], srcs[b], iters) for b in range(K)]
for r in regs[:2]: r(w=0.1)
torch.cuda.synchronize(); t0 = time.perf_counter()
for r in regs: r(w=0.1)
torch.cuda.synchronize(); ds = time.perf_counter() - t0
print(f"sequential lsgcpd_register x{K}: {ds/K*1e3:.2f} ms each  {K/ds:.1f} registrations/s", flush=True)
