import numpy as np, torch, time, sys
sys.path.insert(0, '.')
import oracle, synth
import paper_2103_15039_b200 as lsg
from tests.parity import record_errors
wl = synth.make('tiny')
tg = oracle.prepare_target(wl.target, 10)
n32 = tg['normals'].astype(np.float32); a32 = tg['alpha'].astype(np.float32)
V, ext = oracle.working_volume(wl.target)
tgt = lsg.pack_target(torch.from_numpy(wl.target).cuda(), torch.from_numpy(n32).cuda(), torch.from_numpy(a32).cuda())
print('packed', tgt.volume, V, tgt.extent, ext)
for s2 in (1e-2, 1e-4):
    for w in (0.1, 0.0):
        rec = lsg.estep(tgt, torch.from_numpy(wl.source).cuda(), wl.R_expected, wl.t_expected, s2, w, V)
        torch.cuda.synchronize()
        rec = rec.cpu().numpy()
        ora = oracle.estep(wl.target, n32.astype(np.float64), a32.astype(np.float64), wl.source, wl.R_expected, wl.t_expected, s2, w, V)
        err = record_errors(rec, ora, wl.target, a32)
        print('s2', s2, 'w', w, 'max err per col', np.array2string(err.max(0), precision=1))
t0=time.time()
out = lsg.register(tgt, torch.from_numpy(wl.source).cuda(), 50, w=0.1, volume=V, traces=True)
print('register', time.time()-t0, out['R'], out['t'], out['sigma2'], out['iters'], out['status'])
print('expected', wl.R_expected, wl.t_expected)
