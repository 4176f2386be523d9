"""Which E-step kernel serves a single small registration fastest: time per EM iteration of lsgcpd_register on
desk-corner problems of n points (synth.make_batch) for the CUDA-core variants and the tensor-core kernel.
Each configuration runs in its own process with LSGCPD_TC / LSGCPD_ESTEP_VARIANT set (read once by the library;
the loop at the bottom): CUDA-core configurations 0/1/2 = 768/512/64-point blocks."""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if len(sys.argv) > 1 and sys.argv[1] == "run":
    import torch, synth
    import paper_2103_15039_b200 as lsg
    out = []
    for n in (1000, 2000, 3500, 5000, 7000, 9500):
        wls = synth.make_batch(4, n, seed=31)
        regs = [lsg.Registrar(lsg.prepare_target(torch.from_numpy(w.target).cuda(), w.knn_k),
                              torch.from_numpy(w.source).cuda(), 50) for w in wls]
        for r in regs: r(w=0.1)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(5):
            for r in regs: r(w=0.1)
        e1.record(); torch.cuda.synchronize()
        out.append(f"{e0.elapsed_time(e1) / 20 / 50 * 1e3:6.1f}")
    print(os.environ.get("TAG", ""), " ".join(out), flush=True)
else:
    print("us per EM iteration for n = 1000 2000 3500 5000 7000 9500")
    for tag, env in (("auto", {}), ("tc", {"LSGCPD_TC": "1"}),
                     *[(f"v{v}", {"LSGCPD_TC": "0", "LSGCPD_ESTEP_VARIANT": str(v)}) for v in (2, 1, 0)]):
        subprocess.run([sys.executable, __file__, "run"], env=dict(os.environ, TAG=f"{tag:5s}", **env))
