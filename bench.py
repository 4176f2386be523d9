#!/usr/bin/env python
"""Benchmark: LSG-CPD E-step pair evaluations/s on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config scale|batch|tiny|object|rgbd|lidar] [--replicas] [--impl reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (one process per GPU, NCCL)

A step is one full registration of the workload through the library (lsgcpd_register: σ²₀, then
`iters` EM iterations of E step → moments → NCCL all-reduce → SE(3) Newton + σ²) with the prepared
target and the source shard already resident in HBM.  value = M·N·iters·K / (max over ranks of the
device time of the K steps).  The source is sharded contiguously across ranks, the target is
replicated (strong scaling: the total problem is fixed).

`e2e` is the same metric through the public API from pinned HOST buffers: every step copies the
target and source shard host→device, prepares the target (kNN/normals/α on the GPU), registers and
returns R, t, σ² to the host.  `roofline` is for the dominant kernel (the fused E step), timed with
CUDA events around lsgcpd_estep on the launching stream.  `cpu_baseline` / `--impl reference` time the
FP64 CPU oracle (test infrastructure, never on the product path) on a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "E-step pair evals/s (M·N·iters/s) at 1/2/4/8 B200; % of MUFU/FP32 peak"
UNIT = "pair-evals/s"
SM_MAX_MHZ_FALLBACK = 1965.0
FLOPS_PER_PAIR = 47.0     # SURVEY §8(d).2 algorithmic FP32 flops per (m, n) pair (FMA = 2), + 1 exp
FP32_LANES_PER_SM = 128   # FP32 FMA lanes per SM per clock (B200)
MUFU_EX2_PER_SM = 16      # MUFU.EX2 results per SM per clock (B200 unit count)
# CUDA-core FP32 lane-operations per pair in the tensor-core E step's SASS: tile-centred residual
# 13 (r 3, ñ·r 3, τ 4, exponent 1, Σpτ 1, TF32 remainder of p 1), hi/lo residual 16 (r 6)
LANE_OPS_CENTRED, LANE_OPS_HILO = 13.0, 16.0
TILE_BYTES, TARGET_HDR = 10240, 256


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="scale")
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--skip-cpu", action="store_true", help="skip the cpu_baseline leg (profiling runs)")
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--iters", type=int, default=0, help="override EM iterations per step (0 = config's)")
    ap.add_argument("--replicas", action="store_true",
                    help="every rank registers the whole config on its own (no collective, weak scaling): "
                         "the SURVEY 8(d).3 'replicas' mode for the small configs")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def ensure_ranks(args):
    """`--gpus N` runs N ranks: under torchrun the environment must say WORLD_SIZE = N; launched plainly with
    N > 1, bench.py re-executes itself under torch.distributed.run with N processes (one per GPU), after checking
    that N GPUs are visible.  Any mismatch is an error (never a silent single-rank run)."""
    if "WORLD_SIZE" in os.environ:
        world = int(os.environ["WORLD_SIZE"])
        if world != args.gpus:
            sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
        return
    if args.gpus <= 1 or args.impl == "reference":
        return
    import socket
    import torch
    n = torch.cuda.device_count()
    if n < args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible GPUs, found {n}")
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    os.execv(sys.executable, cmd)


def centred_tile_share(target, sigma2: float, gate: float) -> float:
    """Share of the prepared target's 64-target tiles whose E_tile ≤ gate·σ (the tile-centred residual),
    read from the tile metadata of the tensor-core section (include/lsgcpd.h layout 2)."""
    import torch
    M_pad = (target.M + 255) // 256 * 256
    off = TARGET_HDR + M_pad * 16 * 4
    T = M_pad // 64
    raw = target.buf[off: off + T * TILE_BYTES].view(torch.float32).reshape(T, TILE_BYTES // 4)
    E = raw[:, 31].double().cpu().numpy()   # meta field (7) of target 3 of the tile
    return float(np.mean(E <= gate * np.sqrt(sigma2)))


def microbench_peaks():
    p = os.path.join(ROOT, "profiles", "microbench_peaks.json")
    try:
        return json.load(open(p))
    except Exception:
        return {}


def traffic_per_launch(workload: str, world: int):
    """DRAM bytes per lsgcpd_estep call of one rank (ncu, profiles/estep_dram_bytes.json) for this world size."""
    try:
        tj = json.load(open(os.path.join(ROOT, "profiles", "estep_dram_bytes.json")))
        if tj.get("workload") == workload:
            return tj.get("by_n_gpus", {}).get(str(world))
    except Exception:
        pass
    return None


def shard(n: int, rank: int, world: int):
    """Contiguous, balanced source shard [lo, hi) of rank `rank` (paper_2103_15039_b200.dist)."""
    from paper_2103_15039_b200.dist import shard_range
    return shard_range(n, rank, world)


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + self.FIELDS, "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(smax)), "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return json.load(f), "measured"
    except Exception:
        return {"sm_max_mhz": SM_MAX_MHZ_FALLBACK}, "fallback"


def cpu_oracle_rate(wl, target_sample_pts: int = 0, budget_s: float = 16.0):
    """FP64 oracle E step (C/OpenMP, all host cores) on a bounded sample of source points against the
    full target; returns (pairs/s, cores, sample description)."""
    import oracle
    rng = np.random.default_rng(0)
    tgt_n = rng.standard_normal(wl.target.shape)
    tgt_n /= np.linalg.norm(tgt_n, axis=1, keepdims=True)
    alpha = rng.uniform(0, 50, wl.M)
    V, _ = oracle.working_volume(wl.target)
    cores = int(oracle._lib.lib().ora_max_threads())
    # calibrate on a sample worth ~1 s, then size the sample for ~budget_s of CPU work
    n0 = int(np.clip(2e8 / wl.M, 8, wl.N))
    idx = rng.choice(wl.N, n0, replace=False)
    t0 = time.perf_counter()
    oracle.estep(wl.target, tgt_n, alpha, wl.source[idx], wl.R_expected, wl.t_expected, 1e-3, wl.w, V)
    dt = max(time.perf_counter() - t0, 1e-3)
    n = int(np.clip(n0 * budget_s / dt, 8, wl.N))
    idx = rng.choice(wl.N, n, replace=False)
    t0 = time.perf_counter()
    oracle.estep(wl.target, tgt_n, alpha, wl.source[idx], wl.R_expected, wl.t_expected, 1e-3, wl.w, V)
    dt = time.perf_counter() - t0
    return n * wl.M / dt, cores, f"oracle E step (FP64, OpenMP) for {n} sampled source points x all {wl.M} targets", dt


def run_reference(args, wl, rank):
    """--impl reference: the FP64 CPU oracle (E step + M step on a source sample) as it stands."""
    import oracle
    if rank != 0:
        return
    rng = np.random.default_rng(1)
    # seeded unit normals and α in [0, 50] (the annotation cost is not part of the E-step metric)
    normals = rng.standard_normal(wl.target.shape)
    normals /= np.linalg.norm(normals, axis=1, keepdims=True)
    alpha = rng.uniform(0, 50, wl.M)
    V, ext = oracle.working_volume(wl.target)
    cores = int(oracle._lib.lib().ora_max_threads())
    s = 256 if wl.M > 100000 else min(wl.N, 2048)
    idx = np.sort(rng.choice(wl.N, s, replace=False))
    X = wl.source[idx]
    R, t, s2 = np.eye(3), np.zeros(3), oracle.sigma2_init(X, wl.target)

    def step():
        nonlocal R, t, s2
        rec = oracle.estep(wl.target, normals, alpha, X, R, t, s2, wl.w, V)
        R, t, s2, _ = oracle.mstep(X, rec, R, t, s2, ext, 10, 1e-12 * ext * ext)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = time.perf_counter() - t0
    value = s * wl.M * args.steps / dt
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": wl.name, "M": wl.M, "N": wl.N, "w": wl.w, "sample_source_points": s},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"per step: oracle E step + M step for {s} sampled source points x all "
                                       f"{wl.M} targets"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


BATCH_B, BATCH_N, BATCH_ITERS = 550, 3500, 50


def batch_oracle_rate(wls, budget_s: float = 12.0):
    """The FP64 oracle E step on whole batch problems, one after another, until ~budget_s of CPU work."""
    import oracle
    cores = int(oracle._lib.lib().ora_max_threads())
    rng = np.random.default_rng(0)
    pairs, t_all, used = 0.0, 0.0, 0
    for wl in wls:
        n = rng.standard_normal(wl.target.shape)
        n /= np.linalg.norm(n, axis=1, keepdims=True)
        a = rng.uniform(0, 50, wl.M)
        V, _ = oracle.working_volume(wl.target)
        t0 = time.perf_counter()
        oracle.estep(wl.target, n, a, wl.source, wl.R_expected, wl.t_expected, 1e-3, wl.w, V)
        t_all += time.perf_counter() - t0
        pairs += float(wl.M) * wl.N
        used += 1
        if t_all >= budget_s:
            break
    return pairs / t_all, cores, f"oracle E step (FP64, OpenMP) on {used} whole problems of the batch", t_all


def run_batch(args, rank, world, local):
    """--config batch: 550 desk-corner problems of 3,500 points, 50 EM iterations, all
    registered by lsgcpd_register_batch; under torchrun each rank takes a contiguous share of the problems
    (replicas only: no collective).  value = pair evaluations of all ranks' problems per second."""
    import torch
    import torch.distributed as dist
    import synth
    import paper_2103_15039_b200 as lsg
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    wls = synth.make_batch(BATCH_B, BATCH_N)
    b0, b1 = shard(BATCH_B, rank, world)
    mine = wls[b0:b1]
    iters = args.iters or BATCH_ITERS
    tgts = lsg.prepare_batch([torch.from_numpy(w.target).to(dev) for w in mine], mine[0].knn_k)
    srcs = [torch.from_numpy(w.source).to(dev) for w in mine]
    reg = lsg.BatchRegistrar(tgts, srcs, iters)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        reg(w=0.1)
        flush.fill_(1)
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            out = reg(w=0.1)
            flush.fill_(1)
        e1.record(stream)
        barrier()
    dev_s = max_over_ranks(e0.elapsed_time(e1) / 1e3)
    assert np.all(out["iters"] == iters) and np.all(out["status"] == 0)
    pairs_step = float(sum(float(w.M) * w.N for w in wls)) * iters
    value = pairs_step * args.steps / dev_s
    # roofline over the whole batched step (the batched tensor-core E step is ≈ 96 % of it)
    peaks, peak_src = measured_peaks()
    f_max = float(peaks.get("sm_max_mhz", SM_MAX_MHZ_FALLBACK)) * 1e6
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    fp32_peak = sms * FP32_LANES_PER_SM * 2 * f_max / 1e12
    my_pairs = float(sum(float(w.M) * w.N for w in mine)) * iters
    t_rank = e0.elapsed_time(e1) / 1e3 / args.steps
    ex2_rate = my_pairs / t_rank
    mufu_peak = sms * MUFU_EX2_PER_SM * f_max
    roofline = {"bound": "alu", "achieved": ex2_rate, "peak": mufu_peak, "unit": "ex2/s", "frac": ex2_rate / mufu_peak,
                "traffic": None,
                "kernel": "lsg::estep_batch_tc_kernel, timed as the whole lsgcpd_register_batch step",
                "peak_source": f"MUFU.EX2 roofline: {sms} SMs x {MUFU_EX2_PER_SM} ex2/clk x {f_max/1e6:.0f} MHz "
                               f"(sm_max_mhz {peak_src})",
                "mufu_ex2_frac": ex2_rate / mufu_peak,
                "fp32_equiv_tflops": FLOPS_PER_PAIR * ex2_rate / 1e12,
                "fp32_equiv_frac_of_nominal": FLOPS_PER_PAIR * ex2_rate / 1e12 / fp32_peak}
    e2e = None
    if not args.skip_e2e:   # host clouds → prepare every target → batched registration → poses to the host
        h_t = [torch.from_numpy(w.target).pin_memory() for w in mine]
        h_s = [torch.from_numpy(w.source).pin_memory() for w in mine]

        def e2e_step():
            dt_ = [x.to(dev, non_blocking=True) for x in h_t]
            ds_ = [x.to(dev, non_blocking=True) for x in h_s]
            tg_ = lsg.prepare_batch(dt_, mine[0].knn_k)   # every target in one lsgcpd_prepare_batch call
            return lsg.BatchRegistrar(tg_, ds_, iters)(w=0.1)

        e2e_step()
        barrier()
        t0 = time.perf_counter()
        ne = max(1, min(args.steps, 2))
        for _ in range(ne):
            e2e_step()
        barrier()
        e2e_s = max_over_ranks(time.perf_counter() - t0)
        e2e = {"value": pairs_step * ne / e2e_s, "unit": UNIT, "registrations_per_s": BATCH_B * ne / e2e_s,
               "h2d_bytes_per_step": int(sum(x.numel() * 4 for x in h_t + h_s)),
               "d2h_bytes_per_step": int(len(mine) * (12 + 1 + 1 + 1) * 8), "steps": ne,
               "includes": "H2D of every cloud, lsgcpd_prepare_batch, lsgcpd_register_batch, poses to host"}
    cpu = None
    if rank == 0 and not args.skip_cpu:
        rate, cores, sample, secs = batch_oracle_rate(wls)
        cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample, "seconds": secs}
    if world > 1:
        dist.barrier()
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": dev_s / args.steps * 1e3, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": {"workload": "batch", "problems": BATCH_B, "points_per_cloud": BATCH_N,
                           "iters_per_step": iters, "w": 0.1, "step": "one lsgcpd_register_batch of all problems",
                           "parallelism": f"problems sharded x{world} (replicas only, no collective)",
                           "l2": "flushed between steps (256 MiB write)"},
                "registrations_per_s": BATCH_B * args.steps / dev_s, "roofline": roofline, "cpu_baseline": cpu,
                "e2e": e2e, "gpu_launches": (2 + 5 * iters) * args.steps, "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    ensure_ranks(args)
    rank, world, local = dist_env()
    import synth
    if args.config == "batch":
        if args.impl == "reference":
            if rank == 0:
                wls = synth.make_batch(BATCH_B, BATCH_N)
                rate, cores, sample, secs = batch_oracle_rate(wls, budget_s=10.0)
                print(json.dumps({"impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT,
                                  "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                                  "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                                  "dtype": "f64", "data": "synthetic", "config": {"workload": "batch"},
                                  "cpu_baseline": {"value": rate, "unit": UNIT, "cores": cores, "kind": "oracle",
                                                   "sample": sample},
                                  "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0,
                                          "d2h_bytes_per_step": 0}}), flush=True)
            return
        return run_batch(args, rank, world, local)
    wl = synth.make(args.config)
    if args.impl == "reference":
        return run_reference(args, wl, rank)

    import torch
    import torch.distributed as dist
    import paper_2103_15039_b200 as lsg

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    iters = args.iters or wl.iters
    lo, hi = (0, wl.N) if args.replicas else shard(wl.N, rank, world)
    n_local = hi - lo

    # resident inputs
    tgt_xyz = torch.from_numpy(wl.target).to(dev)
    src = torch.from_numpy(np.ascontiguousarray(wl.source[lo:hi])).to(dev)
    target = lsg.prepare_target(tgt_xyz, wl.knn_k)
    comm = lsg.Comm(rank, world) if world > 1 and not args.replicas else None
    reg = lsg.Registrar(target, src, iters)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)   # 256 MiB > 126 MB L2

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def step():
        return reg(w=wl.w, comm=comm)

    for _ in range(args.warmup):
        out = step()
        flush.fill_(1)
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    iters_done = []
    barrier()
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            out = step()
            iters_done.append(out["iters"])
            flush.fill_(1)
        e1.record(stream)
        barrier()
    dev_s = max_over_ranks(e0.elapsed_time(e1) / 1e3)
    pairs_per_step = float(wl.M) * float(wl.N) * iters * (world if args.replicas else 1)
    assert all(i == iters for i in iters_done), iters_done
    value = pairs_per_step * args.steps / dev_s
    clocks = clk.summary()

    # ---- roofline of the dominant kernel: the fused E step (lsgcpd_estep on this stream) ----
    runner = lsg.EstepRunner(target, src)
    s2_probe = float(out["sigma2"])
    for _ in range(2):
        runner(out["R"], out["t"], s2_probe, wl.w)
    nrep = 3
    barrier()
    k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k0.record(stream)
    for _ in range(nrep):
        runner(out["R"], out["t"], s2_probe, wl.w)
    k1.record(stream)
    barrier()
    t_launch = max_over_ranks(k0.elapsed_time(k1) / 1e3 / nrep)
    pairs_launch = float(wl.M) * float(n_local)
    peaks, peak_src = measured_peaks()
    f_max = float(peaks.get("sm_max_mhz", SM_MAX_MHZ_FALLBACK)) * 1e6
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    mufu_peak = sms * MUFU_EX2_PER_SM * f_max            # ex2/s: unit count x clock (B200_PROFILING / SURVEY)
    fp32_peak_tflops = sms * FP32_LANES_PER_SM * 2 * f_max / 1e12
    ex2_rate = pairs_launch / t_launch                     # one MUFU.EX2 per pair
    share = centred_tile_share(target, s2_probe, float(lsg.get_option("tile_gate")))
    lane_ops = LANE_OPS_CENTRED * share + LANE_OPS_HILO * (1.0 - share)
    mb = microbench_peaks()
    ffma2_meas = mb.get("ffma2_lane_ops_per_s")
    ex2_meas = mb.get("ex2_per_s")
    roofline = {"bound": "alu", "achieved": ex2_rate, "peak": mufu_peak, "unit": "ex2/s",
                "frac": ex2_rate / mufu_peak, "traffic": traffic_per_launch(wl.name, world),
                "kernel": "lsg::estep_tc_kernel (tcgen05 TF32 feature sums; tile-centred residual) + merge, via "
                          "lsgcpd_estep on the launching stream",
                "peak_source": f"MUFU.EX2 roofline: {sms} SMs x {MUFU_EX2_PER_SM} ex2/clk x {f_max/1e6:.0f} MHz "
                               f"(sm_max_mhz {peak_src}, MEASURED_PEAKS.json; the north star's roofline)",
                "pairs_per_launch": pairs_launch, "launch_ms": t_launch * 1e3,
                "mufu_ex2_frac": ex2_rate / mufu_peak,
                "mufu_ex2_frac_vs_microbench": (ex2_rate / ex2_meas) if ex2_meas else None,
                "centred_tile_share": share, "fp32_lane_ops_per_pair": lane_ops,
                "fp32_lane_frac": (lane_ops * ex2_rate / ffma2_meas) if ffma2_meas else None,
                "fp32_lane_peak_source": "measured FFMA2 lane-op/s, profiles/microbench_peaks.json" if ffma2_meas
                                         else None,
                "fp32_equiv_tflops": FLOPS_PER_PAIR * ex2_rate / 1e12,
                "fp32_equiv_frac_of_nominal": FLOPS_PER_PAIR * ex2_rate / 1e12 / fp32_peak_tflops,
                "pairs_per_s_per_gpu": ex2_rate}

    # ---- e2e: host buffers → public API → host results ----
    e2e = None
    if not args.skip_e2e:
        h_tgt = torch.from_numpy(wl.target).pin_memory()
        h_src = torch.from_numpy(np.ascontiguousarray(wl.source[lo:hi])).pin_memory()
        d_tgt = torch.empty_like(h_tgt, device=dev)
        d_src = torch.empty_like(h_src, device=dev)

        def e2e_step():
            d_tgt.copy_(h_tgt, non_blocking=True)
            d_src.copy_(h_src, non_blocking=True)
            tg = lsg.prepare_target(d_tgt, wl.knn_k)
            return lsg.Registrar(tg, d_src, iters)(w=wl.w, comm=comm)

        e2e_step()
        flush.fill_(1)
        ne = max(1, min(args.steps, 3))
        barrier()
        t0 = time.perf_counter()
        for _ in range(ne):
            r = e2e_step()
            flush.fill_(1)
        barrier()
        e2e_s = max_over_ranks(time.perf_counter() - t0)
        e2e = {"value": pairs_per_step * ne / e2e_s, "unit": UNIT,
               "registrations_per_s": ne * (world if args.replicas else 1) / e2e_s,
               "h2d_bytes_per_step": int(h_tgt.numel() * 4 + h_src.numel() * 4),
               "d2h_bytes_per_step": int(9 * 8 + 3 * 8 + 8 + 4), "steps": ne,
               "includes": "H2D target+source, lsgcpd_prepare_target, lsgcpd_register, R/t/sigma2 to host"}

    cpu = None
    if rank == 0 and not args.skip_cpu:   # rank 0 at every world size (the other ranks wait at the barrier)
        rate, cores, sample, secs = cpu_oracle_rate(wl)
        cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample,
               "seconds": secs}

    if world > 1:
        dist.barrier()
    if rank == 0:
        # per registration: setup + σ²₀ sums + σ²₀ init, then per EM iteration the pair kernels (tensor-core
        # E step + CUDA-core E step, which returns at once in the fixed-max mode, per half of the target; one small-block CUDA-core
        # kernel for problems too small to fill the GPU), then merge, moments, Newton — or, for N ≤ 2^17,
        # one em_tail_kernel (plus newton_kernel after the all-reduce when a communicator is used)
        m_pad = -(-wl.M // 256) * 256
        tc = -(-n_local // 768) * (m_pad // 64) >= 2 * torch.cuda.get_device_properties(dev).multi_processor_count
        halves = 2 if tc and (m_pad // 64) * 10240 > (48 << 20) else 1   # target swept in halves
        tail = (1 if comm is None else 2) if n_local <= (1 << 17) else 3
        launches_per_step = 3 + ((2 * halves if tc else 1) + tail) * iters
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dev_s / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak" if args.replicas else "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": wl.name, "M": wl.M, "N": wl.N, "iters_per_step": iters, "w": wl.w,
                       "knn_k": wl.knn_k, "step": "one full registration (lsgcpd_register)",
                       "parallelism": (f"replicas x{world} (independent registrations, no collective)"
                                       if args.replicas else
                                       f"source-sharded x{world}, target replicated, 75-double NCCL all-reduce "
                                       f"per EM iteration"),
                       "l2": "flushed between steps (256 MiB write)"},
            "registrations_per_s": args.steps * (world if args.replicas else 1) / dev_s,
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps, "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
