"""Benchmark: FAS forward + adjoint training step to tolerance, layer*samples/s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2]

A step is one training step of BASELINE.json configs[1] -- dense tanh ResNet, 1024 layers,
width 512, batch 256, 3-level FAS (cf 4, levels [1024, 256, 64]) -- on synthetic data from the
reference's own seeded generators: FAS forward solve to tol 1e-9 (multigrid.py:263-311), FAS
adjoint to tol 1e-9, per-layer parameter gradients and the SGD step (training.py:194-236).
value = N_layers * B / seconds per step, whole job.  Inputs (theta 2 GiB, states 1 GiB) exceed
the 126 MB L2, so no explicit flush is needed between steps.

Under torchrun (--gpus N > 1) the layer axis is partitioned across ranks
(paper_2007_07336_b200.distributed); timing is the max over ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # BASELINE.json configs[1]
    "c2": dict(depth=1024, width=512, batch=256, cf=4, threshold=64, tol=1e-9, max_cycles=50,
               lr=0.1, workload="dense tanh ResNet 1024 layers width 512 batch 256, 3-level FAS "
                                "(cf 4, levels [1024,256,64]) forward+adjoint training step to tol 1e-9"),
    # configs[0]-shaped small case (CPU-runnable reference demo), for quick runs
    "c1": dict(depth=64, width=32, batch=64, cf=4, threshold=None, tol=1e-9, max_cycles=50, lr=0.1,
               workload="dense tanh ResNet 64 layers width 32 batch 64, 2-level FAS cf 4 "
                        "forward+adjoint training step to tol 1e-9"),
    # BASELINE.json configs[2]: conv ResNet (3x3 conv + bias + ReLU, 64 channels, 32x32), 256 layers
    "c3": dict(kind="conv", depth=256, width=64 * 32 * 32, channels=64, side=32, batch=32, cf=4,
               threshold=16, tol=1e-9, max_cycles=50, lr=0.1, input_dim=64,
               workload="conv ResNet 256 layers (3x3 conv+bias+ReLU, 64 ch, 32x32) batch 32, 3-level "
                        "FAS (cf 4, levels [256,64,16]) forward+adjoint training step to tol 1e-9; "
                        "dense tanh opening from 64 features"),
    # BASELINE.json configs[3]: deep dense ResNet, layer-partitioned across 2/4/8 GPUs (SURVEY 8d:
    # cf 4, 2 levels [4096, 1024]); theta 32 GiB, states 32 GiB -- it also fits one B200
    "c4": dict(depth=4096, width=1024, batch=1024, cf=4, threshold=1024, tol=1e-9, max_cycles=50,
               lr=0.1, workload="dense tanh ResNet 4096 layers width 1024 batch 1024, 2-level FAS "
                                "(cf 4, levels [4096,1024]) forward+adjoint training step to tol 1e-9"),
    # configs[4]-style HBM-bound point (q=512, B=16, cf 16)
    "c5": dict(depth=1024, width=512, batch=16, cf=16, threshold=4, tol=1e-9, max_cycles=50, lr=0.1,
               workload="dense tanh ResNet 1024 layers width 512 batch 16, 3-level FAS cf 16 "
                        "forward+adjoint training step to tol 1e-9"),
    # BASELINE.json configs[4]'s shortest-critical-path point at the reference's survey shape
    # (q 16, one sample, cf 16, levels [1024, 64, 4]): the latency-bound regime,
    # where the FAS step beats layer-by-layer GPU propagation already on one GPU
    "c6": dict(depth=1024, width=16, batch=1, cf=16, threshold=4, tol=1e-9, max_cycles=50, lr=0.1,
               workload="dense tanh ResNet 1024 layers width 16 batch 1, 3-level FAS cf 16 "
                        "(levels [1024,64,4]) forward+adjoint training step to tol 1e-9"),
    # the same regime four times deeper (tools/cf_sweep.py --depths: FAS's per-cycle critical path
    # grows with the level count, serial propagation with the depth) -- where the FAS step is
    # faster than layer-by-layer GPU propagation on one GPU
    "c7": dict(depth=4096, width=16, batch=1, cf=16, threshold=16, tol=1e-9, max_cycles=50, lr=0.1,
               workload="dense tanh ResNet 4096 layers width 16 batch 1, 3-level FAS cf 16 "
                        "(levels [4096,256,16]) forward+adjoint training step to tol 1e-9"),
}

METRIC = "FAS fwd+adjoint solve time to tol; layer*samples/s"
UNIT = "layer*samples/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    p.add_argument("--adjoint", default="fas", choices=["fas", "sequential"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--batch", type=int, default=None,
                   help="override the config's batch (functional checks; recorded in config)")
    p.add_argument("--split", type=int, default=None,
                   help="batch slices on concurrent streams (default: 2 when B >= 64)")
    return p.parse_args()


# ---------------------------------------------------------------------------------------------
# CPU side (the oracle port; the reference itself is Python and not on the GPU box)


_POOL = {}  # the parent's network + config, inherited by the forked workers (copy-on-write)


def _cpu_net(cfg):
    """The oracle network of a config (host arrays), built once per process."""
    from oracle import fas

    N, q = cfg["depth"], cfg["width"]
    if cfg.get("kind") == "conv":
        from paper_2007_07336_b200.synthetic import conv_network_arrays

        a = conv_network_arrays(N, cfg["channels"], cfg["side"], [0, N, cfg["channels"]],
                                input_dim=cfg["input_dim"])
        fine = fas.ConvLevel(a["Wc"], a["b"], a["activation"], a["step"], a["side"], a["side"])
        return fas.Net(a["Wo"], a["bo"], "tanh", fine, a["Wr"], a["br"], "identity")
    return fas.net_from_arrays(fas.random_network_arrays(N, q, [0, N, q]))


def _cpu_one_sample(job):
    """One sample of the training step on one host core (one process per
    core, OPENBLAS 1 thread): FAS forward solve to tol, FAS adjoint to tol (the algorithm the GPU
    arm runs), block gradients.  Runs to convergence -- no cycle extrapolation."""
    b, max_cycles = job
    import numpy as np
    from threadpoolctl import threadpool_limits

    from oracle import fas

    cfg, net = _POOL["cfg"], _POOL["net"]
    N, q, c, thr, tol = cfg["depth"], cfg["width"], cfg["cf"], cfg["threshold"], cfg["tol"]
    din = cfg.get("input_dim", q)
    with threadpool_limits(limits=1, user_api="blas"):
        t0 = time.perf_counter()
        X = fas.random_sample(din, [0, N, q, b])[None]
        src = net.source(X)
        U, fh, fconv = fas.solve(fas.build_levels(net.blocks, c, thr), c, src, tol, max_cycles)
        final, logits = fas.adjoint_head(net, U)
        _, dl = fas.loss_and_dlogits(logits, np.array([b % 10]))
        gfin, _ = fas.g_final_from(net, final, dl)
        D = fas.derivs(net.blocks, U)
        s = np.zeros_like(U)
        s[0] = gfin
        adj = fas.adjoint_level(net.blocks, D)
        mu, ah, aconv = fas.solve(fas.build_levels(adj, c, thr), c, s, tol, max_cycles)
        fas.block_grads(net.blocks, U, mu, D, 1.0)
        return dict(fwd=len(fh[0]) - 1, adj=len(ah[0]) - 1, converged=bool(fconv[0] and aconv[0]),
                    final=fh[0][-1], s=time.perf_counter() - t0)


class CpuArm:
    """The reference algorithm on the host cores: a pool of P forked worker processes (P = host
    cores), one sample each per step, every sample solved to tol forward and adjoint.  A step's
    layer*samples/s = N * P / wall seconds of the step (samples are independent; extrapolation
    is across samples only)."""

    def __init__(self, cfg, procs=None):
        import multiprocessing as mp

        self.cfg = cfg
        self.P = procs or os.cpu_count() or 1
        _POOL["cfg"], _POOL["net"] = cfg, _cpu_net(cfg)
        self.pool = mp.get_context("fork").Pool(self.P)
        self.next = 0

    def step(self, max_cycles=None):
        jobs = [((self.next + i) % self.cfg["batch"], max_cycles or self.cfg["max_cycles"])
                for i in range(self.P)]
        self.next += self.P
        t0 = time.perf_counter()
        out = self.pool.map(_cpu_one_sample, jobs, chunksize=1)
        wall = time.perf_counter() - t0
        return self.cfg["depth"] * len(jobs) / wall, wall, out

    def warm(self):
        """Untimed warm-up: every worker runs one bounded solve (1 cycle forward and adjoint)."""
        return self.step(max_cycles=1)

    def close(self):
        self.pool.close()
        self.pool.join()

    def describe(self, out, steps):
        fwd = sorted({o["fwd"] for o in out})
        adj = sorted({o["adj"] for o in out})
        return (f"{self.P} forked processes x 1 BLAS thread (OPENBLAS via threadpoolctl), one "
                f"sample each per step, {steps} step(s): FAS forward to tol {self.cfg['tol']:g} "
                f"({'/'.join(map(str, fwd))} cycles) + FAS adjoint to tol ({'/'.join(map(str, adj))} "
                f"cycles) + block gradients, every sample solved to convergence "
                f"(all converged: {all(o['converged'] for o in out)}); oracle/fas.py (numpy port "
                f"of the reference path, per-sample W @ u like the reference)")


def cpu_reference_sample(cfg, steps=1):
    """Bounded CPU baseline for the GPU arm's JSON line: one warm-up map + `steps` timed steps."""
    arm = CpuArm(cfg)
    try:
        arm.warm()
        vals, out = [], []
        for _ in range(steps):
            v, _, o = arm.step()
            vals.append(v)
            out += o
        return statistics.mean(vals), dict(cores=arm.P, sample=arm.describe(out, steps))
    finally:
        arm.close()


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    arm = CpuArm(cfg)
    # A step solves one sample per worker to tol (c2: ~70 s on one core), so K requested steps can
    # take far longer than "a few minutes": timed steps stop once the next one would overrun the
    # budget (at least one runs); the line reports the steps actually timed.
    budget = float(os.environ.get("LMG_REF_BUDGET_S", "200"))
    try:
        for _ in range(min(args.warmup, 2)):  # bounded: one FAS cycle fwd + adjoint per worker
            arm.warm()
        vals, times, out = [], [], []
        for _ in range(args.steps):
            if times and sum(times) + statistics.mean(times) > budget:
                break
            v, wall, o = arm.step()
            vals.append(v)
            times.append(wall)
            out += o
    finally:
        arm.close()
    steps = len(times)
    value = steps * cfg["depth"] * arm.P / sum(times)
    line = dict(metric=METRIC, value=value, unit=UNIT, n_gpus=args.gpus, steps=steps,
                warmup=min(args.warmup, 2), ms_per_step=1e3 * statistics.mean(times),
                higher_is_better=True, scaling="strong", vs_baseline=None, dtype="f64",
                data="synthetic",
                config=dict(workload=cfg["workload"], samples_per_step=arm.P,
                            steps_requested=args.steps, warmup_requested=args.warmup,
                            time_budget_s=budget,
                            cycles_per_sample=[[o["fwd"], o["adj"]] for o in out]),
                impl="reference",
                cpu_baseline=dict(value=value, unit=UNIT, cores=arm.P, kind="port",
                                  sample=arm.describe(out, steps)),
                e2e=dict(value=value, unit=UNIT, h2d_bytes_per_step=0, d2h_bytes_per_step=0))
    print(json.dumps(line))


# ---------------------------------------------------------------------------------------------
# GPU side


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None

    def __enter__(self):
        """Start polling and wait for the first sample, so nvidia-smi's start-up (NVML init) is
        not inside the timed region (it measurably stalled short, sync-heavy steps like c5)."""
        import threading

        self.lines, self._warm = [], 0
        if os.environ.get("LMG_BENCH_NO_CLOCKS"):  # diagnosis only: no sampler at all
            self.proc = None
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(self.gpu)], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return self
        first = threading.Event()

        def reader():
            for ln in self.proc.stdout:
                self.lines.append(ln)
                first.set()

        self._thread = threading.Thread(target=reader, daemon=True)
        self._thread.start()
        first.wait(timeout=10.0)
        self._warm = len(self.lines)  # samples taken before the timed region
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=10)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self._thread.join(timeout=5)
            # the last pre-region sample stands in when the region was shorter than one period
            keep = self.lines[self._warm:] or self.lines[-1:]
            self.lines = [ln.strip() for ln in keep]
        else:
            self.lines = []

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for nm, val in zip(names, parts[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return dict(sm_mhz=statistics.median(sm) if sm else None, sm_max_mhz=mx,
                    reasons=sorted(reasons), samples=len(sm))


def load_traffic(config):
    """dram bytes per launch of the dominant kernel from the committed ncu --set full summary
    (only when that capture was taken on this config)."""
    import glob

    cands = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_ncu_summary.json")))
    if not cands:
        return None, None
    p = cands[-1]
    try:
        with open(p) as fh:
            d = json.load(fh)
        per = d.get("traffic_per_launch")  # round 2+: {config: dram bytes of one dominant launch}
        if per is not None:
            return per.get(config), d
        if d.get("config") != config:
            return None, d
        return d.get("dram_bytes_per_launch"), d
    except (OSError, ValueError):
        return None, None


class ThetaSnapshot:
    """The trainer's parameters, saved once before the warm-up and restored before every timed
    pass (clean, instrumented, serial, e2e): each pass times the same K SGD steps from the same
    theta, so the passes measure the same work.  The copy is outside every timed region."""

    def __init__(self, torch, dnet):
        self.live = [dnet.stack.W, dnet.stack.b, dnet.Wo, dnet.bo, dnet.Wr, dnet.br]
        need = sum(x.numel() * x.element_size() for x in self.live)
        # on the device only when it leaves room for the serial baseline's extra (N, B, q) stacks
        # (c4 at B 512: theta 32 GiB, each stack 16 GiB)
        where = "cuda" if need < torch.cuda.mem_get_info()[0] // 8 else "cpu"
        self.saved = [x.detach().to(where, copy=True) for x in self.live]
        self.torch = torch

    def restore(self):
        for d, s in zip(self.live, self.saved):
            d.copy_(s)
        self.torch.cuda.synchronize()


def run_ours(args, cfg):
    import numpy as np
    import torch

    import paper_2007_07336_b200 as P
    from paper_2007_07336_b200 import _lib
    from paper_2007_07336_b200.roofline import classify, fp64_peak_tflops, hbm_peak

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus != world and world > 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE {world}")
    # LMG_BENCH_BACKEND=gloo runs the multi-rank path on fewer GPUs than ranks (ranks share
    # devices, halos staged through host memory) -- a functional check, not a measurement
    backend = os.environ.get("LMG_BENCH_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    N, q, B = cfg["depth"], cfg["width"], cfg["batch"]
    conv = cfg.get("kind") == "conv"
    din = cfg.get("input_dim", q)
    X_host = torch.from_numpy(P.random_batch(din, [0, N, q], B)).pin_memory()
    lab_host = torch.from_numpy(np.arange(B) % 10).pin_memory()
    X = X_host.to(dev)
    labels = lab_host.to(dev)

    if world > 1:
        from paper_2007_07336_b200.distributed import LayerParallelTrainer

        tr = LayerParallelTrainer(N, q, [0, N, q], coarsening=cfg["cf"], threshold=cfg["threshold"],
                                  tol=cfg["tol"], max_cycles=cfg["max_cycles"], adjoint=args.adjoint,
                                  learning_rate=cfg["lr"])
    else:
        if conv:
            from paper_2007_07336_b200.synthetic import conv_device_network

            d = conv_device_network(N, cfg["channels"], cfg["side"], [0, N, cfg["channels"]],
                                    device=dev, input_dim=din)
        else:
            d = P.device_network(N, q, [0, N, q], device=dev)
        split = args.split if args.split is not None else 1
        tr = P.DeviceTrainer(d, coarsening=cfg["cf"], threshold=cfg["threshold"], tol=cfg["tol"],
                             max_cycles=cfg["max_cycles"], adjoint=args.adjoint,
                             learning_rate=cfg["lr"], split=split)
    peak = fp64_peak_tflops(torch, dev)
    theta = ThetaSnapshot(torch, tr.dnet)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    import gc

    # no Python GC pauses inside the timed regions (short, sync-heavy steps like c5 saw them)
    gc.collect()
    gc.disable()
    res = None
    theta.restore()
    for _ in range(args.warmup):
        res = tr.step(X, labels)
    barrier()

    # ---- timed region: inputs resident in HBM (no per-launch instrumentation inside)
    theta.restore()
    barrier()
    n0 = _lib.launch_count()
    with ClockSampler(local) as clk:
        barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        cycles = []
        for _ in range(args.steps):
            res = tr.step(X, labels)
            cycles.append((int(np.max(res.fwd_cycles)),
                           None if res.adj_cycles is None else int(np.max(res.adj_cycles))))
        e.record()
        barrier()
    launches = _lib.launch_count() - n0
    ms = s.elapsed_time(e) / args.steps
    if dist is not None:
        t = torch.tensor([ms], device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    # ---- roofline pass: the same K steps again with a CUDA event pair around every launch of
    # the library (recorded on the launching stream), summed per kernel class
    theta.restore()
    _lib.timing_enable(True)
    barrier()
    si, ei = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    si.record()
    for _ in range(args.steps):
        tr.step(X, labels)
    ei.record()
    barrier()
    inst_ms = si.elapsed_time(ei) / args.steps
    f_ms, f_flops, f_bytes, f_n = _lib.timing_read(0)
    a_ms, a_flops, a_bytes, a_n = _lib.timing_read(1)
    s_ms, s_flops, s_bytes, s_n = _lib.timing_read(6)  # split-K serial steps (latency-bound)
    w_ms, w_flops, w_bytes, w_n = (sum(v) for v in zip(_lib.timing_read(4), _lib.timing_read(5)))
    all_ms, _, _, all_n = _lib.timing_read(-1)
    _lib.timing_enable(False)

    # ---- serial layer-by-layer GPU propagation of the same step (north_star comparison): the
    # reference's sequential forward + sequential adjoint + gradients + SGD, same kernels
    serial_ms = None
    if world == 1:
        from paper_2007_07336_b200 import _lib as L_
        from paper_2007_07336_b200.training import _dense_apply, backward

        dn = tr.dnet
        view = dn._lmg_view()
        Us = torch.empty((N, B, q), dtype=torch.float64, device=dev)

        def serial_step():
            f0 = _dense_apply(dn.Wo, dn.bo, dn.open_act, X)
            L_.call("lmg_sequential_forward", view.desc(), B, f0.data_ptr(), L_.SRC_HEAD,
                    Us.data_ptr(), L_.stream_handle())
            backward(dn, Us, X, labels, adjoint="sequential", scale=1.0 / B, lr=cfg["lr"],
                     want_grads=False)

        theta.restore()
        serial_step()
        barrier()
        s3, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s3.record()
        for _ in range(args.steps):
            serial_step()
        e3.record()
        barrier()
        serial_ms = s3.elapsed_time(e3) / args.steps
        del Us
    elif not conv:
        # model-partitioned serial propagation over the same ranks: each rank
        # propagates its layers and hands the state on; timed like the FAS step (max over ranks)
        theta.restore()
        tr.serial_step(X, labels)
        barrier()
        s3, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s3.record()
        for _ in range(args.steps):
            tr.serial_step(X, labels)
        e3.record()
        barrier()
        serial_ms = s3.elapsed_time(e3) / args.steps
        t = torch.tensor([serial_ms], device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        serial_ms = float(t.item())

    # ---- e2e: same step through the public API from pinned host buffers, result read back
    theta.restore()
    barrier()
    s2, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s2.record()
    t_wall = time.perf_counter()
    for _ in range(args.steps):
        X.copy_(X_host, non_blocking=True)
        labels.copy_(lab_host, non_blocking=True)
        r2 = tr.step(X, labels)
        loss_host = r2.loss.cpu()
    e2.record()
    barrier()
    e2e_ms = s2.elapsed_time(e2) / args.steps
    wall_ms = (time.perf_counter() - t_wall) * 1e3 / args.steps
    if dist is not None:
        t = torch.tensor([e2e_ms], device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())

    # dominant kernel class: the relaxation / residual step launches (forward + adjoint layouts);
    # bound by its arithmetic intensity against the FP64 ridge (DGEMM peak / HBM peak)
    gemm_ms = f_ms + a_ms
    gemm_flops = f_flops + a_flops
    gemm_bytes = f_bytes + a_bytes
    hbm, hbm_src = hbm_peak()
    rf = classify(gemm_flops, gemm_bytes, gemm_ms, peak, hbm, force_tensor=conv)
    bound, unit_r, pk, achieved = rf["bound"], rf["unit"], rf["peak"], rf["achieved"]
    intensity, ridge = rf["intensity_flop_per_byte"], rf["fp64_ridge_flop_per_byte"]
    if bound == "tensor":
        pk_src = "cuBLAS DGEMM 8192^3 measured in this run (FP64 is not in MEASURED_PEAKS.json)"
        alg = "(2q^2+5q) flops per F-evaluation x B samples x tasks per launch"
    else:
        pk_src = hbm_src
        alg = ("8q^2 (W_j, read once per layer step for the whole batch) + 8qB per state row read "
               "or written, per task, summed over the launches")
    traffic, prof = load_traffic(args.config)
    theta_bytes = tr.dnet.stack.W.numel() * 8
    line = dict(
        metric=METRIC,
        value=N * B / (ms * 1e-3),
        unit=UNIT, n_gpus=world, steps=args.steps, warmup=args.warmup, ms_per_step=ms,
        higher_is_better=True, scaling="strong", vs_baseline=None,
        dtype="f64", data="synthetic (reference seeded generators: random_network / random_sample)",
        config=dict(workload=cfg["workload"], depth=N, width=q, batch=B, coarsening=cfg["cf"],
                    threshold=cfg["threshold"], tol=cfg["tol"], adjoint=args.adjoint,
                    parallelism=(f"layer-partitioned x{world}" if world > 1 else
                                 f"single GPU, {getattr(tr, 'split', 1)} batch slice(s) on concurrent streams"),
                    l2=(f"inputs larger than L2 (theta {theta_bytes / 2**30:.3f} GiB, states "
                        f"{N * B * q * 8 / 2**30:.2f} GiB), no flush"
                        if max(theta_bytes, N * B * q * 8) > 2 * 126e6 else
                        "theta smaller than L2: cycles re-read it from L2 (no flush; the FAS step "
                        "is latency-bound at this size)"),
                    cycles_per_step=cycles),
        e2e=dict(value=N * B / (e2e_ms * 1e-3), unit=UNIT,
                 h2d_bytes_per_step=int(X_host.numel() * 8 + lab_host.numel() * 8),
                 d2h_bytes_per_step=int(loss_host.numel() * 8), wall_ms_per_step=wall_ms),
        gpu_launches=int(launches),
        roofline=dict(bound=bound, achieved=achieved, peak=pk, unit=unit_r,
                      frac=achieved / pk if pk else None,
                      traffic=traffic,
                      kernel="relaxation/residual layer-step class, FP64 DMMA m8n8k4 with fused FAS "
                             "epilogues: lmg::step_gemm (forward: 2-stage 32x32 tiles; adjoint: "
                             "register-staged act'-scaled 64x128 / 64x32 tiles; batches <= 16: "
                             "16-row tiles) + lmg::chain_gemm (persistent chain launches of "
                             "small-batch sweeps); conv configs: lmg::conv_gemm",
                      peak_source=pk_src,
                      algorithmic=alg,
                      intensity_flop_per_byte=intensity, fp64_ridge_flop_per_byte=ridge,
                      share_of_step=(gemm_ms / (inst_ms * args.steps)) if inst_ms else None,
                      serial_steps=dict(
                          what="split-K serial layer steps (coarsest exact solve): latency-bound "
                               "chain, reported apart from the relaxation class",
                          ms_per_step=s_ms / args.steps, launches_per_step=s_n / args.steps,
                          tflops=(s_flops / (s_ms * 1e-3) / 1e12) if s_ms else None,
                          share_of_step=(s_ms / (inst_ms * args.steps)) if inst_ms else None),
                      fused_sweeps=dict(
                          what="fused persistent FCF / serial sweeps (state on chip; for q 16 / 32 "
                               "the warp-level FMA sweeps, state in registers)",
                          ms_per_step=w_ms / args.steps, launches_per_step=w_n / args.steps,
                          gbs=(w_bytes / (w_ms * 1e-3) / 1e9) if w_ms else None,
                          share_of_step=(w_ms / (inst_ms * args.steps)) if inst_ms else None,
                          bound=("latency: a serial chain of dependent layer steps; the warp FMA "
                                 "sweep runs 992 SM cycles per step against a ~450-cycle "
                                 "dependency floor (profiles/r2_ncu_wsweep.json, DESIGN 3)")
                          if cfg.get("width", 0) in (16, 32) else None),
                      all_step_gemm_tflops=((gemm_flops + s_flops) / ((gemm_ms + s_ms) * 1e-3) / 1e12)
                      if gemm_ms + s_ms > 0 else None,
                      launches=f_n + a_n, all_kernel_ms_per_step=all_ms / args.steps,
                      all_launches_per_step=all_n / args.steps,
                      measured="CUDA events around every step-GEMM launch, on its stream, over a "
                               "second pass of the K timed steps (instrumented step "
                               f"{inst_ms:.2f} ms vs {ms:.2f} ms clean)"),
    )
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, info = cpu_reference_sample(cfg)
        line["cpu_baseline"] = dict(value=v, unit=UNIT, cores=info["cores"], kind="port",
                                    sample=info["sample"])
    if serial_ms is not None:
        line["serial_gpu"] = dict(
            value=N * B / (serial_ms * 1e-3), unit=UNIT, ms_per_step=serial_ms,
            what=("layer-by-layer GPU propagation of the same step with the same kernels: "
                  "sequential_forward (network.py:111-123) + the reference's sequential adjoint "
                  "(training.py:216-224) + gradients + SGD"
                  + ("" if world == 1 else
                     f"; model-partitioned over {world} ranks (each rank propagates its layers "
                     "and hands the state to the next, LayerParallelTrainer.serial_step)")),
            fas_over_serial_time=ms / serial_ms)
    gc.enable()
    line["clocks"] = clk.summary()
    if rank == 0:
        print(json.dumps(line))
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    cfg = dict(CONFIGS[args.config])
    if args.batch is not None:
        cfg["batch"] = args.batch
        cfg["workload"] += f" [batch overridden to {args.batch}]"
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.config == "c4" and world == 1 and cfg["batch"] == 1024 and args.impl != "reference":
        raise SystemExit("c4 (4096 x 1024, batch 1024) needs >= 2 GPUs: theta 32 GiB + states, "
                         "adjoint and act' 3 x 32 GiB + level-0 workspace exceed one B200; run it "
                         "layer-partitioned (torchrun --nproc-per-node 2..8) or with --batch 512")
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
