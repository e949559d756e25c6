#!/usr/bin/env python
"""Throughput benchmark of one full bound+gradient evaluation (Engine::evaluate(true)).

Metric (BASELINE.json): datapoints/sec per bound+grad eval, Bayesian GP-LVM RBF-ARD,
M=100.  Workload C3: N=1M, Q=10, D=50, M=100, N sharded over the ranks (strong
scaling); one step = psi forward kernel -> NCCL allreduce #1 -> fp64 coordinator
-> psi backward kernel -> NCCL allreduce #2 -> gradient assembly.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...      (one rank per GPU, NCCL)

Rank 0 prints ONE JSON line.  ``value`` is device-timed with inputs resident in HBM
(CUDA events on the engine's stream, L2 flushed before every timed step, max over
ranks); ``e2e`` goes through the public API (sgp.Engine / DistributedEngine) with
pinned host mu/S uploaded and d_mu/d_S read back every step.  ``--impl reference``
times the CPU oracle (a restatement of the reference, which cannot be compiled here:
no Eigen) on all host cores on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "datapoints/sec per bound+grad eval (BGPLVM RBF, M=100) at 1/2/4/8 B200 vs CPU"
UNIT = "datapoints/s"
WORKLOADS = {
    # id: (N, Q, D, M, description)
    "C3": (1_000_000, 10, 50, 100, "C3 Bayesian GP-LVM RBF-ARD N=1M Q=10 D=50 M=100, N-sharded"),
    "C2": (100_000, 10, 10, 100, "C2 Bayesian GP-LVM RBF-ARD N=100k Q=10 D=10 M=100"),
    "C5": (4_000_000, 20, 100, 256, "C5 Bayesian GP-LVM RBF-ARD N=4M Q=20 D=100 M=256"),
}
VARIANCE, LENGTHSCALE, BETA, S_INIT = 1.0, 1.0, 100.0, 0.5
PEAK_FP32_TFLOPS = 71.7  # measured FFMA peak, profiles/r01_pipe_microbench.log (148 SMs @ 1965 MHz)


def tensor_peak():
    """Dense bf16 tensor peak from the driver-written MEASURED_PEAKS.json (sustained: the psi
    kernels run inside a long step), else the profiling recipe's nominal 2250 TF/s."""
    try:
        pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(pk["bf16_tflops_sustained"]), "MEASURED_PEAKS.json bf16_tflops_sustained"
    except Exception:
        return 2250.0, "nominal dense bf16 (B200_PROFILING.md fallback)"


def algorithmic_flops(q, d, m):
    """per datapoint and eval, FMA = 2 flops.
    psi2 fwd 4Q+3 / bwd 11Q+4 per (n, pair); psi1 fwd 4Q+2+2D / bwd 11Q+4+2D per (n, m)."""
    p = m * (m + 1) // 2
    fwd = p * (4 * q + 3) + m * (4 * q + 2 + 2 * d)
    bwd = p * (11 * q + 4) + m * (11 * q + 4 + 2 * d)
    return fwd, bwd


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 50 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.path = f"/tmp/sgpx_clocks_{os.getpid()}.csv"

    def _lines(self):
        try:
            with open(self.path) as f:
                return sum(1 for _ in f)
        except OSError:
            return 0

    def __enter__(self):
        try:
            self.f = open(self.path, "w", buffering=1)
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "50"], stdout=self.f,
                                         stderr=subprocess.DEVNULL)
            # nvidia-smi takes a few hundred ms to start: wait for its first sample so that the
            # samples of the timed region (taken from here on) are not lost to the start-up
            t0 = time.time()
            while self._lines() == 0 and time.time() - t0 < 5.0 and self.proc.poll() is None:
                time.sleep(0.01)
        except Exception:
            self.proc = None
        self.first = self._lines()
        return self

    def __exit__(self, *a):
        self.last = self._lines()
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.f.close()

    def summary(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lines = open(self.path).read().splitlines()
        # the samples taken inside the timed region (plus the one just before it, if none landed)
        lines = lines[max(0, self.first - 1):max(self.first, self.last)] if self.last > self.first else lines[-1:]
        for line in lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def synth_shard(n_global, q, d, m, row_begin, n_local, device):
    """Seeded synthetic inputs of the named shape: mu ~ N(0,1), S = 0.5,
    Y ~ N(0,1), Z = M distinct rows of mu (seeded permutation), var = l = 1, beta = 100.
    Generated for the full N on every rank so every world size sees the same dataset."""
    import torch

    g = torch.Generator(device=device).manual_seed(0)
    mu_t = torch.randn(q, n_global, generator=g, device=device, dtype=torch.float64)  # (Q, N) -> col-major N x Q
    y_t = torch.randn(d, n_global, generator=g, device=device, dtype=torch.float64)
    idx = torch.randperm(n_global, generator=torch.Generator().manual_seed(1))[:m]
    z = mu_t[:, idx.to(device)].t().contiguous().cpu().numpy()  # M x Q
    mu = mu_t[:, row_begin:row_begin + n_local].contiguous().t()  # n_local x Q, stride (1, n_local)
    s = torch.full((q, n_local), S_INIT, device=device, dtype=torch.float64).t()
    y = y_t[:, row_begin:row_begin + n_local].contiguous().t()
    del mu_t, y_t
    return mu, s, y, np.asfortranarray(z)


def cpu_sample(q, d, m, n_sample, seed=0):
    rng = np.random.default_rng(seed)
    mu = np.asfortranarray(rng.normal(size=(n_sample, q)))
    s = np.full((n_sample, q), S_INIT, order="F")
    y = np.asfortranarray(rng.normal(size=(n_sample, d)))
    z = np.asfortranarray(mu[rng.permutation(n_sample)[:m]])
    return mu, s, y, z


def time_oracle(q, d, m, n_sample, steps, warmup, threads):
    """CPU oracle (restatement of the reference Engine::evaluate(true), std::thread workers)."""
    import oracle

    mu, s, y, z = cpu_sample(q, d, m, n_sample)
    ls = np.full(q, LENGTHSCALE)
    for _ in range(warmup):
        oracle.engine_evaluate(True, mu, s, y, z, VARIANCE, ls, BETA, workers=threads)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        oracle.engine_evaluate(True, mu, s, y, z, VARIANCE, ls, BETA, workers=threads)
        times.append(time.perf_counter() - t0)
    return float(np.mean(times)), times


def run_reference(args, world, rank):
    """--impl reference: the reference's CPU path (oracle port; the reference itself needs Eigen)."""
    if rank != 0:
        return
    n, q, d, m, desc = WORKLOADS[args.config]
    threads = os.cpu_count() or 1
    n_sample = args.cpu_sample
    t, _ = time_oracle(q, d, m, n_sample, args.steps, args.warmup, threads)
    v = n_sample / t
    sample = f"first-{n_sample} rows of the {args.config} shape (Q={q}, D={d}, M={m}); per-datapoint cost is " \
             f"data-independent (PAPER.md:150 linear in N)"
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (numpy seed 0; S=0.5, Z = M rows of mu)",
            "config": {"workload": desc, "N": n, "Q": q, "D": d, "M": m, "sample_N": n_sample},
            "impl": "reference",
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_b200(args, world, rank, local_rank):
    import torch

    from paper_1410_4984_b200 import sgp
    from paper_1410_4984_b200.engine_dist import DistributedEngine

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    n_cfg, q, d, m, desc = WORKLOADS[args.config]
    if args.scaling == "weak":
        n_global = n_cfg * world
        row_begin, row_end = rank * n_cfg, (rank + 1) * n_cfg
    else:
        n_global = n_cfg
        row_begin, row_end = sgp.make_partition(n_global, world)[rank]
    n_local = row_end - row_begin
    if args.scaling == "weak":
        mu, s, y, z = synth_shard(n_cfg, q, d, m, 0, n_local, dev)  # every rank: its own copy of the C3 data
    else:
        mu, s, y, z = synth_shard(n_global, q, d, m, row_begin, n_local, dev)
    kernel = sgp.KernelSpec(VARIANCE, np.full(q, LENGTHSCALE))
    stream = torch.cuda.current_stream(dev)

    use_dist = world > 1 or args.force_dist
    if use_dist and dist is None:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    eng = DistributedEngine(sgp.ModelKind.latent, mu, s, y, n_global, row_begin,
                            passes=None) if use_dist else None
    if eng is None:
        ctx = sgp.Context(local_rank)
        ctx.set_stream(stream.cuda_stream)
        single = sgp.Engine(sgp.ModelKind.latent, mu, s, y, ctx=ctx)
        single.broadcast(kernel, BETA, z)
        evaluate = lambda lh=False: single.evaluate(True, local_to_host=lh)  # noqa: E731
        launch_count = ctx.launch_count
    else:
        eng.broadcast(kernel, BETA, z)
        evaluate = lambda lh=False: eng.evaluate(True, local_to_host=lh)  # noqa: E731
        launch_count = eng.passes.launch_count

    def barrier():
        torch.cuda.synchronize(dev)
        if dist is not None:
            dist.barrier(device_ids=[local_rank])
        torch.cuda.synchronize(dev)

    def max_over_ranks(x):
        if dist is None:
            return float(x)
        t = torch.tensor([float(x)], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x):
        if dist is None:
            return float(x)
        t = torch.tensor([float(x)], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    # ---------------- device-resident timing (value) ----------------
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2
    for _ in range(args.warmup):
        r = evaluate()
    barrier()
    launches0 = launch_count()
    step_ms, fwd_k, bwd_k, coord_s = [], [], [], []
    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with ClockSampler(local_rank) as clocks:
        for i in range(args.steps):
            flush.zero_()  # untimed L2 flush between timed steps
            ev0[i].record(stream)
            r = evaluate()
            ev1[i].record(stream)
            fwd_k.append(r.timing.fwd_kernel_s)
            bwd_k.append(r.timing.bwd_kernel_s)
            coord_s.append(r.timing.coordinator_s)
        barrier()
    launches = launch_count() - launches0
    step_ms = [a.elapsed_time(b) for a, b in zip(ev0, ev1)]
    total_s = max_over_ranks(sum(step_ms) * 1e-3)
    ms_per_step = total_s / args.steps * 1e3
    value = n_global / (total_s / args.steps)
    clk = clocks.summary()
    total_launches = int(sum_over_ranks(launches))

    # kernel roofline of the dominant kernel (psi backward), per launch on this rank
    fwd_flops, bwd_flops = algorithmic_flops(q, d, m)
    bwd_s = float(np.mean(bwd_k))
    fwd_s = float(np.mean(fwd_k))
    bwd_tf = n_local * bwd_flops / bwd_s / 1e12
    fwd_tf = n_local * fwd_flops / fwd_s / 1e12
    psi_tf = n_local * (fwd_flops + bwd_flops) / (fwd_s + bwd_s) / 1e12
    t_peak, t_src = tensor_peak()
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic_bwd.json")
    if os.path.exists(tpath):
        try:
            tj = json.load(open(tpath))
            if tj.get("config") == args.config and tj.get("n_local") == n_local:
                traffic = tj.get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    # ---------------- end to end through the public API ----------------
    # pinned host mu / S (column-major) uploaded every step by broadcast(); d_mu / d_S read back.
    mu_h = torch.empty(q, n_local, dtype=torch.float64, pin_memory=True)
    s_h = torch.empty(q, n_local, dtype=torch.float64, pin_memory=True)
    mu_h.copy_(mu.t())
    s_h.copy_(s.t())
    mu_np, s_np = mu_h.numpy().T, s_h.numpy().T  # Fortran-ordered views of pinned memory
    gmu_h = torch.empty(q, n_local, dtype=torch.float64, pin_memory=True)
    gs_h = torch.empty(q, n_local, dtype=torch.float64, pin_memory=True)
    target = single if eng is None else eng
    target.set_local_grads_out(gmu_h.numpy().T, gs_h.numpy().T)
    for _ in range(max(1, args.warmup // 2)):
        target.broadcast(kernel, BETA, z, mu_np, s_np)
        evaluate(True)
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        target.broadcast(kernel, BETA, z, mu_np, s_np)
        r_e2e = evaluate(True)
        _ = r_e2e.bound.total
    barrier()
    e2e_s = max_over_ranks(time.perf_counter() - t0)
    e2e_value = n_global / (e2e_s / args.steps)
    mv = (m + 3) // 4 * 4
    h2d = 2 * n_local * q * 8 + m * q * 8 + mv * 12 * 4 + mv * mv * 4 + d * mv * 4
    d2h = 2 * n_local * q * 8 + (4 + m * (m + 1) // 2 + m * d) * 8 + (1 + q + m * q) * 8 + 8
    h2d_all, d2h_all = int(sum_over_ranks(h2d)), int(sum_over_ranks(d2h))

    # ---------------- CPU baseline (rank 0, N=1 only) ----------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        t_cpu, _ = time_oracle(q, d, m, args.cpu_sample, 2, 1, threads)
        cpu = {"value": args.cpu_sample / t_cpu, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"{args.cpu_sample} datapoints of the {args.config} shape, 1 warm-up + 2 timed evals of the "
                         f"fp64 oracle Engine::evaluate(true) restatement with {threads} std::thread workers"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "f32-equivalent: 3-piece fp16 / bf16 split tcgen05 MMAs (~2^-22 / 2^-17 rel.), fp32 exp2, fp64 accumulation and M-sized algebra",
            "data": "synthetic (torch Philox seed 0: mu,Y ~ N(0,1), S=0.5, Z = M rows of mu; var=l=1, beta=100)",
            "config": {"workload": desc, "N": n_global, "Q": q, "D": d, "M": m, "n_local": n_local,
                       "parallelism": f"dp{world}", "l2": "inputs 560 MB > L2 and 256 MB L2 flush before each "
                                                         "timed step (untimed)"},
            "roofline": {"bound": "tensor", "kernel": "psi passes (psi1 + psi2 forward and backward launch sequences)",
                         "achieved": psi_tf, "peak": t_peak, "unit": "TFLOP/s", "frac": psi_tf / t_peak,
                         "traffic": traffic, "peak_source": t_src,
                         "flops_per_launch": n_local * (fwd_flops + bwd_flops), "avg_launch_ms": (fwd_s + bwd_s) * 1e3,
                         "work": "SURVEY.md 8(d) algorithmic FP32-class flops P(15Q+7)+M(15Q+4D+6) per datapoint "
                                 "(FMA = 2), executed as 3-piece fp16 / bf16 split tcgen05 MMAs + MUFU/FMA exp2",
                         "fp32_simt": {"peak": PEAK_FP32_TFLOPS, "frac": psi_tf / PEAK_FP32_TFLOPS,
                                       "note": "SURVEY 8(d) FP32-FMA roofline; > 1 means beyond a SIMT design"},
                         "fwd": {"achieved": fwd_tf, "avg_launch_ms": fwd_s * 1e3, "flops_per_launch": n_local * fwd_flops},
                         "bwd": {"achieved": bwd_tf, "avg_launch_ms": bwd_s * 1e3, "flops_per_launch": n_local * bwd_flops}},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d_all, "d2h_bytes_per_step": d2h_all,
                    "ms_per_step": e2e_s / args.steps * 1e3},
            "cpu_baseline": cpu,
            "clocks": clk,
            "gpu_launches": total_launches,
            "coordinator_ms": float(np.mean(coord_s)) * 1e3,
            "bound_total": float(r.bound.total),
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier(device_ids=[local_rank])
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="C3", choices=sorted(WORKLOADS))
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"])
    ap.add_argument("--cpu-sample", type=int, default=32768)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--force-dist", action="store_true", help="use DistributedEngine (NCCL) even at world size 1")
    args = ap.parse_args()
    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local_rank = env_int("LOCAL_RANK", 0)
    if args.warmup < 3 and args.impl == "b200":
        args.warmup = 3  # timing rule: at least 3 warm-up steps
    if args.impl == "reference":
        run_reference(args, world, rank)
    else:
        run_b200(args, world, rank, local_rank)


if __name__ == "__main__":
    main()
