#!/usr/bin/env python
"""Throughput benchmark of one full bound+gradient evaluation (Engine::evaluate(true)).

Metric (BASELINE.json): datapoints/sec per bound+grad eval, Bayesian GP-LVM RBF-ARD,
M=100.  Workload C3: N=1M, Q=10, D=50, M=100, N sharded over the ranks (strong
scaling); one step = psi forward kernel -> NCCL allreduce #1 -> fp64 coordinator
-> psi backward kernel -> NCCL allreduce #2 -> gradient assembly.  --config C2 / C4 / C5
time the other BASELINE.json configurations.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--config C3]
  torchrun --nproc-per-node N bench.py --gpus N ...      (one rank per GPU, NCCL)

Rank 0 prints ONE JSON line.  ``value`` is device-timed with inputs resident in HBM
(CUDA events on the engine's stream, L2 flushed before every timed step, max over
ranks); ``e2e`` goes through the public API (sgp.Engine / DistributedEngine) with
pinned host mu/S uploaded and d_mu/d_S read back every step.  Inputs are the reference
generator's stream (sgp::Rng), so the CPU arm sees the same data; ``cpu_baseline`` times the
fp64 oracle port at full N (C2, C3) and ``parity`` compares the GPU evaluation with it.
``--impl reference`` times the oracle port (the reference itself needs Eigen, absent here and
on the GPU box) on all host cores.
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
# id: (latent, N, Q, D, M, CPU-baseline rows (full N where ~10-30 s of CPU work), description)
WORKLOADS = {
    "C3": (True, 1_000_000, 10, 50, 100, 1_000_000,
           "C3 Bayesian GP-LVM RBF-ARD N=1M Q=10 D=50 M=100, N-sharded"),
    "C2": (True, 100_000, 10, 10, 100, 100_000, "C2 Bayesian GP-LVM RBF-ARD N=100k Q=10 D=10 M=100"),
    "C5": (True, 4_000_000, 20, 100, 256, 8192, "C5 Bayesian GP-LVM RBF-ARD N=4M Q=20 D=100 M=256"),
    "C4": (False, 10_000_000, 8, 1, 500, 16384, "C4 sparse GP regression, deterministic inputs, N=10M Q=8 D=1 M=500"),
}
INPUTS = "sgp::Rng (common.hpp:45-97): mu|X = Rng(0).normal_matrix(N,Q), Y = Rng(1).normal_matrix(N,D), " \
         "Z = init_gplvm's M rows of mu with Rng(2) (model.hpp:420-429); S = 0.5; latent: var = l = 1, beta = 100; " \
         "regression: var = l = beta = 1 (generated on the GPU by sgpx_rng_normal_matrix)"
PEAK_FP32_TFLOPS = 71.7  # measured FFMA peak, profiles/r01_pipe_microbench.log (148 SMs @ 1965 MHz)
EX2_RATE = 16 * 148 * 1.965e9  # MUFU.EX2 results / s (16 per clk per SM)
DTYPES = {
    "fast": "mixed: psi2 exponents as 2-piece fp16 tcgen05 MMAs (~2^-22), exp2 on MUFU/FMA (2^-22), "
            "bf16 / scaled-fp16 hi-lo contraction MMAs (~2^-17 / 2^-22), psi1 fp32, every sum and all "
            "M-sized algebra fp64",
    "precise": "mixed: psi2 exponents as 3-piece fp16 tcgen05 MMAs (~2^-33), exp2 on MUFU/FMA (2^-22), "
               "scaled-fp16 hi-lo contraction MMAs (~2^-22), psi1 fp32, every sum and all M-sized algebra fp64",
    "direct": "f64: direct-difference exponents, exp and every contraction and sum in fp64",
    "syrk": "mixed: Knm from fp64 exponents split into tf32 hi/lo; Phi = K^T K, Psi = K^T Y and G = [K|Y][2U; dPsi^T] "
            "as three-pass split-TF32 tcgen05 GEMMs (cuBLAS), fp32 accumulation over 512-row sub-chunks, fp64 "
            "across; every gradient contraction and all M-sized algebra fp64",
}


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


def mma_flops_per_pair(q, mode):
    """Tensor-pipe flops the row-tile kernels execute per (datapoint, pair): MMA1 (exponent, K =
    2 K1 halves, 3 or 6 piece products) + MMA3 (contraction, N3 columns, 3 piece products)."""
    k1 = (2 * q + 2 + 15) // 16 * 8
    n3 = (2 * q + 1 + 15) // 16 * 16
    return 2 * (2 * k1) * (6 if mode == "precise" else 3) + 2 * n3 * 3


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


def host_inputs(latent, n, q, d, m):
    """The workload's inputs on the host from the reference generator (oracle restatement of Rng)."""
    import oracle

    mu = oracle.rng_normal_matrix(0, n, q)
    y = oracle.rng_normal_matrix(1, n, d)
    z = np.asfortranarray(mu[oracle.rng_choose_rows(2, n, m)])
    s = np.full((n, q), 0.5, order="F") if latent else None
    return mu, s, y, z


def oracle_eval(latent, mu, s, y, z, q, beta, threads):
    import oracle

    t0 = time.perf_counter()
    r = oracle.engine_evaluate(latent, mu, s, y, z, 1.0, np.ones(q), beta, workers=threads, simd=True)
    return time.perf_counter() - t0, r


def cpu_desc(threads):
    try:
        model = [ln.split(":", 1)[1].strip() for ln in open("/proc/cpuinfo") if ln.startswith("model name")][0]
    except Exception:
        model = "unknown CPU"
    return f"{threads} threads of {model} (nproc {os.cpu_count()})"


def rel_err(a, b):
    """proj/tests/support/oracles.hpp:55-58, element-wise, max over entries."""
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    if a.size == 0:
        return 0.0
    return float(np.max(np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), 1.0)))


def parity_of(r, gmu, gs, ref, latent):
    """GPU evaluation vs the fp64 oracle on identical inputs."""
    out = {"bound_rel": rel_err(r.bound.total, ref.bound["total"])}
    g = r.grads
    pairs = dict(d_z=(g.d_z, ref.d_z), d_lengthscales=(g.d_lengthscales, ref.d_lengthscales),
                 d_variance=([g.d_variance], [ref.d_variance]), d_beta=([g.d_beta], [ref.d_beta]))
    if latent:
        pairs.update(d_mu=(gmu, ref.d_mu), d_s=(gs, ref.d_s))
    worst = 0.0
    for k, (a, b) in pairs.items():
        a, b = np.asarray(a, dtype=np.float64).ravel(), np.asarray(b, dtype=np.float64).ravel()
        e = rel_err(a, b)
        nr = float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
        out[k] = {"elem": e, "norm": nr}
        worst = max(worst, e)
    terms = {f: rel_err(getattr(r.bound, f), ref.bound[f]) for f in ref.bound}
    out["bound_terms_max_rel"] = max(terms.values())
    out["grads_max_elem_rel"] = worst
    worst_norm = max(v["norm"] for k, v in out.items() if isinstance(v, dict))
    out["grads_max_norm_rel"] = worst_norm
    direct = r.timing.precision == "direct"
    out["tolerance"] = ("direct (fp64): element-wise rel_err (oracles.hpp:55-58) <= 1e-9" if direct else
                        "mixed: per gradient block norm-wise <= 5e-5 and element-wise rel_err (oracles.hpp:55-58) "
                        "<= 1e-3 (entries that are residues of cancelling sums), bound terms <= 1e-5")
    out["pass"] = bool(worst <= 1e-9) if direct else bool(worst_norm <= 5e-5 and worst <= 1e-3 and
                                                          out["bound_terms_max_rel"] <= 1e-5)
    return out


def run_reference(args, world, rank):
    """--impl reference: the reference's CPU path on all host cores.  The reference itself needs
    Eigen (absent here and on the GPU box), so this times the fp64 oracle port of Engine::evaluate(true)
    (std::thread workers, vectorised build) on the same Rng inputs the GPU arm uses."""
    if rank != 0:
        return
    latent, n, q, d, m, n_cpu, desc = WORKLOADS[args.config]
    threads = os.cpu_count() or 1
    beta = 100.0 if latent else 1.0
    mu, s, y, z = host_inputs(latent, n_cpu, q, d, m)
    w = min(n_cpu, 16384)  # warm-up on a leading slice (threads, page faults), untimed
    for _ in range(args.warmup):
        oracle_eval(latent, mu[:w], None if s is None else s[:w], y[:w], z, q, beta, threads)
    times = [oracle_eval(latent, mu, s, y, z, q, beta, threads)[0] for _ in range(args.steps)]
    t = float(np.mean(times))
    v = n_cpu / t
    sample = (f"full N = {n_cpu}" if n_cpu == n else f"the first {n_cpu} rows of the Rng stream (per-datapoint "
              f"cost is data-independent, PAPER.md:150)") + f"; {args.steps} timed evals; {cpu_desc(threads)}"
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": "f64", "data": "synthetic: " + INPUTS,
            "config": {"workload": desc, "N": n, "Q": q, "D": d, "M": m},
            "impl": "reference",
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample,
                             "note": "fp64 oracle restatement of Engine::evaluate(true) (oracle/sgp_oracle.cpp), "
                                     "-O3 -march=x86-64-v3 -ffast-math: libmvec SIMD exp and vectorised sums like "
                                     "Eigen's packet math"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_b200(args, world, rank, local_rank):
    import torch

    from paper_1410_4984_b200 import sgp, synthetic
    from paper_1410_4984_b200.engine_dist import DistributedEngine

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    dist = None
    use_dist = world > 1 or args.force_dist
    if use_dist:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    latent, n_cfg, q, d, m, n_cpu, desc = WORKLOADS[args.config]
    kind = sgp.ModelKind.latent if latent else sgp.ModelKind.regression
    if args.scaling == "weak":
        n_global = n_cfg * world
        row_begin, row_end = rank * n_cfg, (rank + 1) * n_cfg
    else:
        n_global = n_cfg
        row_begin, row_end = sgp.make_partition(n_global, world)[rank]
    n_local = row_end - row_begin
    stream = torch.cuda.Stream(dev)  # a capturable stream: the engine replays each evaluation as a CUDA graph
    torch.cuda.set_stream(stream)
    ctx = sgp.Context(local_rank)
    ctx.set_stream(stream.cuda_stream)
    # the reference generator's stream on the device; every rank generates the full dataset (weak
    # scaling: its own copy of the configuration's) and keeps its rows
    w = synthetic.make(latent, n_cfg if args.scaling == "weak" else n_global, q, d, m, seed=0, device=dev, ctx=ctx)
    r0 = 0 if args.scaling == "weak" else row_begin
    mu = w.mu[r0:r0 + n_local].t().contiguous().t()
    s = w.s[r0:r0 + n_local].t().contiguous().t() if latent else None
    y = w.y[r0:r0 + n_local].t().contiguous().t()
    z, kernel, beta = w.z, w.kernel, w.beta
    del w
    torch.cuda.synchronize(dev)

    if use_dist:
        eng = DistributedEngine(kind, mu, s, y, n_global, row_begin, precision=args.precision)
        eng.broadcast(kernel, beta, z)
        evaluate = lambda lh=False: eng.evaluate(True, local_to_host=lh)  # noqa: E731
        launch_count = eng.passes.launch_count
        target = eng
    else:
        single = sgp.Engine(kind, mu, s, y, ctx=ctx, precision=args.precision)
        single.broadcast(kernel, beta, z)
        evaluate = lambda lh=False: single.evaluate(True, local_to_host=lh)  # noqa: E731
        launch_count = ctx.launch_count
        target = single

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
    fwd_k, bwd_k, k2f, k2b, coord_s = [], [], [], [], []
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
            k2f.append(r.timing.psi2_fwd_kernel_s)
            k2b.append(r.timing.psi2_bwd_kernel_s)
            coord_s.append(r.timing.coordinator_s)
        barrier()
    launches = launch_count() - launches0
    step_ms = [a.elapsed_time(b) for a, b in zip(ev0, ev1)]
    total_s = max_over_ranks(sum(step_ms) * 1e-3)
    ms_per_step = total_s / args.steps * 1e3
    value = n_global / (total_s / args.steps)
    clk = clocks.summary()
    total_launches = int(sum_over_ranks(launches))
    mode = r.timing.precision

    # ---------------- roofline of the dominant kernel (the psi2 backward, this rank) ----------------
    fwd_flops, bwd_flops = algorithmic_flops(q, d, m)
    p = m * (m + 1) // 2
    t_peak, t_src = tensor_peak()
    k2b_s, k2f_s = float(np.mean(k2b)), float(np.mean(k2f))
    fwd_s, bwd_s = float(np.mean(fwd_k)), float(np.mean(bwd_k))
    psi2_bwd_alg = n_local * p * (11 * q + 4)
    roof = {
        "bound": "tensor", "kernel": ("rowtile_kernel<Q,0,0,NP> (psi2 backward, tcgen05)" if mode != "direct"
                                      else "dir_pair_bwd_kernel (psi2 backward, direct fp64)"),
        "achieved": psi2_bwd_alg / k2b_s / 1e12 if k2b_s > 0 else None, "peak": t_peak, "unit": "TFLOP/s",
        "frac": psi2_bwd_alg / k2b_s / 1e12 / t_peak if k2b_s > 0 else None, "traffic": None,
        "peak_source": t_src, "flops_per_launch": psi2_bwd_alg, "avg_launch_ms": k2b_s * 1e3,
        "work": "SURVEY.md 8(d) algorithmic flops of the psi2 backward, P(11Q+4) per datapoint (FMA = 2)",
    }
    if mode != "direct" and k2b_s > 0:
        mma = n_local * p * mma_flops_per_pair(q, mode)
        roof["executed_mma"] = {"tflops": mma / k2b_s / 1e12, "frac_of_peak": mma / k2b_s / 1e12 / t_peak,
                                "flops_per_launch": mma,
                                "note": "tensor-pipe work the kernel issues: MMA1 exponent pieces + MMA3 hi/lo "
                                        "contraction products"}
        exps = n_local * p
        roof["mufu_floor"] = {"exps_per_launch": exps, "floor_ms": exps / EX2_RATE * 1e3,
                              "frac": exps / EX2_RATE / k2b_s,
                              "note": "every exp2 on MUFU.EX2 (16/clk/SM at 1965 MHz)"}
    if mode == "syrk":  # the Knm-tile path: its backward pass (split tiles reused, GEMM, contraction)
        kk = (m + d + 3) // 4 * 4
        alg = 2.0 * n_local * m * (m + d)
        ex = 3 * 2.0 * n_local * m * kk
        tf32_peak = t_peak / 2
        roof = {
            "bound": "tensor", "kernel": "SYRK backward pass: split-TF32 G = [K|Y][2U; dPsi^T] GEMMs (cuBLAS, "
                                         "tcgen05) + syrk_reduce_kernel (H = G o K contractions)",
            "achieved": alg / bwd_s / 1e12 if bwd_s > 0 else None, "peak": tf32_peak, "unit": "TFLOP/s",
            "frac": alg / bwd_s / 1e12 / tf32_peak if bwd_s > 0 else None, "traffic": None,
            "peak_source": t_src + " / 2 (dense tf32 = half the bf16 rate)", "flops_per_launch": alg,
            "avg_launch_ms": bwd_s * 1e3,
            "work": "2 N M (M + D): the one exact GEMM the backward stands for (FMA = 2)",
            "executed_mma": {"tflops": ex / bwd_s / 1e12 if bwd_s > 0 else None,
                             "frac_of_peak": ex / bwd_s / 1e12 / tf32_peak if bwd_s > 0 else None,
                             "flops_per_launch": ex, "note": "three tf32 piece products, inner dimension "
                                                             "M + D padded to a multiple of 4"},
        }
    tpath = os.path.join(ROOT, "profiles", "r02_traffic.json")
    if os.path.exists(tpath):
        try:
            tj = json.load(open(tpath))
            if tj.get("config") == args.config and tj.get("n_local") == n_local and tj.get("mode") == mode:
                roof["traffic"] = tj.get("dram_bytes_per_launch")
                roof["traffic_source"] = tj.get("source")
        except Exception:
            pass
    passes = {"psi_fwd_ms": fwd_s * 1e3, "psi_bwd_ms": bwd_s * 1e3, "psi2_fwd_kernel_ms": k2f_s * 1e3,
              "psi2_bwd_kernel_ms": k2b_s * 1e3,
              "psi_passes_tflops": n_local * (fwd_flops + bwd_flops) / (fwd_s + bwd_s) / 1e12,
              "fp32_simt_frac": n_local * (fwd_flops + bwd_flops) / (fwd_s + bwd_s) / 1e12 / PEAK_FP32_TFLOPS,
              "fp32_simt_note": "SURVEY 8(d) FP32-FMA roofline (71.7 TF/s measured FFMA) of all psi kernels"}

    # ---------------- CPU baseline + parity (rank 0, N = 1 only) ----------------
    cpu, parity = None, None
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        n_c = min(n_cpu, n_local)
        mu_h = np.asfortranarray(mu[:n_c].cpu().numpy())
        s_h = np.asfortranarray(s[:n_c].cpu().numpy()) if latent else None
        y_h = np.asfortranarray(y[:n_c].cpu().numpy())
        if n_c == n_local:  # the timed evaluation itself, d_mu / d_S read back from the device
            r_cmp = r
            gmu, gs = target.local_grads() if latent else (None, None)
        else:  # the same leading rows on the GPU
            e_s = sgp.Engine(kind, mu_h, s_h, y_h, ctx=ctx, precision=args.precision)
            e_s.broadcast(kernel, beta, z)
            r_cmp = e_s.evaluate(True)
            gmu, gs = r_cmp.grads.d_mu, r_cmp.grads.d_s
        oracle_eval(latent, mu_h[:4096], None if s_h is None else s_h[:4096], y_h[:4096], z, q, beta, threads)
        t_cpu, ref = oracle_eval(latent, mu_h, s_h, y_h, z, q, beta, threads)
        cpu = {"value": n_c / t_cpu, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": (f"full N = {n_c}" if n_c == n_global else f"the first {n_c} rows of the Rng stream") +
                         f" of {args.config}, one timed fp64 Engine::evaluate(true) of the oracle port "
                         f"(std::thread workers, libmvec SIMD exp build); {cpu_desc(threads)}"}
        parity = parity_of(r_cmp, gmu, gs, ref, latent)
        parity["rows"] = n_c

    # ---------------- end to end through the public API ----------------
    # pinned host mu / S (column-major) uploaded every step by broadcast(); d_mu / d_S read back.
    h2d = d2h = 0
    mv = (m + 3) // 4 * 4
    if latent:
        mu_p = torch.empty(q, n_local, dtype=torch.float64, pin_memory=True)
        s_p = torch.empty(q, n_local, dtype=torch.float64, pin_memory=True)
        mu_p.copy_(mu.t())
        s_p.copy_(s.t())
        mu_np, s_np = mu_p.numpy().T, s_p.numpy().T  # Fortran-ordered views of pinned memory
        gmu_p = torch.empty(q, n_local, dtype=torch.float64, pin_memory=True)
        gs_p = torch.empty(q, n_local, dtype=torch.float64, pin_memory=True)
        target.set_local_grads_out(gmu_p.numpy().T, gs_p.numpy().T)
        h2d += 2 * n_local * q * 8
        d2h += 2 * n_local * q * 8
    h2d += m * q * 8 + mv * 12 * 4 + mv * mv * 4 + d * mv * 4
    d2h += (4 + m * (m + 1) // 2 + m * d) * 8 + (1 + q + m * q) * 8 + 8

    def e2e_step():
        if latent:
            target.broadcast(kernel, beta, z, mu_np, s_np)
        else:
            target.broadcast(kernel, beta, z)
        return evaluate(True)

    for _ in range(max(1, args.warmup // 2)):
        e2e_step()
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        r_e2e = e2e_step()
        _ = r_e2e.bound.total
    barrier()
    e2e_s = max_over_ranks(time.perf_counter() - t0)
    e2e_value = n_global / (e2e_s / args.steps)
    h2d_all, d2h_all = int(sum_over_ranks(h2d)), int(sum_over_ranks(d2h))

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": DTYPES.get(mode, mode), "precision": mode,
            "z_spread": r.timing.z_spread, "data": "synthetic: " + INPUTS,
            "config": {"workload": desc, "N": n_global, "Q": q, "D": d, "M": m},
            "layout": {"n_local": n_local, "parallelism": f"dp{world}",
                       "l2": "inputs > L2 and a 256 MB L2 flush before each timed step (untimed)"},
            "roofline": roof,
            "passes": passes,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d_all, "d2h_bytes_per_step": d2h_all,
                    "ms_per_step": e2e_s / args.steps * 1e3},
            "cpu_baseline": cpu,
            "parity": parity,
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
    ap.add_argument("--precision", default="auto", choices=["auto", "fast", "precise", "direct"])
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
