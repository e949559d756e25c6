"""world_size-2 gloo tests of the multi-rank engine orchestration (CPU, and on the GPU with the product passes).

DistributedEngine (paper_1410_4984_b200/engine_dist.py) runs unchanged: partition,
allreduce #1 of the packed statistics, the product's fp64 coordinator on every
rank, allreduce #2 of the packed global gradients, gradient assembly.  In the CPU
test the per-shard passes are served by the CPU oracle (OraclePasses, test
infrastructure); the GPU test runs the product passes (CudaPasses: libsgpx's
kernels on cuda:0 in both processes) with the same gloo exchanges.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT, norm_rel_err, rel_err


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class OraclePasses:
    """Shard passes on the CPU oracle, packed in the libsgpx allreduce layouts."""

    def __init__(self, kind, x, s, y, n_global):
        import oracle
        from paper_1410_4984_b200 import sgp

        self.o, self.sgp = oracle, sgp
        self.latent = int(kind) == 1
        self.x, self.s, self.y, self.n_global = x, s, y, n_global

    def broadcast(self, kernel, beta, z, mu=None, s=None):
        self.kernel, self.beta, self.z = kernel, beta, np.asfortranarray(z)
        if mu is not None:
            self.x, self.s = mu, s

    def stats_pass(self):
        st, _ = self.o.sweep_stats(self.latent, self.x, self.s if self.latent else None, self.y, self.z,
                                   self.kernel.variance, self.kernel.lengthscales)
        kl = 0.5 * np.sum(self.s + self.x ** 2 - np.log(self.s) - 1.0) if self.latent else 0.0
        return torch.from_numpy(self.sgp.pack_stats(st.phi, st.yy, st.n_count, kl, st.phi_big, st.psi_y))

    def coordinate(self, reduced, with_grads):
        self.co = self.sgp.coordinate_host(1 if self.latent else 0, self.n_global, self.y.shape[1], reduced.numpy(),
                                           self.z, self.kernel, self.beta, adjoints=with_grads)
        self.reduced_stats = reduced.numpy().copy()

    def grad_pass(self):
        co = self.co
        _, g = self.o.sweep_stats(self.latent, self.x, self.s if self.latent else None, self.y, self.z,
                                  self.kernel.variance, self.kernel.lengthscales,
                                  adj=(co["d_phi"], co["d_psi_y"], co["d_phi_big"]))
        if self.latent:
            self.d_mu = g.d_mu - self.x
            self.d_s = g.d_s - 0.5 * (1.0 - 1.0 / self.s)
        return torch.from_numpy(np.concatenate([[g.d_variance], g.d_lengthscales, g.d_z.ravel(order="F")]))

    def finish(self, reduced, with_grads, local_to_host=True):
        dz, dv, dls = self.sgp.finish_host(reduced.numpy(), self.z, self.kernel, self.co["d_kmm"],
                                           self.co["jitter_factor"])
        return dict(bound=self.co["bound"], d_z=dz, d_variance=dv, d_lengthscales=dls, d_beta=self.co["d_beta"],
                    d_mu=getattr(self, "d_mu", None), stats=self.reduced_stats)


def _worker(rank, world, port, latent, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import sys

    sys.path.insert(0, ROOT)
    from paper_1410_4984_b200 import sgp
    from paper_1410_4984_b200.engine_dist import DistributedEngine

    dist.init_process_group("gloo", rank=rank, world_size=world)
    x, s, y, z, var, ls, beta = _problem()
    n = y.shape[0]
    b, e = DistributedEngine.shard_of(n, rank, world)
    kind = sgp.ModelKind.latent if latent else sgp.ModelKind.regression
    passes = OraclePasses(kind, x[b:e], s[b:e], y[b:e], n)
    eng = DistributedEngine(kind, x[b:e], s[b:e], y[b:e], n, b, passes=passes)
    eng.broadcast(sgp.KernelSpec(var, ls), beta, z)
    r = eng.evaluate(True)
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), total=r["bound"].total, d_z=r["d_z"], d_variance=r["d_variance"],
             d_ls=r["d_lengthscales"], d_beta=r["d_beta"], d_mu=r["d_mu"] if latent else np.zeros(1), b=b, e=e,
             stats=r["stats"])
    dist.destroy_process_group()


def _problem():
    rng = np.random.default_rng(9)
    n, q, d, m = 301, 3, 4, 9
    x = rng.normal(size=(n, q))
    s = rng.uniform(0.25, 1.0, (n, q))
    y = rng.normal(size=(n, d))
    z = x[rng.choice(n, m, replace=False)] + 0.01
    return x, s, y, z, 1.2, rng.uniform(0.5, 2.0, q), 30.0


@pytest.mark.parametrize("latent", [True, False])
def test_two_rank_engine_matches_single_process(orc, tmp_path, latent):
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), latent, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    x, s, y, z, var, ls, beta = _problem()
    ref = orc.engine_evaluate(latent, x, s, y, z, var, ls, beta, workers=world)
    res = [np.load(tmp_path / f"r{r}.npz") for r in range(world)]
    for r in res:  # every rank ran the coordinator redundantly and agrees with the reference protocol
        assert rel_err(float(r["total"]), ref.bound["total"]) < 1e-10
        assert rel_err(r["d_z"], ref.d_z) < 1e-10
        assert rel_err(float(r["d_variance"]), ref.d_variance) < 1e-10
        assert rel_err(r["d_ls"], ref.d_lengthscales) < 1e-10
        assert rel_err(float(r["d_beta"]), ref.d_beta) < 1e-10
        if latent:
            b, e = int(r["b"]), int(r["e"])
            assert rel_err(r["d_mu"], ref.d_mu[b:e]) < 1e-10  # local gradients stay on the owning rank
    assert np.array_equal(res[0]["stats"], res[1]["stats"])  # allreduce gave both ranks identical stats


def _cuda_worker(rank, world, port, latent, precision, out_dir):
    """One rank of the product path: CudaPasses (libsgpx kernels on cuda:0) under DistributedEngine,
    the two exchanges over gloo with CUDA tensors (no kernel waits on another rank's kernels: each
    allreduce is host-mediated between the passes)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import sys

    sys.path.insert(0, ROOT)
    from paper_1410_4984_b200 import sgp
    from paper_1410_4984_b200.engine_dist import DistributedEngine

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    x, s, y, z, var, ls, beta = _cuda_problem(latent, precision)
    n = y.shape[0]
    b, e = DistributedEngine.shard_of(n, rank, world)
    kind = sgp.ModelKind.latent if latent else sgp.ModelKind.regression
    eng = DistributedEngine(kind, x[b:e], s[b:e] if latent else None, y[b:e], n, b, precision=precision)
    eng.broadcast(sgp.KernelSpec(var, ls), beta, z)
    r = eng.evaluate(True)
    np.savez(os.path.join(out_dir, f"c{rank}.npz"), total=r.bound.total, d_z=r.grads.d_z,
             d_variance=r.grads.d_variance, d_ls=r.grads.d_lengthscales, d_beta=r.grads.d_beta,
             d_mu=r.grads.d_mu if latent else np.zeros(1), b=b, e=e, precision=r.timing.precision)
    dist.destroy_process_group()


def _cuda_problem(latent, precision):
    if precision == "auto":  # the bench's generator (sgp::Rng stream, init_gplvm Z), as the C2 / C3 tests
        import sys

        sys.path.insert(0, ROOT)
        from paper_1410_4984_b200 import synthetic

        w = synthetic.make(latent, 20_011, 10, 8, 50, seed=3)
        return (np.asarray(w.mu), None if w.s is None else np.asarray(w.s), np.asarray(w.y), np.asarray(w.z),
                w.variance, np.asarray(w.lengthscales), w.beta)
    rng = np.random.default_rng(21)
    n, q, d, m = 20_011, 6, 5, 40
    x = rng.normal(size=(n, q))
    s = rng.uniform(0.25, 1.0, (n, q))
    y = rng.normal(size=(n, d))
    z = x[rng.choice(n, m, replace=False)] + 0.01
    return x, s, y, z, 1.3, rng.uniform(0.7, 1.6, q), 25.0


@pytest.mark.gpu
@pytest.mark.parametrize("latent,precision", [(True, "direct"), (True, "auto"), (False, "auto")])
def test_two_rank_cuda_passes_match_oracle(orc, tmp_path, latent, precision):
    """world_size-2 run of the product passes (engine_dist.CudaPasses on cuda:0 in two processes,
    gloo exchanges) against the oracle engine with the same two workers (parallel.hpp:370-450)."""
    world = 2
    mp.start_processes(_cuda_worker, args=(world, _free_port(), latent, precision, str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    x, s, y, z, var, ls, beta = _cuda_problem(latent, precision)
    ref = orc.engine_evaluate(latent, x, s if latent else None, y, z, var, ls, beta, workers=world)
    res = [np.load(tmp_path / f"c{r}.npz") for r in range(world)]
    tight = str(res[0]["precision"]) == "direct"
    # direct: fp64 throughout; mixed modes: the engine tests' contract (element-wise 1e-3, norm-wise 5e-5)
    tb, te, tn = (1e-10, 1e-9, 1e-9) if tight else (1e-7, 1e-3, 5e-5)
    for r in res:
        assert rel_err(float(r["total"]), ref.bound["total"]) < tb
        pairs = dict(d_z=(r["d_z"], ref.d_z), d_ls=(r["d_ls"], ref.d_lengthscales),
                     d_var=([float(r["d_variance"])], [ref.d_variance]), d_beta=([float(r["d_beta"])], [ref.d_beta]))
        if latent:
            b, e = int(r["b"]), int(r["e"])
            pairs["d_mu"] = (r["d_mu"], ref.d_mu[b:e])
        for k, (a, w) in pairs.items():
            assert rel_err(a, w) < te, k
            assert norm_rel_err(a, w) < tn, k
    assert float(res[0]["total"]) == float(res[1]["total"])  # the redundant coordinators agree bitwise
