"""Multi-rank Engine: one process per GPU, N sharded by make_partition.

Mirrors sgp::Engine's collect/broadcast protocol (proj/include/sgp/parallel.hpp:370-450)
with the in-process ``reduce_reports`` (parallel.hpp:222-258) replaced by two
NCCL allreduces over NVLink (torch.distributed, backend "nccl"):

    psi forward kernel (shard)          -> packed partial stats   [phi, yy, n, KL, Phi(P), Psi(MxD)]
    all_reduce #1 (sum, fp64)
    coordinator on every rank, redundantly (factor_gram, bound_core, adjoints) -- no broadcast needed
    psi backward kernel (shard)         -> packed partial grads   [d_variance, d_l(Q), d_Z(MxQ)]
    all_reduce #2 (sum, fp64)
    gradient assembly (kern_grads(Z,Z,dKmm) + jitter term); d_mu / d_s stay on the owning rank.

The orchestration is independent of where the passes run: ``CudaPasses`` drives
libsgpx on the rank's GPU (the product); the CPU multi-process tests plug in
the oracle as the pass implementation (test infrastructure) and exercise this
same code with the gloo backend.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L
from . import sgp
from ._lib import check


class _CudaArray:
    """Zero-copy __cuda_array_interface__ over a device fp64 vector owned by libsgpx."""

    def __init__(self, ptr: int, n: int, stream: int | None):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False), "version": 3,
                                         "strides": None, "stream": stream if stream else None}


class CudaPasses:
    """The product pass implementation: libsgpx engine phases on this rank's GPU.

    The context runs on torch's current CUDA stream so NCCL (torch.distributed) and
    the psi kernels are ordered on one stream without extra synchronisation.
    """

    def __init__(self, kind, x_or_mu, s, y, n_global, row_begin, jitter_factor=1e-6, device=None,
                 precision="auto"):
        import torch

        self.torch = torch
        dev = torch.cuda.current_device() if device is None else device
        self.ctx = sgp.Context(dev)
        self.stream = torch.cuda.current_stream(dev)
        self.ctx.set_stream(self.stream.cuda_stream)
        self.eng = sgp.Engine(kind, x_or_mu, s, y, ctx=self.ctx, _n_global=n_global, _row_begin=row_begin,
                              jitter_factor=jitter_factor, precision=precision)
        self.kind = sgp.ModelKind(kind)
        self._lib = L.load()

    def broadcast(self, kernel, beta, z, mu=None, s=None):
        self.eng.broadcast(kernel, beta, z, mu, s)

    def stats_pass(self):
        ptr, cnt = C.c_void_p(), C.c_int64()
        check(self._lib.sgpx_engine_stats_pass(self.eng._h, C.byref(ptr), C.byref(cnt)))
        return self.torch.as_tensor(_CudaArray(ptr.value, cnt.value, self.stream.cuda_stream), device="cuda")

    def coordinate(self, reduced_stats, with_grads: bool):
        # the allreduce wrote in place into libsgpx's buffer; the engine reads it from there
        check(self._lib.sgpx_engine_coordinate(self.eng._h, 1 if with_grads else 0))

    def grad_pass(self):
        ptr, cnt = C.c_void_p(), C.c_int64()
        check(self._lib.sgpx_engine_grad_pass(self.eng._h, C.byref(ptr), C.byref(cnt)))
        return self.torch.as_tensor(_CudaArray(ptr.value, cnt.value, self.stream.cuda_stream), device="cuda")

    def finish(self, reduced_grads, with_grads: bool, local_to_host: bool = True) -> sgp.EvalResult:
        r, bufs = self.eng._result_buffers()
        check(self._lib.sgpx_engine_finish(self.eng._h, C.byref(r)))
        return self.eng._pack(r, bufs, with_grads, local_to_host)

    def launch_count(self):
        return self.ctx.launch_count()


class DistributedEngine:
    """sgp::Engine over torch.distributed ranks (one shard per rank).

    ``passes`` defaults to ``CudaPasses`` built from the shard rows; ``group`` is the
    process group (default WORLD).  All ranks must call broadcast/evaluate together.
    """

    def __init__(self, kind, x_or_mu_local, s_local, y_local, n_global: int, row_begin: int, group=None,
                 passes=None, jitter_factor: float = 1e-6, precision: str = "auto"):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.kind = sgp.ModelKind(kind)
        self.n_global = n_global
        self.row_begin = row_begin
        self.n_local = y_local.shape[0]
        self.passes = passes or CudaPasses(kind, x_or_mu_local, s_local, y_local, n_global, row_begin,
                                           jitter_factor=jitter_factor, precision=precision)

    @staticmethod
    def shard_of(n_global: int, rank: int, world: int):
        """This rank's rows under make_partition (parallel.hpp:28-41)."""
        return sgp.make_partition(n_global, world)[rank]

    def broadcast(self, kernel: sgp.KernelSpec, beta: float, z, mu=None, s=None):
        self.passes.broadcast(kernel, beta, z, mu, s)

    def set_local_grads_out(self, dmu, ds):
        self.passes.eng.set_local_grads_out(dmu, ds)

    def local_grads(self, out=None):
        return self.passes.eng.local_grads(out)

    def evaluate(self, with_grads: bool = True, local_to_host: bool = True) -> sgp.EvalResult:
        eng = getattr(self.passes, "eng", None)
        if eng is not None and with_grads and local_to_host and self.kind == sgp.ModelKind.latent:
            eng._register_grads_out()  # d_mu / d_S stream to the host during the gradient pass
        packed = self.passes.stats_pass()
        self.dist.all_reduce(packed, op=self.dist.ReduceOp.SUM, group=self.group)  # allreduce #1
        self.passes.coordinate(packed, with_grads)
        grads = None
        if with_grads:
            grads = self.passes.grad_pass()
            self.dist.all_reduce(grads, op=self.dist.ReduceOp.SUM, group=self.group)  # allreduce #2
        return self.passes.finish(grads, with_grads, local_to_host)
