"""Host-to-host solving of a large parameter set (the reference's per-parameter
loop, experiment.py:149-157, as one streamed call).

Parameters are solved in device-resident sub-batches.  Each instance's solution
is copied to pinned host memory on a side stream as soon as it converges
(rbws_mgcg_solve_to_host), so downloads overlap the iterations of the
instances still running and the solve of the next sub-batch.  Two multigrid
contexts and two solution buffers alternate.
"""

from __future__ import annotations

import numpy as np

from . import _native
from .grid import BatchOperator, ParametricProblem, padded_len
from .krylov import SolveReports
from .multigrid import MgContext, mg_context_for
from .warmstart import MethodConfig, rbi_pcg_solve


def schedule(count: int, sub_batch: int, tail: int) -> list[int]:
    """Sub-batch sizes: full sub-batches, then halving down to ``tail`` so the
    download of the last (un-overlapped) sub-batch is short."""
    sizes, rem = [], int(count)
    while rem > 0:
        if rem > 2 * sub_batch:
            take = sub_batch
        elif rem > tail:
            take = max(tail, min(sub_batch, (rem + 1) // 2))
        else:
            take = rem
        sizes.append(take)
        rem -= take
    return sizes


class HostPipeline:
    """Solve ``mus`` (host array) into a pinned host buffer, sub-batch by sub-batch.

    ``out_host``: pinned float64 tensor with at least ``len(mus) * stride``
    elements; instance m's solution lands at ``out_host[m*stride : (m+1)*stride]`` in the
    problem's device layout: the padded n^3 block or, for problems with free
    boundary nodes (example-2), the (c+1)^3 full-node block (``stride`` attribute).
    Assembled problems (example-1, example-2) have parameter-dependent right-hand sides:
    each sub-batch's f(mu) is assembled on the host and uploaded inside the call.
    """

    def __init__(self, problem: ParametricProblem, method: MethodConfig, model=None,
                 sub_batch: int = 512, nu: int = 1, tail: int | None = None,
                 sizes: list[int] | None = None):
        import torch
        from .fem_fn import FnFemProblem
        _native.require_cuda()
        if sub_batch < 1:
            raise ValueError("sub_batch must be positive")
        self.problem, self.method, self.model, self.sub = problem, method, model, sub_batch
        self.tail = max(1, sub_batch // 4) if tail is None else max(1, int(tail))
        self.sizes = list(sizes) if sizes else None   # explicit sub-batch sizes (cycled)
        if self.sizes:
            sub_batch = max(sub_batch, max(self.sizes))
            self.sub = sub_batch
        n = problem.n
        self.nu = nu
        self.full_node = isinstance(problem, FnFemProblem)
        self.per_mu_rhs = self.full_node or getattr(problem, "stored", False)
        self.stride = problem.nodes() if self.full_node else n ** 3
        if self.full_node:  # FnMgContext is built per sub-batch (operators + plane factors)
            self.ctx = [None, None]
            self.x = [None, None]
            self.f = None
        else:
            self.ctx = [MgContext(problem, sub_batch, nu=nu) for _ in range(2)]
            self.x = [torch.empty(padded_len(n, sub_batch), dtype=torch.float64, device="cuda")
                      for _ in range(2)]
            self.f = None if self.per_mu_rhs else problem.rhs()
        # both streams are side streams: the legacy default stream would serialise
        # with the copies
        self.compute_stream = torch.cuda.Stream()
        self.copy_stream = torch.cuda.Stream()
        self.freed = [torch.cuda.Event() for _ in range(2)]
        self.solved = [torch.cuda.Event() for _ in range(2)]
        for ev in self.freed:
            ev.record()
        self.done = torch.cuda.Event()
        self._slot = 0

    def schedule(self, count: int) -> list[int]:
        if not self.sizes:
            return schedule(count, self.sub, self.tail)
        out, rem, i = [], int(count), 0
        while rem > 0:
            take = min(rem, self.sizes[i % len(self.sizes)])
            out.append(take)
            rem -= take
            i += 1
        return out

    def solve(self, mus, out_host, sync: bool = True):
        """Solve ``mus`` into ``out_host``; returns the SolveReports.

        sync=True: the caller's stream waits for every download (out_host is complete
        once the caller's stream reaches this point).  sync=False: only the compute is
        ordered before the caller's later work; the downloads finish on the copy stream
        (``done`` event) while the next call already computes — back-to-back calls then
        overlap one call's last downloads with the next call's solves.
        """
        import torch
        mus = np.ascontiguousarray(mus, dtype=np.float64)
        n3 = self.stride
        if out_host.numel() < len(mus) * n3 or not out_host.is_pinned():
            raise ValueError("out_host must be a pinned buffer of len(mus) * stride doubles")
        caller = torch.cuda.current_stream()
        compute = self.compute_stream
        compute.wait_stream(caller)
        reports = []
        with torch.cuda.stream(compute):
            reports = self._run(mus, out_host, compute, n3)
        caller.wait_stream(compute)
        self.done.record(self.copy_stream)
        if sync:
            caller.wait_stream(self.copy_stream)
        return reports

    def _run(self, mus, out_host, compute, n3):
        import torch
        reports = []
        c0 = 0
        for size in self.schedule(len(mus)):
            part = mus[c0:c0 + size]
            s = self._slot          # buffers alternate across calls too
            self._slot ^= 1
            compute.wait_event(self.freed[s])     # buffer s no longer being copied out
            m = len(part)
            if self.full_node:
                ctx = mg_context_for(self.problem, part, nu=self.nu)
                f = self.problem.rhs(part)
                x, reps = rbi_pcg_solve(BatchOperator(ctx), f, self.method, mg_ctx=ctx,
                                        l1roc_model=self.model)
                self.x[s] = x                        # kept alive until its copy is done
                done = torch.cuda.Event()
                done.record(compute)
                self.copy_stream.wait_event(done)
                with torch.cuda.stream(self.copy_stream):
                    out_host[c0 * n3:(c0 + m) * n3].copy_(x.reshape(-1), non_blocking=True)
                reports.append(reps)
                self.freed[s].record(self.copy_stream)
                c0 += size
                continue
            ctx = mg_context_for(self.problem, part, ctx=self.ctx[s])
            f = self.problem.rhs(part) if self.per_mu_rhs else self.f
            # each instance's solution streams to the host as soon as it converges,
            # overlapping the iterations of the instances still running
            x, reps = rbi_pcg_solve(BatchOperator(ctx), f, self.method, mg_ctx=ctx,
                                    l1roc_model=self.model, x0_out=self.x[s],
                                    out_host=out_host[c0 * n3:(c0 + m) * n3],
                                    copy_stream=self.copy_stream)
            reports.append(reps)
            self.freed[s].record(self.copy_stream)   # all downloads of buffer s enqueued
            c0 += size
        return SolveReports.concat(reports)
