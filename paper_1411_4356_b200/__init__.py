"""paper_1411_4356_b200 -- B200-native steady states of driven, damped optomechanics.

The hot path of arXiv:1411.4356: restarted GMRES on the reverse
Cuthill-McKee permuted, trace-constrained Liouvillian L~ (Eq. (5)), left-
preconditioned by a dual-threshold incomplete LU (sec. II-IV), as hand-written
CUDA for sm_100a behind the C ABI of include/ss_b200.h.  This package is the thin
Python face of that library: PyTorch supplies device memory and streams
(``torch.cuda``) and process groups (``sweep.py``); every step of the method runs in
libss_b200.so.  There is no CPU fallback.
"""
from __future__ import annotations

from . import _lib
from ._lib import (SSError, ss_build, ss_setup, ss_solve, ss_expect, ss_get_rho, ss_solve_host,
                   ss_destroy, ss_sizes, ss_export_matrix, ss_export_perm, ss_export_colperm, ss_export_factors, ss_spmv,
                   ss_precond, ss_kernel_launches, ss_debug_trace_trsv, ss_ilutp_host, ss_set_sm_budget, ss_debug_poison_smem)

__all__ = ["SteadyState", "SSError", "ss_build", "ss_setup", "ss_solve", "ss_expect", "ss_get_rho",
           "ss_solve_host", "ss_destroy", "ss_sizes", "ss_export_matrix", "ss_export_perm", "ss_export_colperm",
           "ss_export_factors", "ss_spmv", "ss_precond", "ss_kernel_launches", "ss_debug_trace_trsv",
           "ss_ilutp_host", "ss_set_sm_budget", "ss_debug_poison_smem"]


class SteadyState:
    """One Liouvillian on the current CUDA device.

    ``SteadyState(params).setup().solve()`` runs ss_build -> ss_setup -> ss_solve;
    ``rho()`` returns the density matrix as a complex128 torch tensor on the device,
    ``expect()`` the observables (<a^+a>, <b^+b>).
    """

    def __init__(self, params, stream=None, sm_budget: int = 0):
        import torch
        if not torch.cuda.is_available():
            raise SSError(2, "no CUDA device: the B200 path has no CPU fallback")
        _lib.load()
        self.params = params
        self.torch = torch
        self.stream = stream if stream is not None else torch.cuda.current_stream()
        self.handle, self.build_info = ss_build(params, self.stream.cuda_stream)
        if sm_budget:
            ss_set_sm_budget(self.handle, sm_budget)
        self.setup_info = None
        self.solve_info = None

    def setup(self, drop_tol: float | None = None, fill_factor: float | None = None,
              permtol: float | None = None, threads: int = 0):
        p = self.params
        self.setup_info = ss_setup(self.handle, p.drop_tol if drop_tol is None else drop_tol,
                                   p.fill_factor if fill_factor is None else fill_factor,
                                   p.permtol if permtol is None else permtol, threads)
        return self

    def solve(self, restart: int | None = None, tol: float | None = None, max_iter: int | None = None):
        p = self.params
        self.solve_info = ss_solve(self.handle, p.restart if restart is None else restart,
                                   p.tol if tol is None else tol, p.max_iter if max_iter is None else max_iter)
        return self

    @property
    def n(self) -> int:
        return self.build_info["n"]

    def rho(self):
        """Density matrix (N x N complex128, device); vec(rho) is column stacking (Eq. (4))."""
        N = self.build_info["hilbert_dim"]
        flat = self.torch.empty(N * N, dtype=self.torch.complex128, device="cuda")
        ss_get_rho(self.handle, flat.data_ptr(), True)
        return flat.view(N, N).t()       # column-major buffer -> rho[i, j]

    def expect(self) -> tuple[float, float]:
        return ss_expect(self.handle)

    def spmv(self, x):
        y = self.torch.empty_like(x)
        ss_spmv(self.handle, x.data_ptr(), y.data_ptr())
        return y

    def precond(self, x, which: int = 2):
        y = self.torch.empty_like(x)
        ss_precond(self.handle, which, x.data_ptr(), y.data_ptr())
        return y

    def close(self):
        if getattr(self, "handle", None):
            ss_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
