"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no Hamiltonian, no Liouvillian,
no ordering, no factorisation, no Krylov step).  It only carries

  * the parameter sets of BASELINE.json ``configs`` (the paper's workloads are
    parameter points of Eq. (1)/(3), so the "input" of the path is a parameter
    set; sec. IV, Figs. 3-5 use the same kind of parameter points), and
  * a counter-based, seeded generator of random complex vectors/parameter
    jitter used by parity tests of the individual kernels.

Both ``oracle/`` and ``paper_1411_4356_b200/`` consumers read these; neither
imports the other.
"""
from __future__ import annotations

from dataclasses import dataclass, replace, asdict
import math

import numpy as np


@dataclass(frozen=True)
class Params:
    """Physical + numerical parameters of one steady-state problem.

    Symbols follow PAPER.md Eq. (1) (H/hbar = -Delta a^+a + omega_m b^+b
    + g0 (b+b^+) a^+a + E (a+a^+)) and Eq. (3) (kappa D[a],
    Gamma_m (1+n_th) D[b], Gamma_m n_th D[b^+]); N_c, N_m are the Fock cut-offs
    (sec. III); w is the trace weight of Eq. (5) (None -> the paper's sec. IV
    rule, the mean of the diagonal of the Liouvillian); drop_tol / fill_factor
    are the ILUT d, p of sec. II and permtol the pivoting threshold of its iLUTP (R13);
    restart / tol are the GMRES(m) settings.
    """
    N_c: int
    N_m: int
    omega_m: float
    Delta: float
    kappa: float
    g0: float
    E: float
    Gamma_m: float
    n_th: float
    w: float | None = None
    drop_tol: float = 1e-4
    fill_factor: float = 20.0
    permtol: float = 0.01         # iLUTP column-exchange threshold (R13)
    restart: int = 30
    tol: float = 1e-10
    max_iter: int = 2000

    @property
    def hilbert_dim(self) -> int:
        return self.N_c * self.N_m

    @property
    def liouvillian_dim(self) -> int:
        return self.hilbert_dim ** 2

    def with_(self, **kw) -> "Params":
        return replace(self, **kw)

    def as_dict(self) -> dict:
        return asdict(self)


# BASELINE.json configs[0..3] (verbatim numbers); configs[4] is the sweep below.
CONFIGS: dict[str, Params] = {
    "tiny": Params(N_c=4, N_m=10, omega_m=1.0, Delta=-0.5, kappa=0.3, g0=0.4, E=0.1,
                   Gamma_m=1e-3, n_th=0.0, w=1.0, drop_tol=1e-4, fill_factor=20,
                   restart=30, tol=1e-10),
    "small": Params(N_c=6, N_m=30, omega_m=1.0, Delta=-1.0, kappa=0.5, g0=0.6, E=0.3,
                    Gamma_m=1e-3, n_th=0.5, w=None, drop_tol=1e-4, fill_factor=30,
                    restart=30, tol=1e-10),
    "medium": Params(N_c=10, N_m=60, omega_m=1.0, Delta=0.0, kappa=1.0, g0=1.0, E=0.5,
                     Gamma_m=1e-4, n_th=1.0, w=None, drop_tol=1e-5, fill_factor=50,
                     restart=50, tol=1e-10),
    "large": Params(N_c=12, N_m=120, omega_m=1.0, Delta=-1.0, kappa=0.5, g0=1.0, E=0.4,
                    Gamma_m=1e-4, n_th=0.0, w=None, drop_tol=1e-5, fill_factor=80,
                    restart=50, tol=1e-9),
}
CONFIG_ORDER = ["tiny", "small", "medium", "large", "sweep"]

SWEEP_POINTS = 64
# configs[4] gives no d, p: d = 1e-5 (configs[3]'s), p = 100 (the paper's own detuning
# sweep, Fig. 4(a-d)); R15 has the study behind the choice.
SWEEP_BASE = Params(N_c=8, N_m=60, omega_m=1.0, Delta=0.0, kappa=0.5, g0=0.8, E=0.3,
                    Gamma_m=1e-4, n_th=0.2, w=None, drop_tol=1e-5, fill_factor=100,
                    restart=40, tol=1e-10)


def sweep_params(points: int = SWEEP_POINTS, lo: float = -2.0, hi: float = 2.0,
                 base: Params = SWEEP_BASE) -> list[Params]:
    """BASELINE.json configs[4]: Delta uniformly spaced in [lo, hi] (inclusive)."""
    if points == 1:
        return [base.with_(Delta=lo)]
    return [base.with_(Delta=lo + (hi - lo) * k / (points - 1)) for k in range(points)]


def shard(items: list, rank: int, world: int) -> list:
    """Contiguous block sharding of independent units over ranks."""
    n = len(items)
    lo = (n * rank) // world
    hi = (n * (rank + 1)) // world
    return items[lo:hi]


def rand_cvec(n: int, seed: int) -> np.ndarray:
    """Seeded complex128 vector with i.i.d. N(0,1) real and imaginary parts."""
    g = np.random.Generator(np.random.Philox(seed))
    return g.standard_normal(n) + 1j * g.standard_normal(n)


def jittered(p: Params, seed: int, rel: float = 0.1) -> Params:
    """A seeded random parameter point near ``p`` (same truncation/structure)."""
    g = np.random.Generator(np.random.Philox(seed))
    f = lambda x: float(x * (1.0 + rel * (2.0 * g.random() - 1.0)))
    return p.with_(Delta=f(p.Delta) if p.Delta != 0 else float(rel * (2 * g.random() - 1)),
                   kappa=f(p.kappa), g0=f(p.g0), E=f(p.E))


def tiny_params(N_c: int, N_m: int, **kw) -> Params:
    """Convenience constructor for small oracle/parity cases."""
    base = dict(omega_m=1.0, Delta=-0.5, kappa=0.3, g0=0.4, E=0.1, Gamma_m=1e-3,
                n_th=0.5, w=None, drop_tol=1e-4, fill_factor=20, restart=30, tol=1e-10)
    base.update(kw)
    return Params(N_c=N_c, N_m=N_m, **base)


assert math.isclose(CONFIGS["large"].g0 / CONFIGS["large"].kappa, 2.0)
