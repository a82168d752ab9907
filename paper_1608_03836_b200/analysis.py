"""Evolution-operator spectra (R/pkg/src/wadg/analysis.py:22-123) on the device.

``assemble_evolution_matrix`` builds the dense matrix of the full
semi-discrete operator (mass inverse included) column by column: column j is
the right-hand side applied to the unit vector e_j.  As in the reference, the
unknowns are ordered in field blocks of K*Np: (p, u1, u2) in 2D, and
(p, u1, u2, u3) for tetrahedra.  Each column is one device RHS evaluation,
through ``wadg_volume`` + ``wadg_surface`` + ``wadg_mass_inverse``.  The unit
vector, the output and the matrix all stay on the GPU.  ``eigenspectrum`` is
the reference's dense eigen-solve on the host.
"""

from __future__ import annotations

import csv
import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native
from .solver import Discretization, MediumField


class SizeCapExceeded(Exception):
    """Operator assembly would exceed the configured unknown cap."""


class EigenSolveFailure(Exception):
    """Dense eigenvalue solve did not converge."""


@dataclass
class SpectrumResult:
    """Eigenvalues of the time-evolution operator, |lambda|-descending
    (R/.../analysis.py:65-85)."""

    eigenvalues: np.ndarray = field(repr=False)
    max_real_part: float = 0.0

    def __post_init__(self):
        order = np.argsort(-np.abs(self.eigenvalues))
        self.eigenvalues = self.eigenvalues[order]
        self.max_real_part = float(self.eigenvalues.real.max())

    @property
    def spectral_radius(self):
        return float(np.abs(self.eigenvalues[0]))

    def to_csv(self, path):
        with open(path, "w", newline="") as f:
            out = csv.writer(f)
            out.writerow(["re", "im"])
            for lam in self.eigenvalues:
                out.writerow([repr(lam.real), repr(lam.imag)])


def assemble_evolution_matrix(mesh, config, medium=MediumField(), cap=6000):
    """Dense matrix of the full semi-discrete operator (R/.../analysis.py:88-105).

    Column j is ``rhs_full`` applied to e_j. The ordering is field blocks of
    K*Np, element-major within a block, as in the reference. The columns are
    assembled on the device, and the result is returned as a host float64
    array (n, n)."""
    disc = Discretization(mesh, config, medium)
    d = disc.dev
    K, Np, fld = mesh.K, disc.ref.Np, disc.dim + 1
    n = fld * K * Np
    if n > cap:
        raise SizeCapExceeded(f"{n} unknowns exceed cap {cap}")
    Z = d.empty_fields()
    pre = d.empty_fields()
    out = d.empty_fields()
    A = torch.empty((n, n), dtype=torch.float64, device=d.device)
    s = d.struct
    sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    vp = lambda t: ctypes.c_void_p(t.data_ptr())
    for j in range(n):
        c, rem = divmod(j, K * Np)
        k, i = divmod(rem, Np)
        Z[c, i, k] = 1.0
        _native.call("wadg_volume", ctypes.byref(s), vp(Z), vp(pre), sp)
        _native.call("wadg_surface", ctypes.byref(s), vp(Z), vp(pre), disc.flux.tau_p, disc.flux.tau_u,
                     1, 0, -1, sp)
        _native.call("wadg_mass_inverse", ctypes.byref(s), vp(pre), vp(out), sp)
        A[:, j] = out[:, :, :K].permute(0, 2, 1).reshape(-1)
        Z[c, i, k] = 0.0
    return A.cpu().numpy()


def eigenspectrum(matrix):
    """All eigenvalues of the assembled evolution matrix (R/.../analysis.py:108-117)."""
    try:
        lam = np.linalg.eigvals(matrix)
    except np.linalg.LinAlgError as exc:
        raise EigenSolveFailure(str(exc)) from exc
    if np.any(~np.isfinite(lam)):
        raise EigenSolveFailure("non-finite eigenvalues")
    return SpectrumResult(eigenvalues=lam)
