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


def assemble_evolution_matrix(mesh, config, medium=MediumField(), cap=6000, batch=None):
    """Dense matrix of the full semi-discrete operator (R/.../analysis.py:88-105).

    Column j is ``rhs_full`` applied to e_j. The ordering is field blocks of
    K*Np, element-major within a block, as in the reference. Columns are
    assembled in batches: the mesh is replicated ``batch`` times
    (``meshgen.replicate_mesh``), copy b carries the unit vector of column
    j0 + b, and one device RHS pass (``wadg_volume`` + ``wadg_surface`` +
    ``wadg_mass_inverse``) yields the whole batch. The result is returned as a
    host float64 array (n, n)."""
    from . import meshgen
    K, fld = mesh.K, mesh.shape.dim + 1
    probe = Discretization(mesh, config, medium)
    Np = probe.ref.Np
    n = fld * K * Np
    if n > cap:
        raise SizeCapExceeded(f"{n} unknowns exceed cap {cap}")
    B = int(batch or max(1, min(n, (1 << 17) // max(K, 1))))
    disc = Discretization(meshgen.replicate_mesh(mesh, B), config, medium)
    d = disc.dev
    Z, pre, out = d.empty_fields(), d.empty_fields(), d.empty_fields()
    A = torch.empty((n, n), dtype=torch.float64, device=d.device)
    s = d.struct
    sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    vp = lambda t: ctypes.c_void_p(t.data_ptr())
    for j0 in range(0, n, B):
        nb = min(B, n - j0)
        js = torch.arange(j0, j0 + nb, device=d.device)
        c, rem = js // (K * Np), js % (K * Np)
        Z.zero_()
        Z[c, rem % Np, torch.arange(nb, device=d.device) * K + rem // Np] = 1.0
        _native.call("wadg_volume", ctypes.byref(s), vp(Z), vp(pre), sp)
        _native.call("wadg_surface", ctypes.byref(s), vp(Z), vp(pre), disc.flux.tau_p, disc.flux.tau_u,
                     1, 0, -1, sp)
        _native.call("wadg_mass_inverse", ctypes.byref(s), vp(pre), vp(out), sp)
        cols = out[:, :, :nb * K].reshape(fld, Np, nb, K).permute(2, 0, 3, 1).reshape(nb, n)
        A[:, j0:j0 + nb] = cols.T.to(torch.float64)
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
