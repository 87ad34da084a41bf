"""Drop-in of the reference's ``pxst.integration`` (integration.py:1-140):
least-squares integration of 2-D gradient fields on masked grids.

``integrate_gradient`` / ``project_irrotational`` run the conjugate-gradient
solve on the device (``pxst_integrate_gradient``, regularize.cu); ``grad``
and ``curl`` are the elementwise finite differences of the reference,
kept on the host for the numpy boundary.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native
from ._native import PxstCgInfo, check, stream_ptr


def grad(phi: np.ndarray) -> np.ndarray:
    """[2, SS, FS] forward differences, last row/column backward (integration.py:19-31)."""
    phi = np.asarray(phi, dtype=np.float64)
    out = np.empty((2,) + phi.shape)
    out[0, :-1] = phi[1:] - phi[:-1]
    out[0, -1] = phi[-1] - phi[-2]
    out[1, :, :-1] = phi[:, 1:] - phi[:, :-1]
    out[1, :, -1] = phi[:, -1] - phi[:, -2]
    return out


def curl(dx: np.ndarray, dy: np.ndarray) -> np.ndarray:
    """Discrete curl on interior cells (integration.py:137-139)."""
    return (dy[1:, :-1] - dy[:-1, :-1]) - (dx[:-1, 1:] - dx[:-1, :-1])


def linked_components(mask: np.ndarray) -> int:
    """Number of 4-connected components of the mask with at least one link.

    On a component without the anchor the fit is defined up to a constant;
    plain CG from zero returns the zero-sum one (its Krylov space excludes
    constants), which the multigrid-preconditioned solver does not preserve,
    so "auto" keeps plain CG for masks with more than one such component."""
    from scipy import ndimage
    lab, n = ndimage.label(np.asarray(mask, dtype=bool))
    if n <= 1:
        return n
    sizes = np.bincount(lab.ravel())[1:]
    return int(np.count_nonzero(sizes >= 2))


@dataclass
class IntegrationResult:
    phi: np.ndarray
    converged: bool
    residual: float
    iterations: int


def integrate_gradient(gx: np.ndarray, gy: np.ndarray, mask: np.ndarray, tol: float = 1e-12,
                       maxiter: int | None = None, solver: str = "cg") -> IntegrationResult:
    """Potential whose gradient best fits (gx, gy) on the mask (integration.py:61-118),
    solved on the GPU; zero at the first mask pixel.  ``solver="cg"`` runs the
    reference's plain CG (same iteration semantics); ``"mgcg"`` preconditions
    it with an aggregation-multigrid V-cycle (same stopping rule on |r|/|b|,
    far fewer iterations; on masks with several linked components it may
    return another least-squares solution, differing by a constant on the
    components without the anchor); ``"auto"`` picks "mgcg" when that cannot
    happen."""
    import torch
    from .engine import _device, to_device, to_host
    mask = np.asarray(mask, dtype=bool)
    if not mask.any():
        raise ValueError("integrate_gradient: mask has no good pixels")
    ss, fs = mask.shape
    lib = _native.lib()
    dev = _device()
    gx_t = to_device(np.asarray(gx), np.float64, dev)
    gy_t = to_device(np.asarray(gy), np.float64, dev)
    m_t = to_device(mask.astype(np.uint8), np.uint8, dev)
    phi = torch.empty((ss, fs), dtype=torch.float64, device=dev)
    info = PxstCgInfo()
    if solver not in ("cg", "mgcg", "auto"):
        raise ValueError("solver must be 'cg', 'mgcg' or 'auto'")
    if solver == "auto":
        solver = "mgcg" if linked_components(mask) <= 1 else "cg"
    check(lib.pxst_integrate_gradient(gx_t.data_ptr(), gy_t.data_ptr(), m_t.data_ptr(), ss, fs,
                                      float(tol), int(maxiter or 0), int(solver == "mgcg"),
                                      phi.data_ptr(), ctypes.byref(info), stream_ptr()))
    return IntegrationResult(phi=to_host(phi), converged=bool(info.converged),
                             residual=float(info.residual), iterations=int(info.iterations))


def project_irrotational(dx: np.ndarray, dy: np.ndarray, mask: np.ndarray, tol: float = 1e-12,
                         maxiter: int | None = None, solver: str = "cg"):
    """Nearest curl-free field on the mask (integration.py:121-134): (grad(phi), result)."""
    result = integrate_gradient(dx, dy, mask, tol=tol, maxiter=maxiter, solver=solver)
    return grad(result.phi), result
