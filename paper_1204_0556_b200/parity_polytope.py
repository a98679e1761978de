"""Parity-polytope projection on the GPU.

:func:`project_batch` is the drop-in for the reference's
``polylp.project_batch`` (parity_polytope.py:352-421): same argument, same
``ValueError`` cases, fp64 result as a numpy array.  It runs the same
register-resident projection the decoder's check-node pass uses
(csrc/projection.cuh), one thread per row.

:func:`membership` is the drop-in for ``polylp.membership``
(parity_polytope.py:69-91), the verification helper the reference uses for
feasibility at convergence (tests/test_admm.py:147-168); it runs the
batched membership kernel (csrc/steps.cu), as :func:`membership_rows_device`
does for whole CUDA tensors of rows (e.g. every check's replicas of a batch).
"""

from __future__ import annotations

import numpy as np
import torch
from numpy.typing import ArrayLike, NDArray

from . import _lib

PARITY_TOL = 1e-9  # parity_polytope.py:19 (fp64 mode)


def project_rows_device(values: torch.Tensor) -> torch.Tensor:
    """Project every row of a CUDA tensor ([m, d], float32 or float64)."""
    if values.ndim != 2 or values.shape[1] == 0:
        raise ValueError("project_batch expects an (m, d) array with d >= 1")
    if values.dtype not in (torch.float32, torch.float64):
        raise ValueError("project_batch supports float32 and float64")
    v = values.contiguous()
    out = torch.empty_like(v)
    dt = _lib.ADMM_F64 if v.dtype == torch.float64 else _lib.ADMM_F32
    st = torch.cuda.current_stream(v.device)
    _lib.check(_lib.load().admm_project_batch(dt, v.shape[0], v.shape[1], v.data_ptr(),
                                              out.data_ptr(), st.cuda_stream))
    return out


def project_batch(values: ArrayLike) -> NDArray[np.float64]:
    """Row-wise parity-polytope projection of an (m, d) array (fp64)."""
    vals = np.asarray(values, dtype=float)
    if vals.ndim != 2 or vals.shape[1] == 0:
        raise ValueError("project_batch expects an (m, d) array with d >= 1")
    if not np.all(np.isfinite(vals)):
        raise ValueError("projection input must be finite")
    if vals.shape[0] == 0:
        return vals.copy()
    out = project_rows_device(torch.from_numpy(np.ascontiguousarray(vals)).cuda())
    return out.cpu().numpy()


def membership_rows_device(values: torch.Tensor, tol: float = PARITY_TOL) -> torch.Tensor:
    """Membership of every row of a CUDA tensor ([m, d]) in PP_d within
    ``tol`` -> bool tensor [m] (admm_membership_batch)."""
    if values.ndim != 2 or values.shape[1] == 0:
        raise ValueError("membership expects a non-empty 1-D vector per row")
    if values.dtype not in (torch.float32, torch.float64):
        raise ValueError("membership supports float32 and float64")
    v = values.contiguous()
    out = torch.empty(v.shape[0], dtype=torch.uint8, device=v.device)
    dt = _lib.ADMM_F64 if v.dtype == torch.float64 else _lib.ADMM_F32
    st = torch.cuda.current_stream(v.device)
    _lib.check(_lib.load().admm_membership_batch(dt, v.shape[0], v.shape[1], v.data_ptr(), float(tol),
                                                 out.data_ptr(), st.cuda_stream))
    return out.bool()


def membership(u: ArrayLike, tol: float = PARITY_TOL) -> bool:
    """Test whether ``u`` lies in the parity polytope within ``tol``
    (parity_polytope.py:69-91; majorisation characterisation)."""
    u = np.asarray(u, dtype=float)
    if u.ndim != 1 or u.size == 0:
        raise ValueError("membership expects a non-empty 1-D vector")
    t = torch.from_numpy(np.ascontiguousarray(u[None, :])).cuda()
    return bool(membership_rows_device(t, tol)[0].item())


def membership_batch(values: ArrayLike, tol: float = PARITY_TOL) -> NDArray[np.bool_]:
    """Row-wise :func:`membership` of an (m, d) array."""
    vals = np.asarray(values, dtype=float)
    if vals.ndim != 2 or vals.shape[1] == 0:
        raise ValueError("membership expects a non-empty 1-D vector per row")
    if vals.shape[0] == 0:
        return np.zeros(0, dtype=bool)
    return membership_rows_device(torch.from_numpy(np.ascontiguousarray(vals)).cuda(), tol).cpu().numpy()
