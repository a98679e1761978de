"""Parity-polytope projection on the GPU.

:func:`project_batch` is the drop-in for the reference's
``polylp.project_batch`` (parity_polytope.py:352-421): same argument, same
``ValueError`` cases, fp64 result as a numpy array.  It runs the same
register-resident projection the decoder's check-node pass uses
(csrc/projection.cuh), one thread per row.
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
