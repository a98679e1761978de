"""ctypes binding of the C ABI in ``include/admm_b200.h``.

The shared library ``libadmm_b200.so`` is built in-tree (``make`` or
``__graft_entry__.build()``).  There is no fallback: if the library is
missing, every entry point raises ``RuntimeError`` -- the decoder never
silently runs anywhere but the CUDA kernels.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libadmm_b200.so"

ADMM_F32 = 0
ADMM_F64 = 1
ADMM_FLAG_CONVERGED = 1
ADMM_FLAG_INTEGRAL = 2
ADMM_FLAG_CODEWORD = 4
ENGINES = {"auto": 0, "resident": 1, "streaming": 3, "cluster": 4, "wide": 5}
#: Kernel ids of admm_decode_kernel (enum admm_kernel).
KERNELS = {1: "resident", 2: "regular", 3: "sharded", 4: "cluster", 5: "wide"}

#: Every symbol the public header declares (checked by the CPU test-suite).
EXPORTED = (
    "admm_version",
    "admm_build_flags",
    "admm_checked_probe",
    "admm_last_error",
    "admm_graph_create",
    "admm_graph_create_ex",
    "admm_graph_destroy",
    "admm_graph_get_info",
    "admm_workspace_bytes",
    "admm_decode_kernel",
    "admm_decode_batch",
    "admm_decode_synth",
    "admm_synth_llr",
    "admm_project_batch",
    "admm_phase_profile",
    "admm_wide_phase_profile",
    "admm_cluster_phase_profile",
    "admm_bp_decode_batch",
    "admm_x_update",
    "admm_z_update",
    "admm_lambda_update",
    "admm_membership_batch",
)


class Channel(ctypes.Structure):
    """struct admm_channel (include/admm_b200.h)."""

    _fields_ = [("kind", ctypes.c_int32), ("p", ctypes.c_double), ("snr_db", ctypes.c_double),
                ("rate", ctypes.c_double)]


class GraphInfo(ctypes.Structure):
    _fields_ = [
        ("n_vars", ctypes.c_int32), ("n_checks", ctypes.c_int32), ("n_edges", ctypes.c_int32),
        ("max_check_degree", ctypes.c_int32), ("max_var_degree", ctypes.c_int32),
        ("engine", ctypes.c_int32), ("degree_bucket", ctypes.c_int32),
        ("checks_per_thread", ctypes.c_int32), ("threads_per_cta", ctypes.c_int32),
        ("ctas_per_sm_f32", ctypes.c_int32), ("ctas_per_sm_f64", ctypes.c_int32),
        ("smem_bytes_f32", ctypes.c_int32), ("smem_bytes_f64", ctypes.c_int32),
        ("regs_f32", ctypes.c_int32), ("regs_f64", ctypes.c_int32),
        ("num_sms", ctypes.c_int32), ("cluster_size", ctypes.c_int32),
        ("layout_cost_before", ctypes.c_double), ("layout_cost_after", ctypes.c_double),
        ("cluster_active", ctypes.c_int32), ("cluster_threads", ctypes.c_int32), ("cluster_smem", ctypes.c_int32),
        ("cluster_regs", ctypes.c_int32), ("cluster_exchange", ctypes.c_int64),
    ]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


_lib = None


def load() -> ctypes.CDLL:
    """Load (once) and return the library; raise if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("ADMM_B200_LIB", str(LIB_PATH))
    if not Path(path).exists():
        raise RuntimeError(
            f"CUDA extension {path} is not built; run `make` (or __graft_entry__.build()). "
            "The decoder has no CPU fallback.")
    lib = ctypes.CDLL(path)
    P, I32, I64, SZ, D = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t, ctypes.c_double
    lib.admm_version.restype = ctypes.c_int
    lib.admm_build_flags.restype = ctypes.c_int
    lib.admm_checked_probe.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
    lib.admm_checked_probe.restype = ctypes.c_int
    lib.admm_last_error.restype = ctypes.c_char_p
    lib.admm_graph_create.argtypes = [ctypes.c_int, I32, I32, P, P, ctypes.POINTER(P)]
    lib.admm_graph_create.restype = ctypes.c_int
    lib.admm_graph_create_ex.argtypes = [ctypes.c_int, I32, I32, P, P, ctypes.c_int, ctypes.POINTER(P)]
    lib.admm_graph_create_ex.restype = ctypes.c_int
    lib.admm_graph_destroy.argtypes = [P]
    lib.admm_graph_destroy.restype = ctypes.c_int
    lib.admm_graph_get_info.argtypes = [P, ctypes.POINTER(GraphInfo)]
    lib.admm_graph_get_info.restype = ctypes.c_int
    lib.admm_workspace_bytes.argtypes = [P, ctypes.c_int, I64]
    lib.admm_workspace_bytes.restype = SZ
    lib.admm_decode_kernel.argtypes = [P, ctypes.c_int, I64]
    lib.admm_decode_kernel.restype = ctypes.c_int
    lib.admm_decode_batch.argtypes = [
        P, ctypes.c_int, I64, P, I64, D, D, I32, D,
        P, I64, P, I64, P, P, P,
        P, P, P, P, I64, P, SZ, P,
    ]
    lib.admm_decode_batch.restype = ctypes.c_int
    lib.admm_decode_synth.argtypes = [
        P, ctypes.c_int, I64, ctypes.POINTER(Channel), ctypes.c_uint64, ctypes.c_uint32, I64, D, D, I32, D,
        P, I64, P, I64, P, P, P, P, SZ, P,
    ]
    lib.admm_decode_synth.restype = ctypes.c_int
    lib.admm_synth_llr.argtypes = [ctypes.c_int, I64, I32, ctypes.POINTER(Channel), ctypes.c_uint64,
                                   ctypes.c_uint32, I64, P, I64, P]
    lib.admm_synth_llr.restype = ctypes.c_int
    lib.admm_phase_profile.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_uint64)]
    lib.admm_phase_profile.restype = ctypes.c_int
    lib.admm_wide_phase_profile.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_uint64)]
    lib.admm_wide_phase_profile.restype = ctypes.c_int
    lib.admm_cluster_phase_profile.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_uint64)]
    lib.admm_cluster_phase_profile.restype = ctypes.c_int
    lib.admm_project_batch.argtypes = [ctypes.c_int, I64, I32, P, P, P]
    lib.admm_project_batch.restype = ctypes.c_int
    lib.admm_bp_decode_batch.argtypes = [
        P, ctypes.c_int, I64, P, I64, I32, D, I32,
        P, I64, P, I64, P, I64, P, P, P, P, SZ, P,
    ]
    lib.admm_bp_decode_batch.restype = ctypes.c_int
    lib.admm_x_update.argtypes = [P, ctypes.c_int, I64, P, P, I64, P, I64, D, P, I64, P]
    lib.admm_x_update.restype = ctypes.c_int
    lib.admm_z_update.argtypes = [P, ctypes.c_int, I64, P, I64, P, P, I64, D, D, P, P, P]
    lib.admm_z_update.restype = ctypes.c_int
    lib.admm_lambda_update.argtypes = [P, ctypes.c_int, I64, P, P, P, I64, D, P, P]
    lib.admm_lambda_update.restype = ctypes.c_int
    lib.admm_membership_batch.argtypes = [ctypes.c_int, I64, I32, P, D, P, P]
    lib.admm_membership_batch.restype = ctypes.c_int
    _lib = lib
    return lib


def check(rc: int) -> None:
    if rc != 0:
        msg = load().admm_last_error().decode(errors="replace")
        if rc == -1:
            raise ValueError(msg)
        raise RuntimeError(f"admm_b200 error {rc}: {msg}")
