"""B200-native deflated PGMRES (arXiv 1906.04051 linear-solve path).

The product is libpgmres.so (hand-written sm_100a CUDA + C ABI, see
include/pgmres.h); this package is the host-side mirror of the reference's
solver API over that ABI.
"""
from .dgmres import (CsrMatrix, DeflationConfig, DeflationRecord, Deflator, DeviceCsr,
                     DeviceError, DeviceExecutor, GmresConfig, GmresError, GmresReport,
                     InnerRecord, LoopbackGroup, NewtonConfig, NewtonIterRecord,
                     NewtonReport, deflated_gmres, gmres_restarted, nccl_unique_id,
                     newton_solve)

__all__ = [
    "CsrMatrix", "DeflationConfig", "DeflationRecord", "Deflator", "DeviceCsr", "DeviceError",
    "DeviceExecutor", "GmresConfig", "GmresError", "GmresReport", "InnerRecord",
    "LoopbackGroup", "NewtonConfig", "NewtonIterRecord", "NewtonReport", "deflated_gmres",
    "gmres_restarted", "nccl_unique_id", "newton_solve",
]
