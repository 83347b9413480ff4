"""B200-native Falkon hot path (arXiv 2006.10350): fused Knm^T(Knm v), fp64 preconditioner,
device-side preconditioned CG, behind the C ABI of include/falkon.h (libfalkon.so).

The Python layer is argument marshalling only (binding.py) plus multi-rank plumbing
(parallel.py).  All arithmetic of the method runs in libfalkon's sm_100a kernels.
"""
from . import binding  # noqa: F401
from .binding import (Context, FalkonError, GAUSSIAN, LAPLACIAN, PATH_AUTO, PATH_SIMT,  # noqa: F401
                      PATH_TENSOR, get_unique_id, load)

__all__ = ["binding", "Context", "FalkonError", "GAUSSIAN", "LAPLACIAN", "PATH_AUTO",
           "PATH_SIMT", "PATH_TENSOR", "get_unique_id", "load"]
