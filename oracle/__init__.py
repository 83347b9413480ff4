"""CPU fp64 oracle for the Falkon hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this package.  See falkon_oracle.py for the citations and pins.
"""
from .falkon_oracle import *  # noqa: F401,F403
from .falkon_oracle import (GAUSSIAN, LAPLACIAN, DEFAULT_JITTER, NotPositiveDefinite,  # noqa: F401
                            NonFinite)
from . import gsc_oracle as gsc  # noqa: F401,E402  (Alg. 2, GSC-Falkon / LogFalkon)
from . import multi_oracle as multi  # noqa: F401,E402  (multi-output, NEXT-3)
