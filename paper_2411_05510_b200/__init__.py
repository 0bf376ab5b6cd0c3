"""B200-native hot path of RSVD-accelerated CoV-SSI (arXiv 2411.05510).

The compute lives in libssi.so (csrc/, sm_100a CUDA behind the C ABI of include/ssi.h);
this package is the ctypes binding (api) and the record / lag-sweep / batch drivers.
"""
from . import api, drivers  # noqa: F401
from .api import (covariances, toeplitz, rsvd, modal_sweep, stab3d, PoleTable, Criteria,  # noqa: F401
                  philox_words, gaussian_sketch)
from .drivers import SweepParams, Engine, identify_record  # noqa: F401
