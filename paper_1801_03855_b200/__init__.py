"""B200-native tensor-collective hot path of MXNET-MPI (arXiv 1801.03855).

The product is the C-ABI library ``libtc.so`` (include/tc.h; CUDA sources in ``csrc/``) and the
thin ctypes binding in :mod:`paper_1801_03855_b200.tc`.  Importing this package loads libtc.so and
raises if it has not been built -- there is no CPU fallback.
"""
from .tc import (  # noqa: F401
    Comm, Group, Plan, TcError, allreduce, sgd_step, easgd_update, easgd_async_update, esgd_step,
    broadcast, LIB, LIB_PATH, STATUS,
    BucketedStep,
)
