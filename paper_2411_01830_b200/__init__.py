"""B200-native FaaSTube data-passing layer (arxiv 2411.01830).

Drop-in for the reference's data-passing path:

* decision side — ``topology``, ``nvlink_sched``, ``pcie_sched``, ``simcore``,
  ``datastore``, ``dataplane``, ``strategies``, ``stage_sched``: the
  reference's module names and APIs, computed by libfaastube (C++);
* byte side — ``device`` (VMM pool, sm_100a copy kernels, CE legs) and
  ``tube`` (the Listing-1 put/get API: ``unique_id`` / ``store`` / ``fetch``).

Nothing here falls back to Python or to the CPU: without the built
``libfaastube.so`` every call raises ``LibraryMissing``.
"""

from ._lib import (LIB, CudaError, DuplicateStore, HardPressure, InfeasibleDemand, LibraryMissing, MissingData,
                   TopologyError)

__version__ = "0.1.0"

__all__ = ["LIB", "CudaError", "DuplicateStore", "HardPressure", "InfeasibleDemand", "LibraryMissing",
           "MissingData", "TopologyError", "lib_path"]


def lib_path() -> str:
    from ._lib import LIB_PATH
    return LIB_PATH
