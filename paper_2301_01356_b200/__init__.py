"""B200-native FAST-BCC biconnected components (arXiv 2301.01356).

Drop-in for the reference package's BCC entry point
(/root/reference/pkg/src/fastbcc: ``fast_bcc``, ``BccLabeling``,
``articulation_points``, ``extract_bccs``, ``Graph``, ``symmetrize``), with
every stage of the hot path -- spanning forest, Euler-tour rooting, subtree
tags, fence classification, skeleton connectivity, labelling -- as
hand-written sm_100a kernels in ``libfastbcc_b200.so`` (C ABI:
include/fastbcc_b200.h).  No CPU fallback.
"""

from .bcc import BccLabeling, StepTimings, articulation_points, extract_bccs, fast_bcc, run_device
from .graphs import Graph, symmetrize

__version__ = "0.1.0"

__all__ = [
    "BccLabeling",
    "Graph",
    "StepTimings",
    "articulation_points",
    "extract_bccs",
    "fast_bcc",
    "run_device",
    "symmetrize",
    "__version__",
]
