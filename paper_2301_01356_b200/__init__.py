"""B200-native FAST-BCC biconnected components (arXiv 2301.01356).

Drop-in for the reference package's BCC entry point and its public stage
operations (/root/reference/pkg/src/fastbcc): ``fast_bcc``, ``BccLabeling``,
``articulation_points``, ``extract_bccs``, ``connected_components``,
``list_ranking``, ``build_euler_tour``, ``compute_tags``, ``skeleton_record``,
``Graph``, ``symmetrize``, ``load_bin``/``write_bin``.  Every stage of the hot
path -- spanning forest, Euler-tour rooting, subtree tags, fence
classification, skeleton connectivity, labelling -- is a hand-written sm_100a
kernel in ``libfastbcc_b200.so`` (C ABI: include/fastbcc_b200.h).  No CPU
fallback.
"""

from .bcc import BccLabeling, Plan, StepTimings, articulation_points, extract_bccs, fast_bcc, run_device
from .graphs import Graph, load_bin, symmetrize, write_bin
from .stages import (CCResult, EdgeClass, EdgeList, RootedForest, VertexTags, build_euler_tour, classify_edges,
                     compute_tags, compute_w, connected_components, extract_bccs_device, is_ancestor, list_ranking,
                     skeleton_record, symmetrize_device)

__version__ = "0.2.0"

__all__ = [
    "BccLabeling",
    "CCResult",
    "EdgeClass",
    "EdgeList",
    "Graph",
    "Plan",
    "RootedForest",
    "StepTimings",
    "VertexTags",
    "articulation_points",
    "build_euler_tour",
    "classify_edges",
    "compute_tags",
    "compute_w",
    "connected_components",
    "extract_bccs",
    "extract_bccs_device",
    "fast_bcc",
    "is_ancestor",
    "list_ranking",
    "load_bin",
    "run_device",
    "skeleton_record",
    "symmetrize",
    "symmetrize_device",
    "write_bin",
    "__version__",
]
