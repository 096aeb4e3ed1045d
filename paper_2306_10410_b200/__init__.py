"""paper_2306_10410_b200 -- BOBA (Batched Order By Attachment, arXiv
2306.10410) on NVIDIA B200: first-occurrence ranking, linear-time rank
compaction, relabel, stable COO->CSR and fp32 CSR SpMV as sm_100a CUDA
kernels behind a C ABI (include/boba_b200.h, libboba_b200.so).

The public names below mirror the reference package's hot path
(/root/reference/pkg/src/boba: graph.py, ordering.py, kernels.py,
_parallel.py) so the package is a drop-in for it; ``device`` exposes the
same phases on device-resident CUDA tensors.
"""

from .errors import BobaError, MalformedGraphError, ParseError, UndefinedMetricError
from .graph import (CooGraph, CsrGraph, Permutation, apply_permutation, coo_to_csr, degrees, sort_coo_by_destination,
                    total_degrees)
from .kernels import pagerank, spmv_pull
from .metrics import nbr
from .ordering import (
    ORDERING_CHOICES,
    RANK_UNSET,
    BobaOrder,
    DegreeOrder,
    HubOrder,
    IdentityOrder,
    RandomOrder,
    boba_parallel,
    boba_sequential,
    compute_ordering,
    degree_order,
    hub_order,
    identity_order,
    random_order,
)
from . import _native  # noqa: F401  (fails loudly if libboba_b200.so is missing)

__version__ = "0.1.0"

__all__ = [
    "BobaError", "MalformedGraphError", "ParseError", "UndefinedMetricError",
    "CooGraph", "CsrGraph", "Permutation", "apply_permutation", "coo_to_csr", "degrees",
    "total_degrees", "sort_coo_by_destination", "spmv_pull", "pagerank", "nbr", "RANK_UNSET", "ORDERING_CHOICES", "boba_parallel", "boba_sequential",
    "compute_ordering", "random_order", "identity_order", "degree_order", "hub_order", "BobaOrder", "RandomOrder",
    "IdentityOrder", "DegreeOrder", "HubOrder",
    "__version__",
]
