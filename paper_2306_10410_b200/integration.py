"""Rebind the reference package's hot path onto the B200 kernels.

``patch_reference(boba)`` takes the imported reference package (the module
object of ``/root/reference/pkg/src/boba`` or an installed copy) and rebinds:

* the plain-array seam ``boba._parallel`` (reference _parallel.py:1-5; its
  callers look functions up at call time, ordering.py:140-147 and
  graph.py:268) to this package's ``_parallel`` -- same names, signatures and
  int64 results;
* the name-imported structural ops: ``apply_permutation``,
  ``coo_to_csr`` and ``spmv_pull`` in every reference module that imported
  them, returning the reference's own container types;
* the §8f neighbours: ``total_degrees``, ``sort_coo_by_destination``,
  ``degree_order`` and ``hub_order`` (so ``compute_ordering('degree'|'hub')``
  and the ``DegreeOrder``/``HubOrder`` transformers run on the GPU too) and
  ``pagerank`` (kernels.py:57-107).

After patching, the reference's own pipeline (``run_bench``) and tests run on
the GPU.  ``unpatch`` restores the originals.  See INTEGRATION.md.
"""

from __future__ import annotations

from . import _parallel as gpu_parallel
from . import graph as gpu_graph
from . import kernels as gpu_kernels
from . import ordering as gpu_ordering

_SEAM = ("first_hit_order_sequential", "first_hit_chunked", "first_hit_racy", "first_hit_sequential",
         "run_racy_first_hit", "compact_ranks", "scatter_rows")
_saved: dict = {}


def patch_reference(boba) -> None:
    ref_graph = boba.graph

    def apply_permutation(g, p):
        if p.n != g.n:
            raise boba.MalformedGraphError(f"permutation size {p.n} does not match vertex count {g.n}")
        out = gpu_graph.apply_permutation(g, p)
        return ref_graph.CooGraph(g.n, out.I, out.J, g.weights, validate=False)

    def coo_to_csr(g):
        out = gpu_graph.coo_to_csr(g)
        return ref_graph.CsrGraph(g.n, out.offsets, out.indices, out.weights, validate=False)

    def spmv_pull(csr, x):
        return gpu_kernels.spmv_pull(csr, x)

    def pagerank(csr, damping=0.85, tol=1e-6, max_iters=100, return_iterations=False):
        return gpu_kernels.pagerank(csr, damping, tol, max_iters, return_iterations)

    def total_degrees(g):
        return gpu_graph.total_degrees(g)

    def sort_coo_by_destination(g):
        out = gpu_graph.sort_coo_by_destination(g)
        return ref_graph.CooGraph(g.n, out.I, out.J, out.weights, validate=False)

    def degree_order(g):
        p = gpu_ordering.degree_order(g)
        return ref_graph.Permutation(p.order, p.label)

    def hub_order(g):
        p = gpu_ordering.hub_order(g)
        return ref_graph.Permutation(p.order, p.label)

    par = boba._parallel
    for name in _SEAM:
        _saved.setdefault((par, name), getattr(par, name))
        setattr(par, name, getattr(gpu_parallel, name))
    repl = {"apply_permutation": apply_permutation, "coo_to_csr": coo_to_csr, "spmv_pull": spmv_pull,
            "total_degrees": total_degrees, "sort_coo_by_destination": sort_coo_by_destination,
            "degree_order": degree_order, "hub_order": hub_order, "pagerank": pagerank}
    for modname in ("graph", "ordering", "bench", "metrics", "kernels", "io", "cli"):
        mod = getattr(boba, modname, None)
        if mod is None:
            continue
        for name, fn in repl.items():
            if hasattr(mod, name):
                _saved.setdefault((mod, name), getattr(mod, name))
                setattr(mod, name, fn)
    for name, fn in repl.items():
        if hasattr(boba, name):
            _saved.setdefault((boba, name), getattr(boba, name))
            setattr(boba, name, fn)


def unpatch() -> None:
    for (mod, name), fn in _saved.items():
        setattr(mod, name, fn)
    _saved.clear()
