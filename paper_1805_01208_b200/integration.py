"""The reference-side shim: route a `geopart` installation's
partition entry points (`geopart/kmeans.py:502-534`) to the B200 ones.

`install(namespace)` replaces `balanced_kmeans_points` and `balanced_kmeans` in the
given module namespace (the reference's `geopart.kmeans` globals when called from the
one-line shim at the end of that module; every loaded `geopart.*` module that already
bound the names when called with no argument). Results come back as the reference's
own `geopart.graph.Partition` (and the stats as this package's `KMeansStats`, which has
the reference's fields), so code that type-checks the result -- e.g.
`fileio.write_partition`'s `isinstance(partition, Partition)` (`fileio.py:274-276`) --
keeps working.

`install_formats()` does the same for the formats and metrics either side of the path
(SURVEY §8(f) item 4): `geopart.fileio.load_metis_graph / load_coords / read_partition /
write_partition`, `geopart.metrics.edge_cut / comm_volumes / block_diameter_lower_bounds /
evaluate` and `geopart.graph.GeometricGraph.validate` run on the GPU and hand back the
reference's own types and exception classes.
"""

from __future__ import annotations

import sys

NAMES = ("balanced_kmeans_points", "balanced_kmeans")


def _to_reference(result, ref_partition_cls):
    from .types import Partition

    def conv(p):
        if ref_partition_cls is None or not isinstance(p, Partition):
            return p
        return ref_partition_cls(assignment=p.assignment, k=p.k,
                                 balance_failed=p.balance_failed, empty_blocks=p.empty_blocks)

    if isinstance(result, tuple):
        return (conv(result[0]),) + tuple(result[1:])
    return conv(result)


def wrap(fn, ref_partition_cls=None, counter: dict | None = None, name: str | None = None):
    """`fn` (a B200 entry point) returning the reference's Partition type."""

    def wrapped(*a, **kw):
        if counter is not None:
            counter[name] = counter.get(name, 0) + 1
        return _to_reference(fn(*a, **kw), ref_partition_cls)

    wrapped.__name__ = fn.__name__
    wrapped.__doc__ = fn.__doc__
    wrapped.__wrapped__ = fn
    return wrapped


def install(namespace: dict | None = None, counter: dict | None = None) -> dict:
    """Swap the entry points; returns {name: replaced reference function}."""
    from . import kmeans as bk

    try:
        from geopart.graph import Partition as RefPartition
    except ImportError:  # no reference installation: plain B200 results
        RefPartition = None
    replaced = {}
    if namespace is not None:
        for name in NAMES:
            replaced[name] = namespace.get(name)
            namespace[name] = wrap(getattr(bk, name), RefPartition, counter, name)
        return replaced
    import geopart.kmeans as rk

    for name in NAMES:
        ref_fn = getattr(rk, name)
        replaced[name] = ref_fn
        new = wrap(getattr(bk, name), RefPartition, counter, name)
        for mod in list(sys.modules.values()):
            if getattr(mod, "__name__", "").split(".")[0] == "geopart" and \
                    getattr(mod, name, None) is ref_fn:
                setattr(mod, name, new)
    return replaced


# ---------------------------------------------------------------- formats and metrics
FORMAT_NAMES = {
    "fileio": ("load_metis_graph", "load_coords", "read_partition", "write_partition"),
    "metrics": ("edge_cut", "comm_volumes", "block_diameter_lower_bounds", "evaluate"),
}


def _bridge(fn, counter, name, convert):
    """`fn` with this package's exceptions re-raised as the reference's classes and the
    result passed through `convert`."""
    import geopart.fileio as rf
    import geopart.graph as rg

    from . import fileio as bf
    from .types import GraphError

    def wrapped(*a, **kw):
        if counter is not None:
            counter[name] = counter.get(name, 0) + 1
        try:
            return convert(fn(*a, **kw))
        except bf.MetisParseError as e:
            raise rf.MetisParseError(str(e)) from None
        except GraphError as e:
            raise rg.GraphError(str(e)) from None

    wrapped.__name__ = name
    wrapped.__doc__ = fn.__doc__
    wrapped.__wrapped__ = fn
    return wrapped


def install_formats(counter: dict | None = None) -> dict:
    """Swap the reference's readers, partition writer, metrics and graph validation for
    the B200 ones in every loaded `geopart.*` module; returns what was replaced."""
    import geopart.fileio as rf
    import geopart.graph as rg
    import geopart.metrics as rm

    from . import fileio as bf
    from . import graph as bg
    from . import metrics as bm
    from .types import Partition

    def ref_graph(g):
        if not isinstance(g, bg.GeometricGraph):
            return g
        return rg.GeometricGraph(g.offsets, g.neighbors, g.coords, g.vertex_weights,
                                 g.edge_weights)

    def ref_partition(p):
        if not isinstance(p, Partition):
            return p
        return rg.Partition(assignment=p.assignment, k=p.k, balance_failed=p.balance_failed,
                            empty_blocks=p.empty_blocks)

    def ref_report(r):
        if not isinstance(r, bm.MetricsReport):
            return r
        return rm.MetricsReport(**{f: getattr(r, f) for f in r.__dataclass_fields__})

    convert = {"load_metis_graph": ref_graph, "read_partition": ref_partition,
               "evaluate": ref_report}
    replaced = {}
    for modname, names in FORMAT_NAMES.items():
        ref_mod, b200_mod = {"fileio": (rf, bf), "metrics": (rm, bm)}[modname]
        for name in names:
            ref_fn = getattr(ref_mod, name)
            replaced[f"{modname}.{name}"] = ref_fn
            new = _bridge(getattr(b200_mod, name), counter, name,
                          convert.get(name, lambda x: x))
            for mod in list(sys.modules.values()):
                if getattr(mod, "__name__", "").split(".")[0] == "geopart" and \
                        getattr(mod, name, None) is ref_fn:
                    setattr(mod, name, new)

    def validate(self):
        bg.GeometricGraph(self.offsets, self.neighbors, self.coords, self.vertex_weights,
                          self.edge_weights).validate()

    replaced["graph.GeometricGraph.validate"] = rg.GeometricGraph.validate
    rg.GeometricGraph.validate = _bridge(validate, counter, "GeometricGraph.validate",
                                         lambda x: x)
    return replaced
