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
