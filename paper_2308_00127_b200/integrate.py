"""Drop-in for an installed reference package (``hetsched``).

The reference's consumers resolve ``fitness`` / ``decode`` (and the bound
helpers) as module globals at call time (heuristics.py:164, 186, 270, 286,
297, 318, 327, 330; bounds.py:106, 171, 195, 198, 204-205, 218, 224), so
re-binding those globals routes best-device, MET, SA, (1+1) EA and the
lower bound through the B200 evaluator without touching their code. The
wrappers translate errors and results into the reference's own types
(``hetsched.core.GraphError``, ``Schedule``, ``ScheduledBatch``).
"""
from __future__ import annotations

from typing import Callable


def patch_reference() -> Callable[[], None]:
    """Rebind hetsched.heuristics.{fitness, decode} and
    hetsched.bounds.{critical_path_bound, dep_subgraph, pre_subgraph};
    returns a function that restores the originals."""
    import hetsched.bounds as RB
    import hetsched.core as RC
    import hetsched.heuristics as RH

    from . import bounds as B
    from . import heuristics as H
    from .core import GraphError

    def _wrap(fn):
        def call(*a, **k):
            try:
                return fn(*a, **k)
            except GraphError as exc:
                raise RC.GraphError(str(exc)) from None
        call.__name__ = fn.__name__
        call.__doc__ = fn.__doc__
        return call

    def decode(genome, g, hw, table, L):
        s = _wrap(H.decode)(genome, g, hw, table, L)
        if s is None:
            return None
        return RC.Schedule(
            batches=tuple(RC.ScheduledBatch(task=b.task, device=b.device,
                                            size=b.size, inputs=b.inputs,
                                            start=b.start)
                          for b in s.batches),
            objective=s.objective, input_count=s.input_count)

    saved = {(RH, "fitness"): RH.fitness, (RH, "decode"): RH.decode,
             (RB, "critical_path_bound"): RB.critical_path_bound,
             (RB, "dep_subgraph"): RB.dep_subgraph,
             (RB, "pre_subgraph"): RB.pre_subgraph}
    RH.fitness = _wrap(H.fitness)
    RH.decode = decode
    RB.critical_path_bound = _wrap(B.critical_path_bound)
    RB.dep_subgraph = B.dep_subgraph
    RB.pre_subgraph = B.pre_subgraph

    def restore():
        for (mod, name), fn in saved.items():
            setattr(mod, name, fn)

    return restore
