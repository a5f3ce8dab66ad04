"""Route an installed ``stratba`` package onto the B200 path.

The reference's callers of the hot path -- ``pipeline.run_problem``
(pipeline.py:191,209), the CLI and user code -- call ``lm_minimize``
(solvers.py:318-393).  ``enable(stratba)`` rebinds that name in the reference's
``solvers`` and ``pipeline`` modules (the pipeline imported it by name,
pipeline.py:18) to a dispatcher that runs the device ``lm_minimize`` for the
inner solvers the GPU path implements ("power", "pcg") and the reference's own
function otherwise ("direct").  Optionally ``random_init`` (bal_io.py:281-297,
imported by name at pipeline.py:13) is rebound too.  ``disable`` restores the
originals.  Nothing here imports ``stratba``: the caller passes the module.
"""

from __future__ import annotations

from . import solver

_SAVED: dict = {}


def enable(stratba, *, random_init: bool = False) -> None:
    """Switch ``stratba``'s lm_minimize (and optionally random_init) to the device path."""
    if _SAVED:
        disable()
    ref_lm = stratba.solvers.lm_minimize

    def lm_minimize(problem, state, stage, config, trace_sink=None, *, solver_id=None,
                    problem_id=""):
        if config.inner_solver in ("power", "pcg"):
            return solver.lm_minimize(problem, state, stage, config, trace_sink,
                                      solver_id=solver_id, problem_id=problem_id)
        return ref_lm(problem, state, stage, config, trace_sink, solver_id=solver_id,
                      problem_id=problem_id)

    lm_minimize.__doc__ = ref_lm.__doc__
    targets = [(stratba.solvers, "lm_minimize", lm_minimize),
               (stratba.pipeline, "lm_minimize", lm_minimize)]
    if random_init:
        targets += [(stratba.bal_io, "random_init", solver.random_init),
                    (stratba.pipeline, "random_init", solver.random_init)]
    for mod, name, fn in targets:
        _SAVED[(mod, name)] = getattr(mod, name)
        setattr(mod, name, fn)


def disable() -> None:
    """Restore the reference functions rebound by :func:`enable`."""
    for (mod, name), fn in _SAVED.items():
        setattr(mod, name, fn)
    _SAVED.clear()
