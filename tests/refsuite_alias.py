"""pytest plugin (-p refsuite_alias): run the reference's own test suite
(baseline/_ref/evrecon_tests, copied there by tools/install_reference.sh)
against this package by aliasing `evrecon` and its submodules to it
("Reuse" step 1).  evrecon.cli is the reference's unmodified
CLI module executed on top of the aliased modules, so `evrecon reconstruct`
/ `bench` run the B200 path through their own import-time bindings.

Loaded only by tests/test_reference_suite.py, in a subprocess: the alias
never reaches this repo's own test session.
"""

from __future__ import annotations

import importlib.util
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


def _alias():
    if ROOT not in sys.path:
        sys.path.insert(0, ROOT)
    import paper_1607_06283_b200 as ours
    from paper_1607_06283_b200 import events, pgm, pipeline, simulate, solve, surface

    sys.modules["evrecon"] = ours
    for name, mod in (("events", events), ("pgm", pgm), ("pipeline", pipeline),
                      ("simulate", simulate), ("solve", solve), ("surface", surface)):
        sys.modules["evrecon." + name] = mod
    spec = importlib.util.spec_from_file_location(
        "evrecon.cli", os.path.join(REF, "evrecon", "cli.py"),
        submodule_search_locations=None)
    cli = importlib.util.module_from_spec(spec)
    cli.__package__ = "evrecon"
    sys.modules["evrecon.cli"] = cli
    spec.loader.exec_module(cli)
    ours.cli = cli


_alias()


def pytest_sessionstart(session):
    """CUDA context creation and the lazy loading of the operator kernels
    happen once per process: done here, before the first test, so the
    reference's timing budgets (e.g. criterion 1's one second for 600
    operator calls, test_acceptance.py:50-75) time the operators rather than
    driver start-up -- the analogue of the reference paying numpy's import
    before its timers start."""
    import numpy as np

    import paper_1607_06283_b200 as ours

    t = np.linspace(0.0, 3.0, 64).reshape(8, 8)
    m = ours.compute_metric(t)
    u = np.full((8, 8), 1.5)
    p = np.zeros((8, 8, 3))
    ours.surface_gradient(u, m)
    ours.surface_gradient_adjoint(p, m)
    ours.prox_data(u, u, m, 0.1, ours.SolverConfig())
    ours.prox_dual(p, m)
    ours.energy(u, u, m, 0.7)
    ours.denoise_timestamps(ours.TimeSurface(t, 3.0), 1.0, 2)
    ours.primal_dual_solve(u, m, ours.SolverConfig(max_iterations=2))
    ours.rof_manifold_solve(u, m, 8.0, 2)
