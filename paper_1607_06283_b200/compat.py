"""Reroute an imported reference evrecon through the B200 path.

evrecon.pipeline binds primal_dual_solve and the surface functions at
import (pipeline.py:22-29), and run_stream looks up init_state /
process_packet in the pipeline module's globals (pipeline.py:228-229,
:240).  Patching those two names there reroutes run_stream, `evrecon
reconstruct` (cli.py:147-152) and `evrecon bench` (cli.py:273-274) onto
the device state machine; patching evrecon.solve.primal_dual_solve alone
would have no effect.
"""

from __future__ import annotations

import sys

_SAVED = {}


def _patch(mod, name, repl):
    _SAVED.setdefault((id(mod), name), (mod, getattr(mod, name)))
    setattr(mod, name, repl)


def install(evrecon_pipeline=None, evrecon_cli=None):
    """Patch evrecon.pipeline.{init_state, process_packet, run_stream} (and
    the module's primal_dual_solve binding) with this package's versions,
    and evrecon.cli's import-time run_stream binding (cli.py:18) when the
    CLI module is loaded, so `evrecon reconstruct` / `evrecon bench` stream
    through the pipelined run_stream (packet k+1 computes while frame k is
    read back).  The reference config dataclasses and Event objects are
    duck-type compatible (same fields)."""
    from . import pipeline as ours
    from . import solve as ours_solve

    mod = evrecon_pipeline or sys.modules.get("evrecon.pipeline")
    if mod is None:
        import evrecon.pipeline as mod  # noqa: F811
    for name, repl in (("init_state", ours.init_state), ("process_packet", ours.process_packet),
                       ("primal_dual_solve", ours_solve.primal_dual_solve),
                       ("run_stream", ours.run_stream)):
        if hasattr(mod, name):
            _patch(mod, name, repl)
    cli = evrecon_cli or sys.modules.get("evrecon.cli")
    if cli is not None and hasattr(cli, "run_stream"):
        _patch(cli, "run_stream", ours.run_stream)
    return mod


def uninstall():
    for (_, name), (mod, orig) in list(_SAVED.items()):
        setattr(mod, name, orig)
    _SAVED.clear()
