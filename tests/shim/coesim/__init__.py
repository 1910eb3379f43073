"""``coesim`` import-name shim over this package (parity harness only).

Importing ``coesim`` (the reference package's name) yields this repository's
implementation: the hot-path modules (types, routing, costmodel, profiler,
scheduler, expert_pool, baselines, engine, seeding) are aliased to
``paper_2503_02354_b200.*``; ``coesim.workload`` and ``coesim.cli`` (out of
scope: input producer and CLI) resolve to the reference sources under
``COESIM_REF_SRC`` and bind to our modules through their relative imports.
This lets the reference's own test files -- including the ones that spawn
``python -m coesim.cli`` -- run unmodified against this implementation.
Only used in the build container, where ``/root/reference`` exists.
"""

import importlib as _importlib
import os as _os
import sys as _sys

_REF_SRC = _os.environ.get("COESIM_REF_SRC", "/root/reference/pkg/src/coesim")
__path__ = [_REF_SRC]  # submodules we do not alias come from the reference sources

_OURS = ("types", "seeding", "routing", "costmodel", "profiler", "scheduler", "expert_pool", "baselines",
         "engine")
_pkg = _importlib.import_module("paper_2503_02354_b200")
for _name in _OURS:
    _mod = _importlib.import_module(f"paper_2503_02354_b200.{_name}")
    _sys.modules[f"{__name__}.{_name}"] = _mod
    globals()[_name] = _mod
for _name in _pkg.__all__:
    globals()[_name] = getattr(_pkg, _name)

from . import workload  # noqa: E402  (reference input producer, bound to our types/routing)

generate_registry = workload.generate_registry
generate_stream = workload.generate_stream
task_workload = workload.task_workload
