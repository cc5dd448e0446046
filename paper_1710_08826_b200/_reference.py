"""Locate the reference package (parafit) this engine plugs into.

The device engine is a plug-in for the reference's own API: models are the
reference's ``PdfNode`` trees, parameters its ``Variable``s, datasets its
``UnbinnedDataSet``/``BinnedDataSet``, fits its ``FitManager``.  The engine
only replaces what runs *under* that API (the ``Backend`` protocol,
``register_cached_norm`` hooks, engine.py:32-135).

Resolution order for ``import parafit``:

1. an importable ``parafit`` (pip-installed, or already on ``sys.path``);
2. ``$PARAFIT_PATH`` (a directory containing the ``parafit`` package);
3. ``<repo>/baseline/_ref`` -- the unmodified reference installed by
   ``scripts/install_reference.sh`` (git-ignored; it travels with the repo
   snapshot to the GPU box, where ``/root/reference`` does not exist).
"""

from __future__ import annotations

import importlib
import os
import sys

_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASELINE_REF = os.path.join(_ROOT, "baseline", "_ref")


class ReferenceMissing(ImportError):
    """The reference package (parafit) is not importable."""


def _load():
    try:
        return importlib.import_module("parafit")
    except ImportError:
        pass
    for cand in (os.environ.get("PARAFIT_PATH"), BASELINE_REF):
        if cand and os.path.isdir(os.path.join(cand, "parafit")):
            if cand not in sys.path:
                sys.path.append(cand)
            return importlib.import_module("parafit")
    raise ReferenceMissing(
        "the reference package 'parafit' is not importable: install it (pip install <reference>/pkg), "
        f"set PARAFIT_PATH, or run scripts/install_reference.sh to populate {BASELINE_REF}")


parafit = _load()

from parafit import core, dalitz, engine, errors, fitting, mcgen, pdf, reduction, sharding  # noqa: E402

__all__ = ["parafit", "core", "dalitz", "engine", "errors", "fitting", "mcgen", "pdf", "reduction", "sharding",
           "ReferenceMissing", "BASELINE_REF"]
