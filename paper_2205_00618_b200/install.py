"""Install the B200 backend under an already-imported loopsmith.

The reference binds backend names at import time (SURVEY §8(b) binding
hazard): ``from .backend import ...`` in loopsmith/__init__.py:22-23,
session.py:33, tuner.py:20 and cli.py:26; only feedback.benchmark imports
``execute`` lazily (feedback.py:274), which resolves through the
``loopsmith.backend`` module attribute.  ``install()`` rebinds every one of
those names; ``uninstall()`` restores the originals.
"""

from __future__ import annotations

import importlib
import sys

from . import backend as _b200

_NAMES = ("compile", "compile_tree", "compile_single_operand", "execute",
          "CompiledKernel")
_MODULES = ("loopsmith", "loopsmith.backend", "loopsmith.session", "loopsmith.tuner",
            "loopsmith.cli")
_saved: dict[tuple[str, str], object] = {}


def install() -> list[str]:
    """Rebind loopsmith's backend entry points to the B200 backend.
    Returns the list of ``module.name`` bindings replaced."""
    done = []
    for mod_name in _MODULES:
        try:
            mod = sys.modules.get(mod_name) or importlib.import_module(mod_name)
        except Exception:
            continue
        for name in _NAMES:
            if hasattr(mod, name):
                key = (mod_name, name)
                if key not in _saved:
                    _saved[key] = getattr(mod, name)
                setattr(mod, name, getattr(_b200, name))
                done.append(f"{mod_name}.{name}")
    return done


def uninstall() -> None:
    for (mod_name, name), obj in _saved.items():
        mod = sys.modules.get(mod_name)
        if mod is not None:
            setattr(mod, name, obj)
    _saved.clear()
