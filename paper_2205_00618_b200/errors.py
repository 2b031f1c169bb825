"""Exceptions of the drop-in surface.

Callers of the reference catch ``loopsmith.backend.BlockTooLarge`` /
``HasReduction`` (backend.py:41-46; session.py:144-145 maps the first to
"block-too-large") and ``loopsmith.feedback.ShapeMismatch`` (feedback.py:21).
When loopsmith is importable the B200 backend raises *those* classes (or
subclasses), so existing ``except`` clauses keep working; otherwise it uses
stand-ins with the same names.
"""

from __future__ import annotations

try:  # pragma: no cover - depends on the environment
    from loopsmith.backend import BlockTooLarge as _RefBlockTooLarge
    from loopsmith.backend import HasReduction as _RefHasReduction
    from loopsmith.feedback import ShapeMismatch as _RefShapeMismatch
except Exception:  # loopsmith absent (e.g. on the GPU box)
    _RefBlockTooLarge = _RefHasReduction = _RefShapeMismatch = Exception


class BlockTooLarge(_RefBlockTooLarge):
    """The graph cannot be expressed by the B200 kernel set."""


class HasReduction(_RefHasReduction):
    pass


class ShapeMismatch(_RefShapeMismatch):
    pass
