"""pytest plugin: run the reference's own test suite (loopsmith tests/) with
the B200 backend installed in place of the VM backend.

    PYTHONPATH=<loopsmith install>:<repo>:<repo>/tools \
        python -m pytest <loopsmith tests> -p refsuite_plugin

The reference test modules bind ``from loopsmith.backend import ...`` at
import (SURVEY §8(b) binding hazard), so ``install()`` runs when the plugin
loads, before collection.  Test infrastructure only: nothing in the product
or in tests/ imports this.
"""
import loopsmith  # noqa: F401  (the reference, from PYTHONPATH)

from paper_2205_00618_b200 import install as _install, native as _native

try:
    _native.init(0)
    _DEV = "cuda:0"
except _native.NativeError as e:   # CPU container: compile-only tests still run
    _DEV = f"none ({e})"
BOUND = _install()


def pytest_report_header(config):
    return [f"B200 backend installed over: {', '.join(BOUND)}", f"device: {_DEV}"]
