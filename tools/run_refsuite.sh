#!/bin/bash
# Run the reference's own test suite (loopsmith tests/) against the B200
# backend: install the reference package into baseline/_ref (git-ignored; it
# travels to the GPU box with the gpurun snapshot), copy its tests next to
# it, and run them with tools/refsuite_plugin.py, which rebinds loopsmith's
# backend names to paper_2205_00618_b200 before collection.
#   here (dev container, reference mounted):  tools/run_refsuite.sh install
#   on the GPU box:                           tools/run_refsuite.sh run > log
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
REF=$ROOT/baseline/_ref
if [ "$1" = "install" ]; then
    tmp=$(mktemp -d)
    cp -r /root/reference/pkg "$tmp/pkg"
    python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
        --target "$REF" "$tmp/pkg" -q
    rm -rf "$REF/reftests" && cp -r "$tmp/pkg/tests" "$REF/reftests"
    rm -rf "$tmp"
    exit 0
fi
PYTHONPATH=$REF:$ROOT:$ROOT/tools python -m pytest -q "$REF/reftests" -p no:cacheprovider \
    -p refsuite_plugin -rf "${@:2}"
