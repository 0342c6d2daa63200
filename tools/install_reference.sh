#!/bin/bash
# Installs the UNMODIFIED reference package (evrecon 0.1.0) into baseline/_ref
# (git-ignored; it travels to the GPU box with the gpurun snapshot) and puts
# the reference's own test suite beside it as baseline/_ref/evrecon_tests,
# for tests/test_reference_suite.py (the suite run through the drop-in) and
# bench.py's numpy-reference timing.  Needs /root/reference (this container).
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC=/root/reference/pkg
[ -d "$SRC" ] || { echo "no $SRC" >&2; exit 1; }
TMP="$(mktemp -d)"
cp -r "$SRC" "$TMP/pkg"          # the build writes into its source tree
python -m pip install --upgrade --no-index --no-build-isolation --no-deps \
    --find-links /opt/wheelhouse --target "$ROOT/baseline/_ref" "$TMP/pkg" >/dev/null
rm -rf "$ROOT/baseline/_ref/evrecon_tests"
cp -r "$SRC/tests" "$ROOT/baseline/_ref/evrecon_tests"
rm -rf "$TMP"
echo "reference installed in $ROOT/baseline/_ref (tests: evrecon_tests)"
