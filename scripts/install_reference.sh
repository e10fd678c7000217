#!/usr/bin/env bash
# Install the UNMODIFIED reference (graphtables + graphdesk) into baseline/_ref
# (git-ignored, travels to the GPU box with gpurun) with the task's offline
# pip recipe, plus a copy of its own tests for tests/test_reference_suite_gpu.py.
# The build writes into its source tree, so it installs from a copy under /tmp.
set -euo pipefail
REPO=$(cd "$(dirname "$0")/.." && pwd)
SRC=${1:-/root/reference}
TMP=$(mktemp -d /tmp/gtref.XXXXXX)
cp -r "$SRC/pkg" "$TMP/pkg"
rm -rf "$REPO/baseline/_ref"
mkdir -p "$REPO/baseline/_ref"
python -m pip install -q --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$REPO/baseline/_ref" "$TMP/pkg"
if [ -d "$TMP/pkg/frontend" ]; then
  python -m pip install -q --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
      --target "$REPO/baseline/_ref" "$TMP/pkg/frontend"
fi
cp -r "$TMP/pkg/tests" "$REPO/baseline/_ref/graphtables_tests"
rm -rf "$TMP"
ls "$REPO/baseline/_ref"
