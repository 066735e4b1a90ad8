#!/bin/bash
# Offline install of the stock reference package (hosfem, /root/reference/pkg)
# into baseline/_ref -- the reference arm's one sanctioned install -- plus its
# own test suite as baseline/_ref/hosfem_tests for the drop-in test
# (tests/test_reference_suite_gpu.py).  baseline/_ref is git-ignored and not
# gpurun-ignored, so it travels to the GPU box.  Needs /root/reference (this
# container only); the GPU box uses the installed copy.
set -e
cd "$(dirname "$0")/.."
SRC=/root/reference/pkg
[ -d "$SRC" ] || { echo "install_reference: $SRC not found" >&2; exit 1; }
TMP=$(mktemp -d)
cp -r "$SRC" "$TMP/hosfem_src"   # the build writes into its source tree; /root/reference is read-only
python -m pip install -q --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target baseline/_ref --upgrade "$TMP/hosfem_src"
rm -rf baseline/_ref/hosfem_tests
cp -r "$SRC/tests" baseline/_ref/hosfem_tests
rm -rf "$TMP"
echo "installed hosfem into baseline/_ref (+ hosfem_tests)"
