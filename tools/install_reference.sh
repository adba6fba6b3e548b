#!/usr/bin/env bash
# Installs the UNMODIFIED reference package into baseline/_ref (git-ignored,
# travels to the GPU box with gpurun) -- the one offline install the task
# allows -- plus the reference's own test files next to it, so that
# tests/test_gpu_reference_suite.py can run them against the B200 path
# through paper_2604_19004_b200.refbind.  Build container only (needs
# /root/reference); nothing here is committed.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC=/root/reference/pkg
[ -d "$SRC" ] || { echo "no $SRC: nothing to install"; exit 0; }
TMP="$(mktemp -d)"
cp -r "$SRC" "$TMP/pkg"            # the build writes into its source tree
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" "$TMP/pkg" >/dev/null
mkdir -p "$ROOT/baseline/_ref/reference_tests"
cp "$SRC"/tests/*.py "$ROOT/baseline/_ref/reference_tests/"
rm -rf "$TMP"
echo "installed sketchgemm into $ROOT/baseline/_ref (tests in reference_tests/)"
