#!/usr/bin/env bash
# Install the UNMODIFIED reference package gsgp 0.1.0 into baseline/_ref
# (git-ignored; it travels to the GPU box with the repo snapshot):
#   * the package itself (pip --target, offline, --no-deps: numpy is in the
#     image) — bench.py's CPU reference arm imports it (oracle/ref_bench.py);
#   * its own test suite under baseline/_ref/ref_tests — the reference-side
#     binding test (tests/test_gpu_reference_binding.py) applies
#     integration/gsgp_cuda.patch to a temp copy and runs these tests with
#     backend "cuda".
# Run in the build container, where /root/reference exists.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC=/root/reference/pkg
TMP="$(mktemp -d)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"                      # the build writes into the source tree
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target "$ROOT/baseline/_ref" "$TMP/pkg" >/dev/null
cp -r "$SRC/tests" "$ROOT/baseline/_ref/ref_tests"
echo "reference installed: $(ls "$ROOT/baseline/_ref")"
