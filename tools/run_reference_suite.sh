#!/bin/bash
# Drop-in conformance: the reference's own test suite (pkg/tests, staged
# unmodified into baseline/_ref/pkg_tests by `cp -r /root/reference/pkg/tests
# baseline/_ref/pkg_tests` in the build container; git-ignored, travels with
# gpurun) run against this repo's drop-in package pkg/src/caqr on the GPU.
# Writes the pass/fail list to $1 (default gpurun_out/reference_suite.txt).
REPO="$(cd "$(dirname "$0")/.." && pwd)"
OUT="$(realpath -m "${1:-$REPO/gpurun_out/reference_suite.txt}")"
mkdir -p "$(dirname "$OUT")"
cd "$REPO/baseline/_ref/pkg_tests" || { echo "stage the reference tests first" >&2; exit 2; }
PYTHONPATH="$REPO/pkg/src:$REPO/baseline/_ref/pkg_tests" timeout 1200 python -m pytest -c /dev/null \
  --rootdir . -p no:cacheprovider -q -rA . > "$OUT" 2>&1
rc=$?
tail -3 "$OUT"
exit $rc
