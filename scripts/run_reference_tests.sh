#!/usr/bin/env bash
# Stage the reference's unit tests next to the contactamg alias conftest in
# baseline/_ref/ref_tests (git-ignored; travels to the GPU box), or run them.
#   scripts/run_reference_tests.sh stage   # in the build container (/root/reference present)
#   scripts/run_reference_tests.sh run     # on the GPU box
set -e
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
DST="$ROOT/baseline/_ref/ref_tests"
case "${1:-run}" in
  stage)
    rm -rf "$DST"; mkdir -p "$DST"
    cp /root/reference/pkg/tests/test_*.py "$DST/"
    cp "$ROOT/scripts/reference_tests/conftest.py" "$DST/"
    ls "$DST" ;;
  run)
    cp "$ROOT/scripts/reference_tests/conftest.py" "$DST/"
    cd "$DST" && PYTHONDONTWRITEBYTECODE=1 python -m pytest -p no:cacheprovider -q -rfE --rootdir "$DST" . ;;
esac
