#!/usr/bin/env bash
# Stage the UNMODIFIED reference package for the reference arm and for the
# overlay run of the reference's own test suite on the GPU box.
#   baseline/_ref/pdmrender   pip-installed from a /tmp copy of /root/reference/pkg
#   baseline/_ref/pkg_tests   the reference's tests/ directory, as shipped
# baseline/_ref is git-ignored (not product source, never committed) but not
# gpurun-ignored, so it travels to the GPU box where /root/reference does not exist.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
REF=/root/reference/pkg
[ -d "$REF" ] || { echo "no $REF here; nothing staged"; exit 0; }
TMP=$(mktemp -d)
cp -r "$REF" "$TMP/pkg"
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" "$TMP/pkg" >/dev/null
cp -r "$REF/tests" "$ROOT/baseline/_ref/pkg_tests"
cp "$REF/pyproject.toml" "$ROOT/baseline/_ref/pkg_pyproject.toml"
rm -rf "$TMP"
echo "staged: $(ls "$ROOT/baseline/_ref")"
