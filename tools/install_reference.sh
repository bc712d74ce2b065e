#!/bin/bash
# Install the UNMODIFIED reference into baseline/_ref (git-ignored; it travels
# to the GPU box with the gpurun snapshot): the package via pip from a /tmp
# copy (/root/reference is read-only; offline dependency resolution fails, so
# --no-deps), plus its own tests and assets under baseline/_ref/ref_pkg so the
# reference's test suite can run against the B200 kernel seam
# (tests/test_gpu_seam.py). Nothing here is committed.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC=/root/reference/pkg
[ -d "$SRC" ] || { echo "no reference at $SRC" >&2; exit 1; }
TMP=$(mktemp -d)
cp -r "$SRC" "$TMP/pkg"
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target "$ROOT/baseline/_ref" "$TMP/pkg" >/dev/null
mkdir -p "$ROOT/baseline/_ref/ref_pkg"
cp -r "$SRC/tests" "$SRC/assets" "$ROOT/baseline/_ref/ref_pkg/"
chmod -R u+w "$ROOT/baseline/_ref"
rm -rf "$TMP"
echo "installed: $(ls "$ROOT/baseline/_ref")"
