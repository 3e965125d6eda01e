#!/usr/bin/env bash
# TEST INFRASTRUCTURE ONLY: compile the unmodified reference package
# (/root/reference/pkg: pure Python + one Cython kernel, setup.py:5-19)
# into oracle/_ref/ so the CPU baseline and the oracle cross-checks can run
# the reference itself.  The build writes into its source tree, so it runs
# from a scratch copy under /tmp; the output lands only in oracle/_ref/
# (git-ignored; it travels to the GPU box with the snapshot).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC="${REFERENCE_PKG:-/root/reference/pkg}"
if [ ! -d "$SRC" ]; then
  echo "build_ref: $SRC not present; keeping existing oracle/_ref" >&2
  exit 0
fi
TMP="$(mktemp -d /tmp/rf_refbuild.XXXXXX)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"
rm -rf "$HERE/_ref"
python -m pip install --no-index --no-build-isolation --no-deps \
  --find-links /opt/wheelhouse --target "$HERE/_ref" "$TMP/pkg" >/dev/null
# the compiled backend must be present: REFUSION_BACKEND=compiled raises otherwise
ls "$HERE"/_ref/refusion/_kernels_cy*.so >/dev/null
echo "build_ref: reference installed into $HERE/_ref"
