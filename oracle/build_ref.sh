#!/usr/bin/env bash
# Test infrastructure only: build the UNMODIFIED reference package
# (/root/reference/pkg, Cython core + Python modules) into oracle/_ref/ so the
# parity tests can pin the oracle against it and bench.py's reference arm can
# time it.  Never run on the GPU box (no /root/reference there): the built
# oracle/_ref/ travels with the gpurun snapshot instead.
#
# The reference tree is read-only, so the build runs from a scratch copy under
# /tmp; outputs land only in oracle/_ref/ (git-ignored, not gpurun-ignored).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC="${EXPSTENCIL_REF_SRC:-/root/reference/pkg}"
OUT="$HERE/_ref"
if [ ! -d "$SRC" ]; then
  echo "build_ref: reference source $SRC not present; keeping existing $OUT" >&2
  exit 0
fi
SCRATCH="$(mktemp -d /tmp/expstencil_ref.XXXXXX)"
trap 'rm -rf "$SCRATCH"' EXIT
cp -r "$SRC" "$SCRATCH/pkg"
rm -rf "$OUT"
python -m pip install --quiet --no-index --no-build-isolation --no-deps \
  --target "$OUT" "$SCRATCH/pkg" >"$SCRATCH/pip.log" 2>&1 || {
  cat "$SCRATCH/pip.log" >&2; exit 1; }
# the compiled core must be present: the reference arm times the Cython path
ls "$OUT"/expstencil/_core*.so >/dev/null
echo "build_ref: reference installed into $OUT"
