#!/usr/bin/env bash
# Build the REFERENCE's own CPU kernel (tilecast backend/_core.pyx, Cython -> C,
# OpenMP) from the sources where they lie under /root/reference, into
# oracle/_ref/ (git-ignored; it travels to the GPU box with the snapshot).
#
# This is test/baseline infrastructure only: tests use it to pin the oracle
# port, bench.py --impl reference times it. It is never on the product path.
#
# Recipe mirrors the reference's compile flags (pkg/setup.py:23-27:
# -O2 -ffp-contract=off -fopenmp) but does not run its setup.py. The
# reference is a Python package around one Cython module, so the package's
# .py files are copied next to the compiled module (the equivalent of the
# pip install the base contract describes) -- they stay out of git history.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REF="${TILECAST_REF_SRC:-/root/reference/pkg/src/tilecast}"
OUT="$HERE/_ref"
if [ ! -d "$REF" ]; then
  echo "build_ref: $REF not present; keeping prebuilt $OUT" >&2
  exit 0
fi
PY="${PYTHON:-python3}"
rm -rf "$OUT.tmp"
mkdir -p "$OUT.tmp"
cp -r "$REF" "$OUT.tmp/tilecast"
# the reference's own test suite, so tests/test_reference_suite.py can run it
# against the CUDA kernel through the drop-in backend (tests/ref_shim.py)
if [ -d "$REF/../../tests" ]; then
  cp -r "$REF/../../tests" "$OUT.tmp/tests"
  # the tests read maps from <pkg>/src/tilecast/maps
  mkdir -p "$OUT.tmp/src/tilecast" && cp -r "$REF/maps" "$OUT.tmp/src/tilecast/maps"
fi
chmod -R u+w "$OUT.tmp"
find "$OUT.tmp" -name '__pycache__' -prune -exec rm -rf {} +
"$PY" -m cython -3 "$OUT.tmp/tilecast/backend/_core.pyx" -o "$OUT.tmp/tilecast/backend/_core.c"
EXT="$("$PY" -c 'import sysconfig; print(sysconfig.get_config_var("EXT_SUFFIX"))')"
INC="$("$PY" -c 'import sysconfig; print(sysconfig.get_paths()["include"])')"
/usr/bin/gcc -O2 -ffp-contract=off -fopenmp -fPIC -shared -I"$INC" \
  "$OUT.tmp/tilecast/backend/_core.c" -o "$OUT.tmp/tilecast/backend/_core$EXT" -fopenmp
rm -f "$OUT.tmp/tilecast/backend/_core.c" "$OUT.tmp/tilecast/backend/_core.pyx"
[ -d "$OUT" ] && chmod -R u+w "$OUT"
rm -rf "$OUT"
mv "$OUT.tmp" "$OUT"
echo "build_ref: built $OUT/tilecast/backend/_core$EXT"
