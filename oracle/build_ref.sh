#!/usr/bin/env bash
# Test infrastructure only (the checker, never the product path).
# Builds the UNMODIFIED reference fmmkit (Python + its Cython kernel core
# pkg/src/fmmkit/_ckernels.pyx) into oracle/_ref/ so the reference's own CPU
# path can run beside the GPU build (bench.py --impl reference, parity tests).
#
# Recipe (no reference build system is run): copy the package sources into the
# git-ignored oracle/_ref/, cythonize _ckernels.pyx and compile it with gcc
# -O3 -fopenmp exactly as pkg/setup.py:16-31 asks. oracle/_ref/ travels to the
# GPU box with gpurun (it is git-ignored, not gpurun-ignored).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REF="${FMMB_REFERENCE:-/root/reference}"
OUT="$HERE/_ref"
if [ ! -d "$REF/pkg/src/fmmkit" ]; then
  echo "reference not present at $REF; keeping prebuilt $OUT" >&2
  exit 0
fi
mkdir -p "$OUT"
rm -rf "$OUT/fmmkit" "$OUT/tests"
cp -r "$REF/pkg/src/fmmkit" "$OUT/fmmkit"
cp -r "$REF/pkg/tests" "$OUT/tests"
chmod -R u+w "$OUT"
PY="${PYTHON:-python}"
cd "$OUT"
"$PY" -m cython -3 fmmkit/_ckernels.pyx -o fmmkit/_ckernels.c
INC_NP="$("$PY" -c 'import numpy; print(numpy.get_include())')"
INC_PY="$("$PY" -c 'import sysconfig; print(sysconfig.get_paths()["include"])')"
SUF="$("$PY" -c 'import sysconfig; print(sysconfig.get_config_var("EXT_SUFFIX"))')"
/usr/bin/gcc -O3 -fopenmp -fPIC -shared -DNPY_NO_DEPRECATED_API=NPY_1_7_API_VERSION \
  -I"$INC_NP" -I"$INC_PY" fmmkit/_ckernels.c -o "fmmkit/_ckernels$SUF"
"$PY" -c "import sys; sys.path.insert(0, '$OUT'); import fmmkit; assert fmmkit.backend_name() == 'compiled', fmmkit.backend_name(); print('oracle/_ref: fmmkit', fmmkit.backend_name())"
