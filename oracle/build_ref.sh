#!/usr/bin/env bash
# Compile the reference's own butterfly kernel (pkg/src/fftshield/kernels/_stockham.pyx)
# from where it lies under /root/reference into oracle/_ref/ (git-ignored; travels to the
# GPU box with the snapshot). Only the generated C and the .so land in oracle/_ref/.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC=/root/reference/pkg/src/fftshield/kernels/_stockham.pyx
if [ ! -f "$SRC" ]; then echo "reference absent; oracle/_ref not built"; exit 0; fi
OUT="$HERE/_ref"
mkdir -p "$OUT"
PY=${PYTHON:-python}
"$PY" -m cython -3 --module-name fftshield.kernels._stockham -o "$OUT/_stockham.c" "$SRC"
INC_PY=$("$PY" -c 'import sysconfig;print(sysconfig.get_paths()["include"])')
INC_NP=$("$PY" -c 'import numpy;print(numpy.get_include())')
SUFFIX=$("$PY" -c 'import sysconfig;print(sysconfig.get_config_var("EXT_SUFFIX"))')
${CC:-gcc} -O2 -fwrapv -fPIC -shared -DNPY_NO_DEPRECATED_API=NPY_1_7_API_VERSION \
    -I"$INC_PY" -I"$INC_NP" -o "$OUT/_stockham$SUFFIX" "$OUT/_stockham.c"
echo "built $OUT/_stockham$SUFFIX"
