#!/bin/bash
# Build development variants of the library with extra nvcc macros, e.g.
#   tools/build_variants.sh rs144:-DFPM_WS_GRAM_REGS=144 rs200:-DFPM_WS_GRAM_REGS=200
# -> tools/_variants/lib_<name>.so, loaded with FPM_LIB=<path>.
set -e
cd "$(dirname "$0")/.."
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  FPM_NVCC_EXTRA="$flags" FPM_BUILD_OBJ=tools/_variants/obj_$name FPM_BUILD_OUT=tools/_variants/lib_$name.so \
    python -m paper_2504_09820_b200.build --force &
done
wait
ls -la tools/_variants/*.so
