#!/bin/bash
# Diagnostic library for tools/sanitize_cases.py --racecheck: phase traces,
# FPM_DEBUG skip / schedule-perturbation bits (-DFPM_DIAG), deadlock and
# shared-memory layout traps (-DFPM_CHECKED).  Never loaded by the product
# path (only through FPM_LIB).
set -e
cd "$(dirname "$0")/.."
FPM_NVCC_EXTRA="-DFPM_DIAG -DFPM_CHECKED" FPM_BUILD_OBJ=/tmp/fpm_obj_checked \
  FPM_BUILD_OUT=paper_2504_09820_b200/libfpmimo_b200_checked.so python -m paper_2504_09820_b200.build
# timing diagnostics only (phase traces, FPM_DEBUG skip bits; no checks): tools/kbench.py --wstrace
FPM_NVCC_EXTRA="-DFPM_DIAG" FPM_BUILD_OBJ=/tmp/fpm_obj_diag \
  FPM_BUILD_OUT=paper_2504_09820_b200/libfpmimo_b200_diag.so python -m paper_2504_09820_b200.build
