cd "$GRAFT_REPO_ROOT"
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
FPM_NVCC_EXTRA="-DFPM_DIAG" FPM_BUILD_OBJ=/tmp/fpm_obj_diag FPM_BUILD_OUT=paper_2504_09820_b200/libfpmimo_b200_diag.so python -m paper_2504_09820_b200.build > /dev/null 2>&1
D=paper_2504_09820_b200/libfpmimo_b200_diag.so
for bits in 0 32 1 64; do FPM_LIB=$D FPM_DEBUG=$bits timeout 300 python tools/cfgbench.py --only $1 --T 32768 2>&1 | tail -1 | sed "s/^/dbg$bits /" | sed 's/"kernel.*fp64_frac"/ /'; done
