#!/bin/bash
# diag pass: phase timelines of the WS kernel on c5 fp64 / fp16, c1, c2; ncu of c1 / c5 fp64; sanitizer probe
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out/b
O=gpurun_out/b
FPM_NVCC_EXTRA="-DFPM_DIAG" FPM_BUILD_OBJ=/tmp/fpm_obj_diag FPM_BUILD_OUT=paper_2504_09820_b200/libfpmimo_b200_diag.so \
  python -m paper_2504_09820_b200.build > $O/diag_build.log 2>&1 || { echo diag build failed; tail $O/diag_build.log; }
D=paper_2504_09820_b200/libfpmimo_b200_diag.so
run() { name=$1; shift; timeout 300 env FPM_LIB=$D python tools/kbench.py --only detect --wstrace --reps 3 "$@" > $O/trace_$name.json 2> $O/trace_$name.err; echo "$name $?"; }
run c5fp64 --T 16384 --precision fp64
run c5fp16 --T 16384 --precision fp16
run c1 --T 65536 --M 128 --N 16 --alg cg --precision fp64 --iters 8
run c2 --T 32768 --M 128 --N 32 --alg fp_cg --precision fp16 --iters 10
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fpm_detect_ws_kernel -c 1 -o $O/c1 \
  python tools/kbench.py --only detect --reps 1 --T 65536 --M 128 --N 16 --alg cg --precision fp64 --iters 8 > $O/ncu_c1.log 2>&1; echo "ncu c1 $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fpm_detect_ws_kernel -c 1 -o $O/c5fp64 \
  python tools/kbench.py --only detect --reps 1 --T 16384 --precision fp64 > $O/ncu_c5fp64.log 2>&1; echo "ncu c5fp64 $?"
timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > $O/sanitizer_memcheck_smoke.log 2>&1; echo "memcheck $?"
tail -5 $O/sanitizer_memcheck_smoke.log
