#!/bin/bash
# experiments: planner knob variants per config (product lib), serial-mode trace (diag lib)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out/c; O=gpurun_out/c
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
FPM_NVCC_EXTRA="-DFPM_DIAG" FPM_BUILD_OBJ=/tmp/fpm_obj_diag FPM_BUILD_OUT=paper_2504_09820_b200/libfpmimo_b200_diag.so \
  python -m paper_2504_09820_b200.build > $O/diag_build.log 2>&1
D=paper_2504_09820_b200/libfpmimo_b200_diag.so
cb() { tag=$1; cfg=$2; shift 2; echo "== $tag $cfg $*" >> $O/cfg.log; timeout 300 env "$@" python tools/cfgbench.py --only $cfg --T 32768 >> $O/cfg.log 2>&1; }
cb base c2_fp16 FPM_X=0
cb ncg2 c2_fp16 FPM_WS_NCG=2 FPM_WS_NSLOT=2
cb ncg1s2 c2_fp16 FPM_WS_NCG=1 FPM_WS_NSLOT=2
cb base c5_fp64 FPM_X=0
cb ct224 c5_fp64 FPM_WS_CT=224
cb base c1 FPM_X=0
cb r8 c1 FPM_R=8
cb nospl c5_fp64 FPM_WS_NOSPLIT=1
tr() { name=$1; shift; timeout 300 env FPM_LIB=$D "$@" python tools/kbench.py --only detect --wstrace --reps 3 $KB > $O/trace_$name.json 2> $O/trace_$name.err; echo "$name $?"; }
KB="--T 16384 --precision fp64" tr c5fp64_serial FPM_DEBUG=8
KB="--T 16384 --precision fp64" tr c5fp64_nogram FPM_DEBUG=4
KB="--T 16384 --precision fp64" tr c5fp64_nocg FPM_DEBUG=1
KB="--T 16384 --precision fp16" tr c5fp16_nogram FPM_DEBUG=4
KB="--T 16384 --precision fp16" tr c5fp16_nocg FPM_DEBUG=1
KB="--T 32768 --M 128 --N 32 --alg fp_cg --precision fp16 --iters 10" tr c2_nogram FPM_DEBUG=4
KB="--T 32768 --M 128 --N 32 --alg fp_cg --precision fp16 --iters 10" tr c2_ncg2 FPM_WS_NCG=2 FPM_WS_NSLOT=2
KB="--T 65536 --M 128 --N 16 --alg cg --precision fp64 --iters 8" tr c1_nocg FPM_DEBUG=1
cat $O/cfg.log | grep -v "^$" | cut -c1-300
