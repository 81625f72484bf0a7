cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out/ncu
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python tools/kbench.py --only cg --T 131072 --precision fp64 2>&1 | tail -1
timeout 300 python tools/kbench.py --only cg --T 131072 --precision fp32 2>&1 | tail -1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fpm_cgw_kernel -c 1 -o gpurun_out/ncu/cgw64 \
  python tools/kbench.py --only cg --T 32768 --precision fp64 --reps 1 > gpurun_out/ncu/cgw64.log 2>&1; echo "ncu $?"
