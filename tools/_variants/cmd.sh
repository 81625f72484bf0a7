timeout 300 python tools/kbench.py --only cg --T 65536 --reps 1 > /dev/null 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:fpm_cg_kernel -c 1 -o gpurun_out/prof_cg2 python tools/kbench.py --only cg --T 65536 --reps 1 > gpurun_out/ncu_cg2.log 2>&1; tail -1 gpurun_out/ncu_cg2.log
