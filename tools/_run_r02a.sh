#!/bin/bash
# round-2 evidence pass: tests, smoke, bench, reference arm, launch list, full ncu capture
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
nvidia-smi > gpurun_out/r02_nvsmi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02_build.log 2>&1 || { echo BUILD FAIL; tail gpurun_out/r02_build.log; exit 1; }
timeout 2400 python -m pytest tests -m gpu -x -q --durations=25 > gpurun_out/r02_pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02_pytest_gpu.log
tail -3 gpurun_out/r02_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1; echo "smoke exit $?"; tail -2 gpurun_out/r02_smoke.log
timeout 1500 python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo "bench exit $?"
cp gpurun_out/clocks_rank0.csv gpurun_out/r02_clocks.csv 2>/dev/null
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02_ref.json 2> gpurun_out/r02_ref.err; echo "ref exit $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches.csv \
  python bench.py --T 65536 --steps 2 --warmup 1 --no-cpu --no-e2e --no-configs > gpurun_out/r02_ncu_launch.log 2>&1; echo "ncu launches exit $?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:fpm_detect_ws_kernel -c 1 -o gpurun_out/r02_detect_ws \
  python bench.py --T 16384 --steps 1 --warmup 0 --no-cpu --no-e2e --no-configs > gpurun_out/r02_ncu_full.log 2>&1; echo "ncu full exit $?"
