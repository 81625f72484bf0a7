python bench.py --steps 5 --warmup 3 > gpurun_out/bench_full.log 2>&1; tail -c 2600 gpurun_out/bench_full.log
