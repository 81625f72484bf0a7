python bench.py > gpurun_out/bench_full.log 2>&1; tail -c 3000 gpurun_out/bench_full.log; cp gpurun_out/clocks_rank0.csv gpurun_out/clocks_full.csv
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; tail -c 1500 gpurun_out/bench_ref.log
