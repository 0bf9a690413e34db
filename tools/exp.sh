python bench.py > gpurun_out/bench_r1b.log 2>&1; echo rc=$?; tail -c 2500 gpurun_out/bench_r1b.log
