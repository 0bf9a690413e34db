python -m pytest tests -q -m gpu > gpurun_out/gpu_tests_r1.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/gpu_tests_r1.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r1.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/smoke_r1.log
python bench.py > gpurun_out/bench_r1c.log 2>&1; echo bench_rc=$?
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_r1c.log 2>&1; echo ref_rc=$?
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-extras"
$B > gpurun_out/plain_r1c.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1c.csv $B > gpurun_out/ncu_launch_r1c.log 2>&1; echo ncu1=$?
C="python tools/profile_kernels.py --policy 129"
$C > gpurun_out/prof_plain_r1c.log 2>&1 && ncu --set full --clock-control none --import-source on --profile-from-start off -o gpurun_out/prof_full_r1c $C > gpurun_out/prof_full_r1c.log 2>&1; echo ncu2=$?
