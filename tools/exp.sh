set -x
python bench.py > gpurun_out/bench_r1.log 2>&1; echo bench_rc=$?
tail -c 4000 gpurun_out/bench_r1.log
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_r1.log 2>&1; echo ref_rc=$?
tail -c 1500 gpurun_out/bench_ref_r1.log
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-extras"
$B > gpurun_out/plain_r1.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv $B > gpurun_out/ncu_launch_r1.log 2>&1; echo ncu1=$?
C="python tools/profile_kernels.py --policy 1"
$C > gpurun_out/prof_plain_r1.log 2>&1 && ncu --set full --clock-control none --import-source on --profile-from-start off -o gpurun_out/prof_full_r1 $C > gpurun_out/prof_full_r1.log 2>&1; echo ncu2=$?
