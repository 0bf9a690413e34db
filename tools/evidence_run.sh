# Round-end evidence on one B200: full GPU suite, smoke, bench (driver's flags), the reference
# arm, the bench's ncu launch list, and one ncu --set full of the headline gather.
set -x
python -m pytest tests -m gpu -q --durations=15 > gpurun_out/ev_gputests.log 2>&1; tail -3 gpurun_out/ev_gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev_smoke.log 2>&1; tail -2 gpurun_out/ev_smoke.log
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/ev_bench.json 2> gpurun_out/ev_bench.err; tail -c 300 gpurun_out/ev_bench.json
python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/ev_ref.json 2> gpurun_out/ev_ref.err; tail -c 300 gpurun_out/ev_ref.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/ev_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ev_ncu_launch.log 2>&1
python tools/profile_r2.py --ops gather_c2,gather_c2_rand > /dev/null 2>&1
ncu --set full --import-source on --clock-control none --profile-from-start off -o /tmp/ev_gather python tools/profile_r2.py --ops gather_c2,gather_c2_rand > gpurun_out/ev_ncu_gather.log 2>&1
ncu -i /tmp/ev_gather.ncu-rep --page raw --csv > gpurun_out/ev_ncu_gather_raw.csv
ncu -i /tmp/ev_gather.ncu-rep --page details --csv > gpurun_out/ev_ncu_gather_details.csv
ls -la gpurun_out | tail -20
