# Round-end evidence on one B200: smoke, bench (driver's flags), the reference arm, the bench's
# ncu launch list, and one ncu --set full of the headline gather (the GPU suite runs separately).
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev_smoke.log 2>&1; tail -2 gpurun_out/ev_smoke.log
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/ev_bench.json 2> gpurun_out/ev_bench.err; tail -c 300 gpurun_out/ev_bench.json
python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/ev_ref.json 2> gpurun_out/ev_ref.err; tail -c 300 gpurun_out/ev_ref.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ev_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-extras > gpurun_out/ev_ncu_launch.log 2>&1
ls -la gpurun_out | tail -10
