M=gpu__time_duration.sum,lts__t_sectors_op_red.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,smsp__thread_inst_executed_per_inst_executed.ratio
for v in orig hist0 sel0; do
  if [ $v = orig ]; then unset SKX_LIBSKX; else export SKX_LIBSKX=$PWD/tools/variants/libskx_$v.so; fi
  python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --configs c4,c5 > gpurun_out/ab1_$v.json 2>gpurun_out/ab1_$v.err
  python -c "import json;d=json.load(open('gpurun_out/ab1_$v.json'));print('$v', 'c4', d['index_build_c4']['ms_per_build'], d['index_build_c4']['phases_ms'], 'c5', d['select_c5']['ms_per_step'])"
  ncu --metrics $M --clock-control none --profile-from-start off --csv python tools/profile_r2.py --ops index_c4,select_c5 > gpurun_out/ab1_ncu_$v.csv 2>gpurun_out/ab1_ncu_$v.err
done
