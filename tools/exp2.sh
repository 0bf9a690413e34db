C="python tools/select_sweep.py --rows 536870912 --steps 1"
$C > gpurun_out/psel.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"k_select|k_category" --csv --log-file gpurun_out/sel_launch3.csv $C > gpurun_out/sel_ncu3.log 2>&1; echo rc=$?
