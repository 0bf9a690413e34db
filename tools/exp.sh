C="python tools/select_sweep.py --rows 536870912 --steps 1"
$C > gpurun_out/psel.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,smsp__inst_executed.sum --clock-control none -k regex:"k_select|k_scan" --csv --log-file gpurun_out/sel_launch.csv $C > gpurun_out/sel_ncu.log 2>&1; echo rc=$?
