#!/bin/bash
# ncu counters for l2_probe configurations (2nd launch of each).
M=dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,lts__t_requests_srcunit_tex_op_read.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_hit.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_write.sum
ncu --metrics $M --clock-control none -k regex:"k_l2|k_async" --csv --log-file gpurun_out/ncu_l2.csv python tools/probe/l2_one.py "$@" > gpurun_out/ncu_l2.log 2>&1
