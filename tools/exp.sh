python tools/gather_sweep.py --z 1.0,1.5 --gran 0 --policies 129,641 2>&1 | grep -v device_info | cut -c1-100
C="python tools/profile_kernels.py --ops gather_freq --policy 641"; $C > gpurun_out/p641.log 2>&1 && ncu --set full --clock-control none --profile-from-start off -o gpurun_out/prof_641 $C > gpurun_out/prof_641.log 2>&1; echo rc=$?
