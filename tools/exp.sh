python tools/gather_sweep.py --z 1.0,1.5 --gran 0 --policies 129 > gpurun_out/gs.log 2>&1
python tools/gather_sweep.py --z 1.0 --gran 0 --policies 129 --width 4 --domain 4194304 --rows 16777216 --steps 50 >> gpurun_out/gs.log 2>&1
cut -c1-100 gpurun_out/gs.log
