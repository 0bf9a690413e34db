python tools/gather_sweep.py --z 1.0,1.5 --gran 0 --policies 129,641,1153 2>&1 | grep -v device_info | cut -c1-100
python tools/gather_ceilings.py 129,1153 2>&1 | grep -E "L2_random|DRAM"
