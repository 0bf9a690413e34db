python tools/gather_sweep.py --z 1.0 --gran 0 --policies 1,5,69 --tiers 0:160:0.25,0:160:0.5,0:160:0.75 2>&1 | grep -v device_info | cut -c1-110
