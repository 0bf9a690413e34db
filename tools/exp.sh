timeout 120 python -m pytest tests/test_gpu_parity.py -q -x -k "aggregate or golden or kat" 2>&1 | tail -2
timeout 120 python tools/groupby_sweep.py --z 1.0,1.5,0.5 --modes 0 2>&1 | grep count_sum | cut -c1-110
