timeout 200 python -m pytest tests/test_gpu_parity.py -q -x -k "select or kat or golden" 2>&1 | tail -2
timeout 200 python tools/select_sweep.py 2>&1 | tail -1
