python -m pytest tests/test_gpu_parity.py tests/test_gpu_refsuite.py -q -x 2>&1 | tail -3
python tools/index_sweep.py 2>&1 | tail -1
python tools/index_sweep.py --domain 134217728 --z 1.0 2>&1 | tail -1
