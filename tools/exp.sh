python -m pytest tests/test_gpu_refsuite.py -q -x -s 2>&1 | tail -30
