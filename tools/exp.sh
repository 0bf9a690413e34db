for r in 8388608 16777216 33554432 67108864 134217728; do echo range=$r; SKX_HIST_RANGE=$r python tools/index_sweep.py 2>&1 | tail -1 | cut -c1-120; done
SKX_HIST_RANGE=134217728 python tools/index_sweep.py --domain 134217728 --z 1.0 2>&1 | tail -1 | cut -c1-120
