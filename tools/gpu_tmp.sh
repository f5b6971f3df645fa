timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
timeout -s KILL 120 python tools/df_profile.py 2>&1 | head -3
CC_LIB=variants/nopft.so timeout -s KILL 120 python tools/df_profile.py 2>&1 | head -3
