timeout -s KILL 60 python tools/t_e2e_debug.py 128 8
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
timeout -s KILL 200 python tools/e2e_profile.py 2>&1 | head -9
CC_EARLY_COPIES=0 timeout -s KILL 200 python tools/e2e_profile.py 2>&1 | head -9 | grep re-prep
