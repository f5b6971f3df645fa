timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for i in 1 2; do timeout -s KILL 120 python tools/df_profile.py 2>&1 | head -4; done
