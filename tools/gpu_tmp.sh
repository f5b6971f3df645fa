timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for v in "" variants/s5.so; do for r in 2 3; do echo "== lib '$v' ratio $r"; CC_LIB=$v CC_DF_TR_RATIO=$r timeout -s KILL 120 python tools/df_profile.py 2>&1 | head -3; done; done
