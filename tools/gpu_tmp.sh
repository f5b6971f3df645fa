timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for v in variants/nopft.so variants/s6.so "" ""; do echo "== $v"; CC_LIB=$v timeout -s KILL 120 python tools/df_profile.py 2>&1 | head -1; done
