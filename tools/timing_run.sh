CC_TIMING=1 timeout -s KILL 300 python tools/e2e_profile.py c2 2>&1 | grep -E "cc timing|re-prepared" | head -60
