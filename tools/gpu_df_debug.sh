#!/bin/bash
# dataflow smoke with short timeouts
timeout -s KILL 60 python -m pytest tests/test_gpu_parity.py -x -q -k "c1_all_ones" 2>&1 | tail -5
timeout -s KILL 120 python -m pytest tests/test_gpu_parity.py -x -q -k "c1 or c2_small or invariance or c3 or c4 or partitions" 2>&1 | tail -8
