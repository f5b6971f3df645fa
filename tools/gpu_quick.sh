#!/bin/bash
# Quick GPU iteration: parity tests, kernel bench, bench line.
mkdir -p gpurun_out
timeout -s KILL 400 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout -s KILL 300 python tools/kbench.py 2>&1 | tail -12
timeout -s KILL 600 python bench.py --no-cpu-baseline 2>&1 | tail -2 | tee gpurun_out/bench_quick.json
