#!/bin/bash
# One GPU call: parity tests, smoke, bench, launch list, ncu full of the top kernels.
set -x
mkdir -p gpurun_out
timeout -s KILL 400 python -m pytest tests -m gpu -q 2>&1 | tail -15
timeout -s KILL 120 python __graft_entry__.py smoke 2>&1 | tail -3
timeout -s KILL 600 python bench.py 2>&1 | tail -3 | tee gpurun_out/bench.json
timeout -s KILL 300 python tools/kbench.py --quick 2>&1 | tail -5
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/launches_bench.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:df_worker -s 1 -c 1 -o gpurun_out/prof_df -f python tools/prof_df.py > gpurun_out/prof_df.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:zgemm -s 2 -c 1 -o gpurun_out/prof_zgemm -f python tools/prof_kernels.py > gpurun_out/prof_zgemm.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:trace_kernel -s 2 -c 1 -o gpurun_out/prof_trace -f python tools/prof_kernels.py > gpurun_out/prof_trace.log 2>&1
ls -la gpurun_out
