#!/bin/bash
# quick GPU check: parity tests + small bench; prints stage times
python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log; grep -E "^E " gpurun_out/gpu_tests.log | head -5
python bench.py --freq 10 --n-off 20000 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/b_small.json 2>gpurun_out/b_small.err; tail -1 gpurun_out/b_small.err
