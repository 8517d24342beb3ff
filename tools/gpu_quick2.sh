#!/bin/bash
# correctness subset + cfg4 timing (3 steps) for kernel iteration
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -q -x -k "cfg1_all_pairs or zeta or row_chunks or schedule or tables" > gpurun_out/q_tests.log 2>&1; echo "rc=$?" >> gpurun_out/q_tests.log
python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/q_b15.json 2> gpurun_out/q_b15.err
[ "${MASK3:-0}" = "1" ] && python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --mask 3 > gpurun_out/q_b3.json 2> gpurun_out/q_b3.err
exit 0
