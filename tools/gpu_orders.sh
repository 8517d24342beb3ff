#!/bin/bash
# the other orders: parity tests touching p = 4, 6, 10, 12, 14 and their bench lines (kernel iteration)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_highorder.py -q -x -k "cfg1_all_pairs or full_size or cfg5 or high_order" > gpurun_out/o_tests.log 2>&1; echo "rc=$?" >> gpurun_out/o_tests.log
for c in 3 5; do python bench.py --config $c --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/o_cfg$c.json 2> gpurun_out/o_cfg$c.err; done
python bench.py --config 6 --p 12 --steps 2 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/o_cfg6_p12.json 2> gpurun_out/o_cfg6_p12.err
[ -n "$P14" ] && python bench.py --config 6 --p 14 --chunk-pairs 3000000 --steps 2 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/o_cfg6_p14.json 2> gpurun_out/o_cfg6_p14.err
exit 0
