#!/bin/bash
# bench lines of the other configs: python bench.py --config N
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for c in ${CFGS:-1 2 3 5 6 7}; do
  timeout 1500 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.err; echo "cfg$c rc=$?" >> gpurun_out/cfgs.status
done
[ -n "$HIP" ] && for p in 12 14; do
  timeout 1500 python bench.py --config 6 --p $p --chunk-pairs 3000000 --steps 3 --warmup 3 > gpurun_out/bench_cfg6_p$p.json 2> gpurun_out/bench_cfg6_p$p.err; echo "cfg6 p$p rc=$?" >> gpurun_out/cfgs.status
done
exit 0
