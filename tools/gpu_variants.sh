#!/bin/bash
# time cfg4 with each library variant under variants/ (and the product library)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/v_base.json 2> gpurun_out/v_base.err
for f in variants/librrq_*.so; do
  n=$(basename $f .so)
  RRQ_LIBRARY=$PWD/$f python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/v_$n.json 2> gpurun_out/v_$n.err
done
exit 0
