#!/bin/bash
# one ncu --set full capture of kernel $1 in the cfg4 launch configuration, summarised on the box:
# gpurun_out/ncu_$2_$1.txt (tools/ncu_hot.py) and gpurun_out/ncu_$2_$1_regions.txt (tools/ncu_regions.py)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
K=$1; TAG=${2:-x}
timeout 900 ncu --set full --import-source on --clock-control none -k regex:$K --launch-skip 12 --launch-count 1 \
  -o /tmp/ncu_${TAG}_$K -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_${TAG}_$K.log 2>&1
python tools/ncu_hot.py /tmp/ncu_${TAG}_$K.ncu-rep 30 > gpurun_out/ncu_${TAG}_$K.txt 2>&1
python tools/ncu_regions.py /tmp/ncu_${TAG}_$K.ncu-rep ${3:-400} > gpurun_out/ncu_${TAG}_${K}_regions.txt 2>&1
exit 0
