#!/bin/bash
# ncu --set full captures of one launch of each build kernel in the bench's own cfg4 launch configuration,
# summarised on the box (tools/ncu_hot.py: key metrics, stall reasons, hottest SASS lines); the reports stay in /tmp
# (gpurun_out/ is capped at 64 MiB).  usage (on the GPU box): bash tools/ncu_cfg4.sh TAG [kernels...]
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-v}
shift
KS=${@:-k_newton k_edge_lines k_target_gamma k_qmap k_translate k_contract}
for K in $KS; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$K --launch-skip 12 --launch-count 1 \
    -o /tmp/ncu_${TAG}_$K -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline \
    > gpurun_out/ncu_${TAG}_$K.log 2>&1
  echo "$K rc=$?" >> gpurun_out/ncu_${TAG}.status
  { echo "# ncu --set full --import-source on --clock-control none -k regex:$K --launch-skip 12 --launch-count 1 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline";
    echo "# (cfg4 launch configuration, 13th launch of the kernel; summary by tools/ncu_hot.py)";
    python tools/ncu_hot.py /tmp/ncu_${TAG}_$K.ncu-rep 30; } > gpurun_out/ncu_${TAG}_$K.txt 2>&1
done
python tools/ncu_traffic.py $TAG > gpurun_out/traffic_$TAG.json 2> gpurun_out/traffic_$TAG.err
for K in $KS; do python tools/ncu_regions.py /tmp/ncu_${TAG}_$K.ncu-rep 800 > gpurun_out/ncu_${TAG}_${K}_regions.txt 2>&1; done
exit 0
