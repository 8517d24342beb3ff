#!/bin/bash
# round-end evidence: GPU tests, smoke, the cfg4 bench line (5 steps), its ncu launch list, p = 14 bench line
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x > gpurun_out/gputests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_launch.log
python tools/launch_summary.py /tmp/launches.csv "python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline (cfg4; 4 build steps: 1 warm-up + 2 timed + 1 serial with the overlap off)" > gpurun_out/launch_summary.txt 2>&1
python bench.py --config 6 --p 14 --chunk-pairs 3000000 --steps 3 --warmup 3 > gpurun_out/bench_cfg6_p14.json 2> gpurun_out/bench_cfg6_p14.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
exit 0
