cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b15.json 2> gpurun_out/b15.err
python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --mask 3 > gpurun_out/b3.json 2> gpurun_out/b3.err
bash tools/ncu_cfg4.sh r2a
