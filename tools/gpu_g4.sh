cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
bash tools/ncu_cfg4.sh r2a
python tools/phase_prof.py > gpurun_out/phase_prof.txt 2>&1
