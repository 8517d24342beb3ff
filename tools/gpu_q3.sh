#!/bin/bash
# kernel-iteration check: correctness subset, cfg4 timing (3 steps), k_pair_edge phase split, optional extras
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -q -x -k "cfg1_all_pairs or zeta or row_chunks or schedule or tables or cfg5" > gpurun_out/q_tests.log 2>&1; echo "rc=$?" >> gpurun_out/q_tests.log
python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/q_b15.json 2> gpurun_out/q_b15.err
python tools/phase_prof.py > gpurun_out/phase_prof.txt 2>&1
[ -n "$EXTRA" ] && bash -c "$EXTRA"
exit 0
