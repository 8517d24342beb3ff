#!/bin/bash
# experiments: bench lines under environment switches; usage: NAME="ENV=.. ENV=.." pairs in $EXPS (semicolon separated "name:envs")
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
IFS=';' read -ra E <<< "$EXPS"
for x in "${E[@]}"; do
  name=${x%%:*}; envs=${x#*:}
  env $envs python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/exp_$name.json 2> gpurun_out/exp_$name.err
done
exit 0
