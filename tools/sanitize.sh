cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python tools/sanitize_cfg1.py > gpurun_out/san_plain.log 2>&1
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_cfg1.py > gpurun_out/san_$tool.log 2>&1
  echo "$tool exit $?" >> gpurun_out/san_summary.txt
  tail -3 gpurun_out/san_$tool.log >> gpurun_out/san_summary.txt
done
timeout 1200 compute-sanitizer --tool memcheck python tools/sanitize_cfg1.py 8 > gpurun_out/san_memcheck_p8.log 2>&1
echo "memcheck p8 exit $?" >> gpurun_out/san_summary.txt; tail -3 gpurun_out/san_memcheck_p8.log >> gpurun_out/san_summary.txt
