#!/bin/bash
# compute-sanitizer (memcheck / racecheck / synccheck) over the GPU parity tests of the
# solver, the frame pipeline and the operators. Each tool's full log goes
# to gpurun_out/sanitizer_<tool>.log and its summary line to gpurun_out/sanitizer_summary.txt.
#   bash tools/sanitize.sh [pytest selection...]
set -u
SEL=${*:-tests/test_gpu_solver.py tests/test_gpu_pipeline.py tests/test_gpu_ops.py tests/test_gpu_orb.py}
mkdir -p gpurun_out
: > gpurun_out/sanitizer_summary.txt
for tool in memcheck racecheck synccheck; do
  extra=""
  [ "$tool" = "memcheck" ] && extra="--leak-check full"
  start=$(date +%s)
  timeout 1500 compute-sanitizer --tool $tool $extra --target-processes all --print-limit 50 \
    --log-file gpurun_out/sanitizer_$tool.log \
    python -m pytest $SEL -x -q -p no:cacheprovider > gpurun_out/sanitizer_${tool}_pytest.log 2>&1
  rc=$?
  end=$(date +%s)
  summ=$(grep -h "ERROR SUMMARY\|RACECHECK SUMMARY\|LEAK SUMMARY" gpurun_out/sanitizer_$tool.log | sort | uniq -c | tr '\n' ';')
  tests=$(tail -1 gpurun_out/sanitizer_${tool}_pytest.log)
  echo "$tool rc=$rc wall=$((end-start))s tests=[$tests] summary=[$summ]" >> gpurun_out/sanitizer_summary.txt
done
cat gpurun_out/sanitizer_summary.txt
