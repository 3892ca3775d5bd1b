#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over tools/sanitize_target.py;
# summaries -> gpurun_out/r2/sanitizer_<tool>.log
mkdir -p gpurun_out/r2
for t in memcheck racecheck synccheck initcheck; do
  timeout -s KILL 900 /usr/local/cuda/bin/compute-sanitizer --tool $t --print-limit 20 \
      python tools/sanitize_target.py > gpurun_out/r2/sanitizer_$t.log 2>&1
  echo "$t rc=$?" >> gpurun_out/r2/sanitizer_$t.log
  tail -4 gpurun_out/r2/sanitizer_$t.log
done
