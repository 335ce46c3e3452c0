#!/bin/bash
# compute-sanitizer on the persistent kernels at small shapes; logs under
# gpurun_out/TAG/ (copied to profiles/ when clean).   usage: tools/gpu_sanitize.sh TAG
TAG=${1:-san}; O=gpurun_out/$TAG; mkdir -p $O
CS=/usr/local/cuda/bin/compute-sanitizer
for what in dense csc batch; do
  for mode in ${MODES:-2 0}; do
    [ "$what" != dense ] && [ "$mode" != 2 ] && continue
    for tool in memcheck racecheck synccheck; do
      GS_CD_GRAM=$mode timeout 900 $CS --tool $tool --print-limit 20 python tools/sanitize_case.py $what \
         > $O/${tool}_${what}_mode$mode.log 2>&1
      echo "rc=$?" >> $O/${tool}_${what}_mode$mode.log
    done
  done
done
grep -H "ERROR SUMMARY\|RACECHECK SUMMARY\|rc=" $O/*check_*.log > $O/summary.txt
