O=gpurun_out/bt2; mkdir -p $O
timeout 900 python tools/time_batch.py 256 > $O/cfg4_256.json 2>&1
if grep -q "launch failure\|watchdog" $O/cfg4_256.json; then
  for c in "148 175" "175 202" "202 229" "229 256"; do set -- $c; timeout 400 python tools/batch_chunks.py $1 $2 > $O/chunk_$1.log 2>&1; done
fi
