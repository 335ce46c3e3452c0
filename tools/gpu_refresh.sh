O=gpurun_out/rf; mkdir -p $O
for e in 32 8 2 0; do GS_REFRESH_EXCESS=$e timeout 300 python tools/time_path.py cfg1 --once --lambdas 80 > $O/cfg1_80_re$e.json 2>&1; done
