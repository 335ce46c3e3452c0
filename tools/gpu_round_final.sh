bash tools/gpu_round.sh r01e 2
timeout 900 python tools/time_path.py cfg3 --once > gpurun_out/r01e/cfg3.json 2>&1
