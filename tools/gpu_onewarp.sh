O=gpurun_out/ow; mkdir -p $O
GS_CD_ONEWARP=1 timeout 300 python tools/time_path.py cfg1 --once --lambdas 60 > $O/cfg1_60_onewarp.json 2>&1
timeout 300 python tools/time_path.py cfg1 --once --lambdas 60 > $O/cfg1_60_default.json 2>&1
GS_CD_ONEWARP=1 GS_CD_GRAM=0 timeout 600 python tools/time_path.py cfg1 --once > $O/cfg1_onewarp.json 2>&1
GS_CD_ONEWARP=1 timeout 600 python -m pytest tests/test_gpu_path.py -q -k "cfg1" > $O/pytest_onewarp.log 2>&1
