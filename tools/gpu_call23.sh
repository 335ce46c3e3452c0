#!/bin/bash
O=gpurun_out/c23; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_path.py tests/test_gpu_kernels.py tests/test_gpu_fullsize.py tests/test_gpu_csc_api.py -m gpu -q -rf -x -k "sparse or csc or cfg3 or elastic or tail" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 900 python tools/time_path.py cfg3 --once --lambdas 70 > $O/cfg3_l70.json 2> $O/cfg3_l70.err
GS_CSC_SEQ=0 timeout 900 python tools/time_path.py cfg3 --once --lambdas 70 > $O/cfg3_l70_waves.json 2> $O/cfg3_l70_waves.err
timeout 1500 python tools/time_path.py cfg3 --once > $O/cfg3.json 2> $O/cfg3.err
for ch in 4096 65536 0; do
GS_CD_CHUNK=$ch timeout 900 python tools/time_path.py cfg3 --once --lambdas 70 > $O/cfg3_l70_chunk$ch.json 2> $O/cfg3_chunk$ch.err
done
