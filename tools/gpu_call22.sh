#!/bin/bash
O=gpurun_out/c22; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_path.py tests/test_gpu_kernels.py tests/test_gpu_fullsize.py -m gpu -q -rf -x -k "sparse or csc or cfg3" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 900 python tools/time_path.py cfg3 --once --lambdas 70 > $O/cfg3_l70.json 2> $O/cfg3_l70.err
timeout 600 python tools/time_path.py cfg1 --once > $O/cfg1.json 2> $O/cfg1.err
