O=gpurun_out/fin; mkdir -p $O
timeout 900 python tools/time_batch.py 256 > $O/cfg4_256.json 2>&1
timeout 300 python tools/time_path.py cfg1 --once --lambdas 60 > $O/cfg1_60.json 2>&1
timeout 900 python -m pytest tests/test_gpu_path.py tests/test_gpu_kernels.py tests/test_gpu_batch.py -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
GS_CSC_PAR=1 timeout 600 python -m pytest tests -m gpu -q -k "csc or sparse" > $O/pytest_cscpar.log 2>&1; echo "rc=$?" >> $O/pytest_cscpar.log
GS_CSC_PAR=1 timeout 900 python tools/time_path.py cfg3 --once > $O/cfg3_par.json 2>&1
