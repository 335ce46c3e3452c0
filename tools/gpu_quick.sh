# quick GPU cycle: gpu tests + path timings (tag as $1)
O=gpurun_out/${1:-q}; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 300 python tools/time_path.py cfg1 --once --lambdas 60 > $O/cfg1_60.json 2>&1
timeout 400 python tools/time_batch.py 148 > $O/cfg4_148_gram.json 2>&1
GS_CD_GRAM=0 timeout 400 python tools/time_batch.py 148 > $O/cfg4_148_direct.json 2>&1
timeout 600 python tools/time_path.py cfg2 20000 --once > $O/cfg2_p20000.json 2>&1
