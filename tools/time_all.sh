# Path wall times of every BASELINE config on one B200 (round-end record)
O=gpurun_out/${1:-all}; mkdir -p $O
timeout 300 python tools/time_path.py cfg0 --once > $O/cfg0.json 2>&1
timeout 900 python tools/time_path.py cfg3 --once > $O/cfg3.json 2>&1
timeout 900 python tools/time_path.py cfg2 200000 --once > $O/cfg2_p200000.json 2>&1
timeout 900 python tools/time_batch.py 256 > $O/cfg4_256.json 2>&1
