timeout 900 python -m pytest tests/test_tp_gpu.py -q -s > gpurun_out/r03c_tp_tests.log 2>&1; tail -3 gpurun_out/r03c_tp_tests.log
timeout 600 python tools/tp_decode.py --shape 7b --steps 32 > gpurun_out/r03c_tp1_7b.json 2>&1; tail -1 gpurun_out/r03c_tp1_7b.json
timeout 600 python tools/tp_decode.py --shape 7b --steps 32 --no-graphs > gpurun_out/r03c_tp1_7b_nograph.json 2>&1; tail -1 gpurun_out/r03c_tp1_7b_nograph.json
timeout 600 python tools/tp_decode.py --shape 7b --local 2 --steps 16 > gpurun_out/r03c_tp2local_7b.json 2>&1; tail -1 gpurun_out/r03c_tp2local_7b.json
