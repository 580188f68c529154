timeout 900 python -m pytest tests/test_tp_gpu.py -q -x -s > gpurun_out/r03_tp_tests.log 2>&1; tail -3 gpurun_out/r03_tp_tests.log
timeout 300 python tools/tp_decode.py --local 2 --layers 2 --steps 8 > gpurun_out/r03_tp_local.json 2>&1; tail -2 gpurun_out/r03_tp_local.json
timeout 600 python tools/tp_decode.py --shape 7b --steps 32 > gpurun_out/r03_tp1_7b.json 2>&1; tail -2 gpurun_out/r03_tp1_7b.json
echo done
