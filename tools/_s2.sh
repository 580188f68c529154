timeout 300 python tools/_dbg_tp.py > gpurun_out/r03_dbg.log 2>&1; tail -12 gpurun_out/r03_dbg.log
timeout 900 python -m pytest tests/test_tp_gpu.py -q -s > gpurun_out/r03_tp_tests.log 2>&1; tail -3 gpurun_out/r03_tp_tests.log
