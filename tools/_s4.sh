timeout 900 python -m pytest tests/test_kernels_gpu.py -q -x -k "gemv" > gpurun_out/r03_gemv_tests.log 2>&1; tail -2 gpurun_out/r03_gemv_tests.log
FQ_GEMV_DIRECT_ALL=1 timeout 1200 python tools/gemv_sweep.py --iters 10 > gpurun_out/r03c_gemv_sweep.jsonl 2> gpurun_out/r03c_gemv_sweep.err; tail -2 gpurun_out/r03c_gemv_sweep.err
