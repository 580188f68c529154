set -x
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_c3_shape_gpu.py tests/test_model_gpu.py -m gpu -q -x -k "tcgen05 or c3 or tensor_core or kl_calibration" > gpurun_out/gemm_tests.log 2>&1; tail -3 gpurun_out/gemm_tests.log; grep "max rel" gpurun_out/gemm_tests.log | head -20
timeout 600 python tools/gemm_bench.py --T 256,512,2048 --iters 10 > gpurun_out/gemm_bench_r02b.jsonl 2>&1; cat gpurun_out/gemm_bench_r02b.jsonl
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_ws -s 2 -c 1 -o gpurun_out/gemm_ws_r02b python tools/gemm_bench.py --T 2048 --shapes 1 --bits 8 --iters 2 > gpurun_out/ncu_gemm.log 2>&1; tail -1 gpurun_out/ncu_gemm.log
