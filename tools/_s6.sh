timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r03b_gputests.log 2>&1; tail -3 gpurun_out/r03b_gputests.log
timeout 1200 python tools/gemv_sweep.py --iters 10 > gpurun_out/r03b_gemv_sweep.jsonl 2> gpurun_out/r03b_gemv_sweep.err
timeout 600 python bench.py > gpurun_out/r03b_bench.json 2> gpurun_out/r03b_bench.err; tail -c 600 gpurun_out/r03b_bench.json
