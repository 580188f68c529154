timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r03_gputests.log 2>&1; tail -3 gpurun_out/r03_gputests.log
timeout 600 python bench.py > gpurun_out/r03_bench.json 2> gpurun_out/r03_bench.err; tail -2 gpurun_out/r03_bench.json
echo done
