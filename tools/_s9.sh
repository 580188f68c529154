timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r03d_gputests.log 2>&1; tail -3 gpurun_out/r03d_gputests.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r03d_bench.json 2> gpurun_out/r03d_bench.err; tail -c 400 gpurun_out/r03d_bench.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r03d_bench_ref.json 2> gpurun_out/r03d_bench_ref.err; tail -c 400 gpurun_out/r03d_bench_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r03d_launches.csv python bench.py --steps 2 --warmup 1 > gpurun_out/r03d_ncu_bench.log 2>&1; tail -2 gpurun_out/r03d_ncu_bench.log
