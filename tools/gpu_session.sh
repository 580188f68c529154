set -x
timeout 900 python -m pytest tests/test_batched_gpu.py -m gpu -q -x 2>&1 | tail -2
timeout 900 python tools/batched_decode.py --shape 13b --batches 16,32 --prompt 128 --steps 8 2>&1 | tail -3
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/batched_launches.csv python tools/batched_decode.py --shape 13b --batches 32 --prompt 128 --steps 1 > gpurun_out/ncu_batched.log 2>&1; tail -2 gpurun_out/ncu_batched.log
