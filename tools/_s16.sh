timeout 900 python -m pytest tests/test_model_gpu.py -q -k "chain or teacher_forced" > gpurun_out/r03m_chain_tests.log 2>&1; tail -3 gpurun_out/r03m_chain_tests.log
for i in 1 2; do timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r03m_bench_$i.json 2>gpurun_out/r03m_bench_$i.err; tail -2 gpurun_out/r03m_bench_$i.err; python -c "
import json; d=json.loads(open('gpurun_out/r03m_bench_$i.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['per_launch_ms'], d['roofline']['frac'], d['config']['scheduler'], d['gpu_launches'])"; done
timeout 600 python bench.py > gpurun_out/r03m_bench200.json 2>gpurun_out/r03m_bench200.err; python -c "
import json; d=json.loads(open('gpurun_out/r03m_bench200.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['per_launch_ms'], d['roofline']['frac'], d['config']['scheduler'])"
