for i in 1 2; do timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r03o_bench_$i.json 2>gpurun_out/r03o_bench_$i.err; tail -1 gpurun_out/r03o_bench_$i.err; python -c "
import json; d=json.loads(open('gpurun_out/r03o_bench_$i.json').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d['e2e']['value'], d['e2e']['trace'], d['e2e']['note'][-18:], d['gpu_launches'])"; done
timeout 600 python bench.py > gpurun_out/r03o_bench200.json 2>gpurun_out/r03o_bench200.err; python -c "
import json; d=json.loads(open('gpurun_out/r03o_bench200.json').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d['e2e']['value'], d['e2e']['trace'])"
