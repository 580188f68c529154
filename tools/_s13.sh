for i in 1 2 3 4; do timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r03j_bench_$i.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/r03j_bench_$i.json').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d['e2e']['value'], d['e2e']['trace'], d['e2e']['note'][-18:])"; done
