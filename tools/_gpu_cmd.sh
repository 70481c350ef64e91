mkdir -p gpurun_out
timeout 900 python bench.py --config c5 --steps 1 --warmup 3 --no-cpu > gpurun_out/bench_c5.log 2>&1
timeout 600 python bench.py --config c1 --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_c1.log 2>&1
timeout 600 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_c2.log 2>&1
for f in bench_c5 bench_c1 bench_c2; do python -c "
import json
l=[x for x in open('gpurun_out/$f.log') if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print('$f', d and (d['value'], d['e2e']['value'], d['roofline']['product_ms_median'], d['roofline']['frac'], d['config'].get('entries_per_pixel')))
"; done
