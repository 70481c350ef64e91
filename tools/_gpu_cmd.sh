mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/pytest_gpu.log
timeout 900 python bench.py --config c4 --steps 2 --warmup 3 --no-cpu > gpurun_out/bench_c4.log 2>&1
timeout 900 python bench.py --no-cpu > gpurun_out/bench_c3_chk.log 2>&1
timeout 600 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_c2.log 2>&1
cat gpurun_out/pytest_gpu.log
for f in bench_c4 bench_c3_chk bench_c2; do python -c "
import json
l=[x for x in open('gpurun_out/$f.log') if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print('$f', d and (d['value'], d['e2e']['value'], d['roofline']['product_ms_median'], d['roofline']['frac']))
"; done
