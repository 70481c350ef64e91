mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_c2_subset.py tests/test_large_regime.py -m gpu -q -x 2>&1 | tail -2 > gpurun_out/pytest_gpu.log
timeout 900 python bench.py --config c4 --steps 2 --warmup 3 --no-cpu > gpurun_out/bench_c4.log 2>&1
cat gpurun_out/pytest_gpu.log; python -c "
import json
l=[x for x in open('gpurun_out/bench_c4.log') if x.startswith('{')]
d=json.loads(l[-1]); print(d['value'], d['e2e']['value'], d['roofline']['product_ms_median'], d['roofline']['frac'])
"
