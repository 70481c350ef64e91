mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_offload.py tests/test_distributed_gpu.py tests/test_lm_outer.py tests/test_c2_subset.py -m gpu -q -x 2>&1 | tail -15 > gpurun_out/ov_tests.log
SLM_OVERLAP=0 timeout 900 python bench.py --no-cpu > gpurun_out/ov_off.log 2>&1
timeout 900 python bench.py --no-cpu > gpurun_out/ov_on.log 2>&1
cat gpurun_out/ov_tests.log
for f in ov_off ov_on; do python -c "
import json
l=[x for x in open('gpurun_out/$f.log') if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print('$f', d and (d['value'], d['e2e']['value'], d['roofline']['product_ms_median'], d['roofline']['frac']))
"; done
tail -5 gpurun_out/ov_on.log | cut -c1-300
