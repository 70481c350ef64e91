mkdir -p gpurun_out
for v in "" dg8; do
  if [ -n "$v" ]; then export SLM_LIB=paper_2409_12892_b200/_variants/$v/libsplatlm_b200.so; else unset SLM_LIB; fi
  timeout 600 python bench.py --config c4 --steps 1 --warmup 3 --no-cpu > gpurun_out/b4_$v.log 2>&1
  python -c "
import json
l=[x for x in open('gpurun_out/b4_$v.log') if x.startswith('{')]
d=json.loads(l[-1]); print('c4 ${v:-default}', d['value'], round(d['config']['phases_ms_per_step']['rhs']/8,2))
"
done
