timeout 600 python bench.py --workload rqc7x7 --depths 12,16 --steps 3 --warmup 2 > gpurun_out/r3g_7x7.jsonl 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/r3g_7x7.jsonl').read().strip().splitlines()[-1])
for r in d.get('depths', []): print(r.get('depth'), {k: v.get('ms_per_amplitude') for k, v in r.get('modes', {}).items()})
print({k: v for k, v in d.items() if k in ('value','unit')})"
TCEC_VIEW_GATHER=0 timeout 600 python bench.py --workload rqc7x7 --depths 16 --steps 3 --warmup 2 > gpurun_out/r3g_7x7_noview.jsonl 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/r3g_7x7_noview.jsonl').read().strip().splitlines()[-1])
print('noview', [(r.get('depth'), {k: v.get('ms_per_amplitude') for k, v in r.get('modes', {}).items()}) for r in d.get('depths', [])])"
timeout 600 python bench.py --workload sycamore --steps 3 --warmup 2 > gpurun_out/r3g_syc.jsonl 2>/dev/null; head -c 250 gpurun_out/r3g_syc.jsonl
