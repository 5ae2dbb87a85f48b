for th in 14 8; do TCEC_STAGE_THREADS=$th timeout 600 python bench.py --steps 5 --warmup 3 --no-sweep --no-sliced --no-legs --no-cpu > gpurun_out/r3f_$th.jsonl 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/r3f_$th.jsonl').read().strip().splitlines()[-1])
print('threads=$th', d['value'], d['e2e']['value'], d['e2e'].get('pageable',{}).get('value'), d['e2e']['pipeline']['reruns'], d['clocks']['sm_mhz'])"; done
timeout 600 python -m pytest tests/test_gpu_dispatch.py tests/test_cpp_dropin.py -x -q -k "host or pageable or dropin" 2>&1 | tail -2
