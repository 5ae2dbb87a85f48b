for f in 4 2 3 6; do
  TCEC_HOST_BFRONT=$f timeout 600 python bench.py --steps 5 --warmup 3 --no-sweep --no-sliced --no-legs --no-cpu --no-pageable > gpurun_out/r2x_bfront$f.jsonl 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/r2x_bfront$f.jsonl').read().strip().splitlines()[-1])
print('BFRONT=$f', d['value'], d['e2e']['value'], d['e2e']['pipeline'], d['clocks']['sm_mhz'])"
done
