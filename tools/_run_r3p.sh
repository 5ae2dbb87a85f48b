for g in 4 2 8 6; do TCEC_GROUP_M=$g timeout 600 python bench.py --steps 5 --warmup 3 --no-sweep --no-sliced --no-legs --no-cpu --no-pageable > gpurun_out/r3p_g$g.jsonl 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/r3p_g$g.jsonl').read().strip().splitlines()[-1])
print('group_m=$g', d['value'], d['roofline']['achieved'], d['roofline']['frac_at_clock'], d['clocks']['sm_mhz'])"; done
