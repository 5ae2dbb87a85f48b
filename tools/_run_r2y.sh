nproc
timeout 600 python bench.py --steps 5 --warmup 3 --no-sweep --no-sliced --no-legs --no-cpu > gpurun_out/r2y_bench.jsonl 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/r2y_bench.jsonl').read().strip().splitlines()[-1])
print(d['value'], d['e2e']['value'], d['e2e'].get('pageable'), d['e2e']['pipeline']['reruns'], d['clocks']['sm_mhz'])"
timeout 900 python -m pytest tests/test_gpu_dispatch.py tests/test_cpp_dropin.py tests/test_reference_suite.py -x -q > gpurun_out/r2y_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2y_pytest.log; tail -2 gpurun_out/r2y_pytest.log
