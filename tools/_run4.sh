timeout 1200 python bench.py > gpurun_out/bench_r2c.jsonl 2> gpurun_out/bench_r2c.err
echo "rc=$?" >> gpurun_out/bench_r2c.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_r2c.jsonl 2> gpurun_out/bench_ref_r2c.err
