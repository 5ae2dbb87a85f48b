timeout 1200 python bench.py > gpurun_out/r2r_bench.jsonl 2> gpurun_out/r2r_bench.err
echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/r2r_bench_ref.jsonl 2> gpurun_out/r2r_bench_ref.err
echo "ref rc=$?"
tail -c 600 gpurun_out/r2r_bench_ref.jsonl
