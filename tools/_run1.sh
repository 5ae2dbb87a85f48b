timeout 300 python -m pytest tests/test_gpu_cgemm.py -q -x -k "multicast or (variants and wide_mc) or (all_positive and wide_mc)" > gpurun_out/t_mc.log 2>&1
echo "mc_tests rc=$?" >> gpurun_out/t_mc.log
if grep -q "passed" gpurun_out/t_mc.log && ! grep -q "failed" gpurun_out/t_mc.log; then
  timeout 600 python tools/ab_headline.py 16384 wide,wide_mc 1 AUTO,FP16TCEC > gpurun_out/ab_headline.log 2>&1
  TCEC_TF32_FLUSH=2 timeout 300 python tools/ab_headline.py 16384 wide,wide_mc 1 AUTO >> gpurun_out/ab_headline.log 2>&1
fi
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool initcheck --target-processes all --print-limit 20 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_prep.py tests/test_gpu_cgemm.py tests/test_gpu_network.py tests/test_gpu_batch_errors.py -q -x -k 'not full_size and not long_k_kernels and not extreme_aspect and not split_k and not accuracy_uniform and not golden and not 4096 and not 8192 and not all_positive and not multicast' -p no:cacheprovider > gpurun_out/sanitizer_initcheck2.log 2>&1
