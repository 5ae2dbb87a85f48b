SH="2x67108864x2,8x16777216x8,16x4194304x16,16x16777216x16,4x16777216x32,16x4194304x64,32x8388608x8,16777216x8x8,67108864x2x2,4194304x32x8,2097152x16x32,1048576x16x16,4194304x16x64"
for x in 0 1; do echo "TCEC_SKINNY_X2=$x"; SHAPES=$SH TCEC_SKINNY_X2=$x timeout 300 python tools/bench_skinny.py; done > gpurun_out/skinny_x2.log 2>&1
timeout 600 python -m pytest tests/test_gpu_cgemm.py tests/test_gpu_network.py -q -x -k "skinny or extreme or long_k or fp32 or rqc or network" > gpurun_out/t_skinny.log 2>&1
echo "rc=$?" >> gpurun_out/t_skinny.log
