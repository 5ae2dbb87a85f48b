# rasterization sweep of the wide kernel at n=16384: DRAM bytes (ncu) and time
for g in ${GMS:-1 2 4 8}; do
 echo "GROUP_M=$g"
 TCEC_GROUP_M=$g timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:tcec_gemm_wide --launch-count 1 --csv python tools/prof_gemm.py --n ${N:-16384} --mode AUTO --reps 1 2>&1 | grep -E "dram__bytes_read|duration" | awk -F'","' '{print $13, $15}'
done
for r in 1 2; do for g in ${GMS:-1 2 4 8}; do
 echo -n "GROUP_M=$g "; TCEC_GROUP_M=$g VARIANTS=wide NS=${N:-16384} MODES=AUTO ROUNDS=1 timeout 300 python tools/ab_gemm.py
done; done
