for lib in new old; do
  if [ $lib = old ]; then export TCEC_LIB_PATH=oldlib/libtcec_prev.so; else unset TCEC_LIB_PATH; fi
  for v in 1 0; do
    TCEC_VIEW_GATHER=$v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2u_$lib$v.csv python tools/bench_skinny_view.py 28 6 4 1 > /dev/null 2>&1
    echo "== lib=$lib view=$v"; python tools/launch_summary.py gpurun_out/r2u_$lib$v.csv | head -4
  done
done
