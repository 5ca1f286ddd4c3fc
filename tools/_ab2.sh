S="${S:-C2:;C1:}"
for m in ${MASKS:-3 7 11 15}; do
  LW_TRACE_PERSIST=$m SWEEP="$S" bash tools/gpu_sweep.sh > /dev/null; cp gpurun_out/sweep.log gpurun_out/sweep_m$m.log
done
