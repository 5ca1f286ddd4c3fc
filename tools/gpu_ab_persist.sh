# A/B of LW_TRACE_PERSIST masks: S="C2:;C1:" MASKS="3 15" bash tools/gpu_ab_persist.sh -> gpurun_out/sweep_m<mask>.log
S="${S:-C2:;C1:}"
for m in ${MASKS:-3 7 11 15}; do
  LW_TRACE_PERSIST=$m SWEEP="$S" bash tools/gpu_sweep.sh > /dev/null; cp gpurun_out/sweep.log gpurun_out/sweep_m$m.log
done
