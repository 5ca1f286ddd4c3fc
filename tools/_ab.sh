S="${S:-C2:;C3:;C4:;C5:}"
for v in ${VARIANTS:-old new}; do
  if [ $v = new ]; then unset LIB; else export LIB=variants/liblw_$v.so; fi
  SWEEP="$S" bash tools/gpu_sweep.sh > /dev/null; cp gpurun_out/sweep.log gpurun_out/sweep_$v.log
done
