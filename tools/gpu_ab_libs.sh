# A/B of library variants (variants/liblw_<name>.so, "new" = the in-tree build) + the GPU tests:
# S="C2:;C3:" VARIANTS="old new" bash tools/gpu_ab_libs.sh -> gpurun_out/sweep_<name>.log
S="${S:-C3:;C4:;C5:}"
for v in ${VARIANTS:-old spec new}; do
  if [ $v = new ]; then unset LIB; else export LIB=variants/liblw_$v.so; fi
  SWEEP="$S" bash tools/gpu_sweep.sh > /dev/null; cp gpurun_out/sweep.log gpurun_out/sweep_$v.log
done
unset LIB
python -m pytest tests -m gpu -x -q 2>&1 | tail -2 > gpurun_out/gpu_tests.txt
