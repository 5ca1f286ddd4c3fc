# run gpu_sweep.sh for the default library and every variant in csrc/build/var_*.so
for lib in "" paper_1705_01263_b200/csrc/build/var_*.so; do
  echo "== ${lib:-default}"
  LIB=$lib bash tools/gpu_sweep.sh
done 2>&1 | tee gpurun_out/multi.log
