# parity suite, then C2/C3 bench per library variant (LW_B200_LIB)
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
for lib in paper_1705_01263_b200/csrc/build/liblw_b200.so paper_1705_01263_b200/csrc/build/var_*.so; do
  for c in ${CONFIGS:-C2 C3}; do
    echo "$lib $c $(LW_B200_LIB=$PWD/$lib timeout 600 $B --config $c 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(round(d["value"]/1e6,1), "Mpaths/s", round(d["gsegments_per_s"],3), "Gseg/s trace_ms", round(r["avg_launch_ms"],4), "frac", round(r["frac"],3), "nodes", round(r["nodes_per_ray"],2))')"
  done
done > gpurun_out/variants.log 2>&1
cat gpurun_out/pytest_gpu.log gpurun_out/variants.log
