# Interleaved A/B of bench throughput over variants (environment overrides and/or library builds):
#   AB="base|LW_MATCLASS=0|;m5||variants/liblw_m5.so;cmp|||--state compact" CONFIGS="C2 C5" REPS=2 bash tools/gpu_ab.sh
# (fields: name | environment overrides | library variant | extra bench.py flags)
# -> gpurun_out/ab.log, one line per (rep, config, variant): Mpaths/s and the stage shares
: > gpurun_out/ab.log
for rep in $(seq 1 ${REPS:-2}); do
  for c in ${CONFIGS:-C2}; do
    echo "$AB" | tr ';' '\n' | while IFS='|' read -r name envs lib extra; do
      [ -z "$name" ] && continue
      out=$(env $envs ${lib:+LW_B200_LIB=$PWD/$lib} timeout 600 python bench.py --steps ${STEPS:-10} --warmup 3 \
            --no-cpu-baseline --no-e2e --no-per-config --config $c ${FLAGS} $extra 2>>gpurun_out/ab.err)
      echo "$rep $c $name $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e6,1), {k["stage"]: round(k["avg_launch_ms"],3) for k in d["roofline"]["kernels"]})')" >> gpurun_out/ab.log
    done
  done
done
cat gpurun_out/ab.log
