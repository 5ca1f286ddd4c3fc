# bench sweep over extra bench.py flags: SWEEP="C2:--pool-log2 18;C3:--pool-log2 19;..."
# optional LIB=<path of a variant liblw_b200.so relative to the repo>
B=(python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e)
[ -n "$LIB" ] && export LW_B200_LIB=$PWD/$LIB
: > gpurun_out/sweep.log
echo "$SWEEP" | tr ';' '\n' | while read -r item; do
  [ -z "$item" ] && continue
  c=${item%%:*}; flags=${item#*:}
  echo "$c [$flags] $(timeout 600 "${B[@]}" --config $c $flags 2>>gpurun_out/sweep.err | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(round(d["value"]/1e6,1), "Mpaths/s", round(d["gsegments_per_s"],3), "Gseg/s trace_ms", round(r["avg_launch_ms"],4), "share", round(r["trace_share_of_step"],3), "launches", d["gpu_launches"])')" >> gpurun_out/sweep.log
done
cat gpurun_out/sweep.log
