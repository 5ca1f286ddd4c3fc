# per-config evidence for bench.py's roofline: DRAM bytes + duration of every k_trace_ext launch
# (ncu lightweight metrics, serialised), plus the full launch list of the C2 headline run.
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
for c in ${CONFIGS:-C1 C2 C3 C4 C5}; do
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:k_trace_ext --csv --log-file gpurun_out/traffic_$c.csv $B --config $c > /dev/null 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
  --log-file gpurun_out/launches_C2.csv $B --config C2 > /dev/null 2>&1
ls gpurun_out
