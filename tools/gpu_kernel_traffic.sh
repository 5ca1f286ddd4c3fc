# ncu DRAM bytes + duration of every wavefront stage kernel launch (timed instantiations and the
# count pass alike; tools/kernel_traffic_json.py keeps the timed ones), per config, at the bench's
# default pool size: evidence for bench.py's roofline.kernels (profiles/r02_kernel_traffic.json).
# ncu serialises launches and replays each for its metrics: cold-cache numbers, shares not absolutes.
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-per-config"
for c in ${CONFIGS:-C1 C2 C3 C4 C5}; do
  timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:'k_generate|k_trace_ext|k_shade|k_trace_shadow' --csv --log-file gpurun_out/ktraffic_$c.csv \
    $B --config $c > gpurun_out/ktraffic_$c.log 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
  --log-file gpurun_out/launches_C2.csv $B --config C2 > /dev/null 2>&1
python tools/kernel_traffic_json.py > gpurun_out/r02_kernel_traffic.json  # copy to profiles/ after the call
ls gpurun_out
