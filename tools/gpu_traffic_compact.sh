B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-per-config --state compact"
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:'k_generate|k_trace_ext|k_shade|k_trace_shadow' --csv --log-file gpurun_out/ktraffic_C2cmp.csv $B --config C2 > /dev/null 2>&1
