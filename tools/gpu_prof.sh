# ncu --set full captures of the wavefront stage kernels (steady-state launches, after the
# untimed instrumented pass and warm-up)
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:k_trace_ext|k_trace_shadow|k_shade|k_generate' -s 600 -c 5 -o gpurun_out/prof_C2 -f $B --config C2 > gpurun_out/prof_C2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:k_trace_ext|k_trace_shadow' -s 120 -c 2 -o gpurun_out/prof_C3 -f $B --config C3 > gpurun_out/prof_C3.log 2>&1
ls -la gpurun_out
