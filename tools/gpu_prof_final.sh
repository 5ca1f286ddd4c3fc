# steady-state ncu --set full captures of every wavefront stage kernel (timed instantiations only;
# the <true> instantiations run in bench.py's untimed work-counting pass)
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
N="ncu --set full --clock-control none --import-source on"
timeout 900 $N --kernel-name-base mangled -k 'regex:k_trace_extILb0E' -s 4 -c 1 -o gpurun_out/r01_C2_trace_ext -f $B --config C2 > /dev/null 2>&1
timeout 900 $N --kernel-name-base mangled -k 'regex:k_trace_shadowILb0E' -s 4 -c 1 -o gpurun_out/r01_C2_trace_shadow -f $B --config C2 > /dev/null 2>&1
timeout 900 $N -k 'regex:^k_shade$' -s 30 -c 1 -o gpurun_out/r01_C2_shade -f $B --config C2 > /dev/null 2>&1
timeout 900 $N -k 'regex:k_shade_nee' -s 30 -c 1 -o gpurun_out/r01_C2_shade_nee -f $B --config C2 > /dev/null 2>&1
timeout 900 $N -k 'regex:k_generate' -s 30 -c 1 -o gpurun_out/r01_C2_generate -f $B --config C2 > /dev/null 2>&1
timeout 900 $N --kernel-name-base mangled -k 'regex:k_trace_extILb0E' -s 4 -c 1 -o gpurun_out/r01_C3_trace_ext -f $B --config C3 > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
