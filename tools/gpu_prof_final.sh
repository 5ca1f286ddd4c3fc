# steady-state ncu --set full captures of every wavefront stage kernel (timed instantiations only;
# the <true> COUNT instantiations run in bench.py's untimed work-counting pass)
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
N="ncu --set full --clock-control none --import-source on"
for c in C1 C2 C3 C4 C5; do
  timeout 900 $N --kernel-name-base mangled -k 'regex:k_trace_ext(_p)?ILb0E' -s 4 -c 1 -o gpurun_out/r01_${c}_trace_ext -f $B --config $c > /dev/null 2>&1
done
timeout 900 $N --kernel-name-base mangled -k 'regex:k_trace_shadow(_p)?ILb0ELb0E' -s 4 -c 1 -o gpurun_out/r01_C2_trace_shadow -f $B --config C2 > /dev/null 2>&1
timeout 900 $N --kernel-name-base mangled -k 'regex:k_shadeILb0E' -s 20 -c 1 -o gpurun_out/r01_C2_shade -f $B --config C2 > /dev/null 2>&1
timeout 900 $N --kernel-name-base mangled -k 'regex:k_shade_neeILb0E' -s 20 -c 1 -o gpurun_out/r01_C2_shade_nee -f $B --config C2 > /dev/null 2>&1
timeout 900 $N --kernel-name-base mangled -k 'regex:k_generateILb0E' -s 20 -c 1 -o gpurun_out/r01_C2_generate -f $B --config C2 > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
