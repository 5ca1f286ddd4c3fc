# Round-2 evidence in one GPU call: the default bench line (headline + per_config + roofline.kernels
# + CPU baselines), ncu --set full captures of the stage kernels (timed instantiations, a
# full-size wave), the per-stage-kernel DRAM traffic (tools/gpu_kernel_traffic.sh) and the C2/C3
# launch lists.  Copy the gpurun_out/ products into profiles/ afterwards (tools/prof_r02_collect.sh).
# DRAM traffic first, so the bench line's roofline.kernels carries this code's ncu bytes
bash tools/gpu_kernel_traffic.sh > /dev/null 2>&1
cp gpurun_out/r02_kernel_traffic.json profiles/r02_kernel_traffic.json
python bench.py > gpurun_out/r02_bench_final.json 2> gpurun_out/r02_bench_final.err
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-per-config"
N="ncu --set full --clock-control none --import-source on --kernel-name-base mangled"
# launch indices among the matching kernels: COUNT pass excluded by the mangled <0>; -s 1 = wave 2 of the warm-up pass
timeout 900 $N -k 'regex:k_shadeILb0ELb0ELb0E' -s 9 -c 1 -o gpurun_out/r02_C2_shade -f $B --config C2 > /dev/null 2>&1
timeout 900 $N -k 'regex:k_shade_neeILb0ELb0ELb0E' -s 9 -c 1 -o gpurun_out/r02_C2_shade_nee -f $B --config C2 > /dev/null 2>&1
timeout 900 $N -k 'regex:k_trace_ext_pILb0E' -s 1 -c 1 -o gpurun_out/r02_C2_trace_ext -f $B --config C2 > /dev/null 2>&1
timeout 900 $N -k 'regex:k_trace_shadow_pILb0ELb0E' -s 1 -c 1 -o gpurun_out/r02_C2_trace_shadow -f $B --config C2 > /dev/null 2>&1
timeout 900 $N -k 'regex:k_generateILb0ELb0E' -s 9 -c 2 -o gpurun_out/r02_C2_generate -f $B --config C2 > /dev/null 2>&1
for c in C3 C5; do
  timeout 900 $N -k 'regex:k_trace_ext_pILb0E' -s 1 -c 1 -o gpurun_out/r02_${c}_trace_ext -f $B --config $c > /dev/null 2>&1
done
timeout 900 $N -k 'regex:k_shadeILb0ELb0ELb0E' -s 9 -c 1 -o gpurun_out/r02_C4_shade -f $B --config C4 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
  --log-file gpurun_out/launches_C3.csv $B --config C3 > /dev/null 2>&1
# summaries on the box (gpurun brings back at most 64 MiB: the reports themselves stay there)
for r in gpurun_out/r02_*.ncu-rep; do
  b=$(basename $r .ncu-rep)
  python tools/ncu_summary.py $r --json gpurun_out/${b}_summary.json > /dev/null 2>&1
  k=$(echo $b | sed -e 's/r02_C[0-9]_//')
  python tools/ncu_lines.py $r "k_${k}" 40 > gpurun_out/${b}_lines.txt 2>&1
done
rm -f gpurun_out/*.ncu-rep
ls -la gpurun_out/
