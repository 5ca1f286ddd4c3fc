# final-state refresh of the round-2 evidence that depends on the code path: the default bench
# line and the per-stage-kernel DRAM traffic (the ncu --set full summaries are from
# tools/gpu_prof_r02.sh)
python bench.py > gpurun_out/r02_bench_final.json 2> gpurun_out/r02_bench_final.err
bash tools/gpu_kernel_traffic.sh > /dev/null 2>&1
rm -f gpurun_out/ktraffic_*.csv
ls -la gpurun_out/
