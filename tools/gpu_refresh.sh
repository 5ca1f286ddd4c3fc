# refresh every committed profile in one GPU call: launch list + per-config trace traffic
# (gpu_evidence.sh), steady-state --set full captures (gpu_prof_final.sh) summarised on the box
# (the .ncu-rep files are too large to bring back), and the L1TEX breakdown of the C3 traversal
set -x
bash tools/gpu_evidence.sh > /dev/null 2>&1
python tools/traffic_json.py r01 > /dev/null
python tools/launch_summary.py gpurun_out/launches_C2.csv > gpurun_out/launch_shares.txt
bash tools/gpu_prof_final.sh > /dev/null 2>&1
python tools/profile_json.py r01 > /dev/null
for f in gpurun_out/r01_*.ncu-rep; do
  ncu -i $f --page raw --csv > ${f%.ncu-rep}_raw.csv 2>/dev/null
done
rm -f gpurun_out/*.ncu-rep
cp profiles/r01_ncu_stage_kernels.json profiles/trace_ext_traffic.json gpurun_out/
