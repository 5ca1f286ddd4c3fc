# L1TEX breakdown of one launch: CFG, KREGEX (demangled-name regex), SKIP, OUT
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e $EXTRA"
timeout 900 ncu --kernel-name-base demangled --set full --clock-control none --import-source on -k "regex:$KREGEX" -s ${SKIP:-2} -c 1 -o gpurun_out/$OUT -f $B --config $CFG > gpurun_out/$OUT.log 2>&1
ncu -i gpurun_out/$OUT.ncu-rep --page raw --csv > gpurun_out/${OUT}_raw.csv
ncu -i gpurun_out/$OUT.ncu-rep --page source --csv --print-source sass > gpurun_out/${OUT}_sass.csv 2>/dev/null
rm -f gpurun_out/$OUT.ncu-rep
