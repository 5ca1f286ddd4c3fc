# one ncu --set full capture: CFG (config) KREGEX (kernel regex) SKIP (launches to skip) CNT OUT
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e $EXTRA"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$KREGEX" -s ${SKIP:-300} -c ${CNT:-3} -o gpurun_out/$OUT -f $B --config $CFG > gpurun_out/$OUT.log 2>&1
tail -2 gpurun_out/$OUT.log
