S="C3:;C5:;C4:"
SWEEP="$S" bash tools/gpu_sweep.sh > /dev/null; cp gpurun_out/sweep.log gpurun_out/sweep_base.log
export LW_PERSIST=1
SWEEP="$S" bash tools/gpu_sweep.sh > /dev/null; cp gpurun_out/sweep.log gpurun_out/sweep_p.log
export LW_PERSIST_SH=1
SWEEP="$S" bash tools/gpu_sweep.sh > /dev/null; cp gpurun_out/sweep.log gpurun_out/sweep_psh.log
python -m pytest tests -m gpu -x -q 2>&1 | tail -2 > gpurun_out/gpu_tests.txt
