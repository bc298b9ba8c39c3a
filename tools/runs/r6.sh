python -m pytest tests -m gpu -x -q > gpurun_out/t6.log 2>&1; tail -5 gpurun_out/t6.log
bash tools/quick.sh C4 C5 C3 > gpurun_out/q6.log 2>&1; cat gpurun_out/q6.log
FL_LABELS=first bash tools/quick.sh C5 > gpurun_out/q6f.log 2>&1; cat gpurun_out/q6f.log
bash tools/launch_list.sh C5 C3
