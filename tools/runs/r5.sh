python -m pytest tests -m gpu -x -q > gpurun_out/t5.log 2>&1; tail -5 gpurun_out/t5.log
bash tools/quick.sh C4 C5 C3 > gpurun_out/q5.log 2>&1; cat gpurun_out/q5.log
bash tools/launch_list.sh C5
