python -m pytest tests -m gpu -x -q > gpurun_out/t4.log 2>&1; tail -15 gpurun_out/t4.log
bash tools/quick.sh C4 C5 C3 > gpurun_out/q4.log 2>&1; cat gpurun_out/q4.log
ncu --set full --import-source on --clock-control none -k regex:k_columns4 -c 1 -o gpurun_out/c4_cols4c python tools/one_step.py C4 1 > gpurun_out/ncu_c4c.log 2>&1; tail -1 gpurun_out/ncu_c4c.log
