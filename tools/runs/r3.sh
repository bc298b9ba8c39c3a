python -m pytest tests -m gpu -x -q > gpurun_out/t3.log 2>&1; tail -15 gpurun_out/t3.log
bash tools/quick.sh C4 C5 C3 > gpurun_out/q3.log 2>&1; cat gpurun_out/q3.log
ncu --set full --import-source on --clock-control none -k regex:k_columns4 -c 1 -o gpurun_out/c4_cols4b python tools/one_step.py C4 1 > gpurun_out/ncu_c4b.log 2>&1; tail -2 gpurun_out/ncu_c4b.log
