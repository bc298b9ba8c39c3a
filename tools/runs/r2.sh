set -x
python -m pytest tests -m gpu -x -q -k "partition or adapter or system_bitwise" > gpurun_out/t2.log 2>&1; tail -5 gpurun_out/t2.log
ncu --set full --import-source on --clock-control none -k regex:k_columns4 -c 1 -o gpurun_out/c4_cols4 python tools/one_step.py C4 1 > gpurun_out/ncu_c4.log 2>&1; tail -3 gpurun_out/ncu_c4.log
bash tools/launch_list.sh C4 C5
