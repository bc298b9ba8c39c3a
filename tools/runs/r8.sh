python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -x -q > gpurun_out/t8.log 2>&1; tail -2 gpurun_out/t8.log
bash tools/quick.sh C4 C5 C3 C2 C1 > gpurun_out/q8.log 2>&1; cat gpurun_out/q8.log
FL_V4_MINB=8 bash tools/quick.sh C5 > gpurun_out/q8b.log 2>&1; cat gpurun_out/q8b.log
ncu --set full --import-source on --clock-control none -k regex:k_columns4 -c 1 -o gpurun_out/c4_cols4e python tools/one_step.py C4 1 > /dev/null 2>&1
