python -m pytest tests/test_gpu_parity.py -x -q -k "stiffness or system" > gpurun_out/t7.log 2>&1; tail -2 gpurun_out/t7.log
for cfg in "FL_V4_MINB=8" "FL_V4_MINB=10" "FL_V4_SHAPE=16x2 FL_V4_MINB=8" "FL_V4_SHAPE=16x2 FL_V4_MINB=10"; do
  echo "== $cfg"; env $cfg bash tools/quick.sh C4 C5
done > gpurun_out/q7.log 2>&1; cat gpurun_out/q7.log
ncu --set full --import-source on --clock-control none -k regex:k_columns4 -c 1 -o gpurun_out/c4_cols4d python tools/one_step.py C4 1 > /dev/null 2>&1
