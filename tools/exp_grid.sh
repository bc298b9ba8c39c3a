mkdir -p gpurun_out
for c in C5 C4; do
  for u in 1 2 4 8; do
    FL_FILL_U=$u TAG="U$u" timeout 300 python tools/quick_phases.py $c 5 >> gpurun_out/exp.log 2>&1
  done
done
for fb in 0 1; do FL_FILLB_GRID=$fb TAG="fillb$fb" timeout 300 python tools/quick_phases.py C3 5 >> gpurun_out/exp.log 2>&1; done
cat gpurun_out/exp.log
