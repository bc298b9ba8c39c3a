#!/bin/bash
# Round-end evidence on one B200 (run under gpurun from the repo root):
#   bench lines per config -> gpurun_out/f_<cfg>.json, reference arm -> f_ref.json,
#   ncu launch lists per config -> gpurun_out/ll_<cfg>.csv,
#   ncu --set full of the dominant kernels on C5 -> gpurun_out/full_<kernel>_C5.ncu-rep
# then locally: tools/make_summary.py, tools/make_profiles.py, tools/ncu_summary.py
set -x
mkdir -p gpurun_out
for c in C1 C2 C3 C4 C5; do
  python bench.py --config $c > gpurun_out/f_$c.json 2> gpurun_out/f_$c.err
done
python bench.py --impl reference > gpurun_out/f_ref.json 2> gpurun_out/f_ref.err
for c in C1 C2 C3 C4 C5; do python tools/one_step.py $c 1 > /dev/null 2>&1; done
bash tools/launch_list.sh C1 C2 C3 C4 C5
python tools/one_step.py C5 1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_columns4 -c 1 \
      -o gpurun_out/full_k_columns4_C5 python tools/one_step.py C5 1 > gpurun_out/ncu_full1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_columns4 -c 1 \
      -o gpurun_out/full_k_columns4_C4 python tools/one_step.py C4 1 > gpurun_out/ncu_full2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k4_fill -c 1 \
      -o gpurun_out/full_k4_fill_C5 python tools/one_step.py C5 1 > gpurun_out/ncu_full3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k4_place -c 1 \
      -o gpurun_out/full_k4_place_C5 python tools/one_step.py C5 1 > gpurun_out/ncu_full4.log 2>&1
ls -la gpurun_out
