#!/bin/bash
# After tools/runs/evidence.sh (gpurun_out/ merged back): write the tracked summaries under profiles/.
#   usage: bash tools/runs/collect.sh <tag>        e.g. r02
tag=${1:-r02}
[ -f gpurun_out/ev_ref_full_c5.json ] || cp profiles/${tag}_ref_full_C5.json gpurun_out/ev_ref_full_c5.json 2>/dev/null
python tools/make_summary.py $tag > /dev/null
python tools/make_profiles.py $tag C1 C2 C3 C4 C5 | grep "^# total"
K3=_ZN2fl10k_columns4ILi3ELi8ELi4ELb0ELi10EEEvNS_9ColParamsE
K2=_ZN2fl10k_columns4ILi2ELi8ELi1ELb0ELi8EEEvNS_9ColParamsE
python tools/ncu_summary.py gpurun_out/full_k_columns4_C5.ncu-rep profiles/${tag}_ncu_k_columns4_C5.txt "k_columns4<3,8,4> on C5 (unit_cube:256 permuted + coefficient): steady-state step" $K3 fl_columns4.cu > /dev/null
python tools/ncu_summary.py gpurun_out/full_k_columns4_C4.ncu-rep profiles/${tag}_ncu_k_columns4_C4.txt "k_columns4<3,8,4> on C4 (unit_cube:128): steady-state step" $K3 fl_columns4.cu > /dev/null
python tools/ncu_summary.py gpurun_out/full_k_columns4_C3.ncu-rep profiles/${tag}_ncu_k_columns4_C3.txt "k_columns4<2,8,1> on C3 (unit_square:4096 permuted): steady-state step" $K2 fl_columns4.cu > /dev/null
python tools/ncu_summary.py gpurun_out/full_k4_fill_C5.ncu-rep profiles/${tag}_ncu_k4_fill_C5.txt "k4_fill<4> on C5: steady-state step" > /dev/null
python tools/ncu_summary.py gpurun_out/full_k4_place_C5.ncu-rep profiles/${tag}_ncu_k4_place_C5.txt "k4_place on C5: steady-state step" > /dev/null
cp gpurun_out/ev_shards.jsonl profiles/${tag}_shard_ranks.jsonl
for c in 1 2 3 4 5; do cp gpurun_out/ev_bench_C$c.json profiles/${tag}_bench_C$c.json; done
cp gpurun_out/ev_ref.json profiles/${tag}_bench_reference.json
sed -n 5,12p profiles/${tag}_summary.md
