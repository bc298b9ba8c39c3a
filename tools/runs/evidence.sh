#!/bin/bash
# Round evidence on one B200 (run under gpurun from the repo root):
#   bench lines per config        -> gpurun_out/ev_bench_<cfg>.json
#   reference arm                 -> gpurun_out/ev_ref.json
#   ncu launch lists (last step)  -> gpurun_out/ll_<cfg>.csv
#   ncu --set full captures of the steady-state launch of the top kernels
#   single-rank times of a sharded step (tools/shard_step.py) -> ev_shards.jsonl
# then locally: tools/make_summary.py, tools/make_profiles.py, tools/ncu_summary.py
mkdir -p gpurun_out
nproc > gpurun_out/ev_nproc.txt; free -g >> gpurun_out/ev_nproc.txt; lscpu | head -20 >> gpurun_out/ev_nproc.txt
python bench.py > gpurun_out/ev_bench_C5.json 2> gpurun_out/ev_bench_C5.err
for c in C1 C2 C3 C4; do python bench.py --config $c > gpurun_out/ev_bench_$c.json 2> gpurun_out/ev_bench_$c.err; done
python bench.py --impl reference > gpurun_out/ev_ref.json 2> gpurun_out/ev_ref.err
bash tools/launch_list.sh C1 C2 C3 C4 C5
full() {  # kernel regex, config, output name: the second (steady-state) launch of the kernel
  ncu --set full --clock-control none --import-source on -k regex:$1 --launch-skip 1 -c 1 \
      -o gpurun_out/full_$3 python tools/one_step.py $2 1 > gpurun_out/ncu_full_$3.log 2>&1
}
full k_columns4 C5 k_columns4_C5
full k_columns4 C4 k_columns4_C4
full k_columns4 C3 k_columns4_C3
full k4_fill C5 k4_fill_C5
full k4_place C5 k4_place_C5
: > gpurun_out/ev_shards.jsonl
for c in C5 C4 C3; do
  python tools/shard_step.py $c 1 0 >> gpurun_out/ev_shards.jsonl 2>/dev/null
  python tools/shard_step.py $c 2 0 1 >> gpurun_out/ev_shards.jsonl 2>/dev/null
  python tools/shard_step.py $c 4 0 3 >> gpurun_out/ev_shards.jsonl 2>/dev/null
  python tools/shard_step.py $c 8 0 5 >> gpurun_out/ev_shards.jsonl 2>/dev/null
done
[ "$1" = "--ref-full" ] && python tools/ref_full_c5.py > gpurun_out/ev_ref_full_c5.json 2> gpurun_out/ev_ref_full_c5.err
tail -c 600 gpurun_out/ev_bench_C5.json; echo; head -c 400 gpurun_out/ev_ref.json; echo; cat gpurun_out/ev_shards.jsonl
