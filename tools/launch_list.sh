#!/bin/bash
# usage: tools/launch_list.sh CONFIG...  -> gpurun_out/ll_<cfg>.csv (one assemble_system step)
for c in "$@"; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      python tools/one_step.py $c 1 > gpurun_out/ll_$c.csv 2>/dev/null
done
