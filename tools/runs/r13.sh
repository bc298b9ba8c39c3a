for cn in 64 8 1; do echo "== FL_CELL_NODES=$cn"; FL_CELL_NODES=$cn bash tools/quick.sh C4 C5 C3; done > gpurun_out/q13.log 2>&1; cat gpurun_out/q13.log
