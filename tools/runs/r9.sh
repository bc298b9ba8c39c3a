python -m pytest tests -m gpu -x -q > gpurun_out/t9.log 2>&1; tail -25 gpurun_out/t9.log
