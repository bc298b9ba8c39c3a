python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py tests/test_gpu_api.py -x -q > gpurun_out/t12.log 2>&1; tail -3 gpurun_out/t12.log
bash tools/quick.sh C4 C5 C3 > gpurun_out/q12.log 2>&1; cat gpurun_out/q12.log
FL_PLAN=d bash tools/quick.sh C5 > gpurun_out/q12d.log 2>&1; cat gpurun_out/q12d.log
bash tools/launch_list.sh C5
