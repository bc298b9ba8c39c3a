python -m pytest tests/test_gpu_shard.py tests/test_gpu_adapter.py tests/test_gpu_api.py tests/test_gpu_solver.py tests/test_gpu_text.py tests/test_gpu_triplets.py tests/test_gpu_unstructured.py tests/test_gpu_boundary.py tests/test_gpu_parity.py -x -q > gpurun_out/t11.log 2>&1; tail -4 gpurun_out/t11.log
bash tools/quick.sh C4 C5 C3 > gpurun_out/q11.log 2>&1; cat gpurun_out/q11.log
